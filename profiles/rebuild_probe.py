import sys, time
sys.path.insert(0, "/root/repo")
import bench
from paper_1803_04782_b200 import socfield as sf
for wl in ("c4r", "c2", "paper1000"):
    w = bench.WORKLOADS[wl]
    cfg = sf.parse_scenario(w["text"])
    eng = sf.Engine(cfg)
    eng.seed_resident(cfg)
    eng.step_resident(30)            # ticks 0..29
    eng.step_resident(10); a = eng.counters()["last_run_ms"]   # 30..39: no rebuild
    eng.step_resident(10); b = eng.counters()["last_run_ms"]   # 40..49: rebuild after tick 49
    print(wl, "10 ticks without rebuild %.3f ms, with one rebuild %.3f ms -> rebuild %.3f ms" % (a, b, b - a))
