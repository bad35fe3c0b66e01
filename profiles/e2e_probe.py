import sys, time
sys.path.insert(0, "/root/repo")
import bench
from paper_1803_04782_b200 import socfield as sf
cfg, state = bench.build_state(sf, bench.WORKLOADS["c2"])
eng = sf.Engine(cfg)
for _ in range(3):
    eng.run(state, 100)
def t(f, n=5):
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e3
print("upload ms", t(lambda: eng.upload(state)))
print("step_resident(100) ms", t(lambda: eng.step_resident(100)))
print("download ms", t(lambda: eng.download(state)))
print("verify_state ms", t(lambda: eng.verify_state(state)))
print("run(100) ms", t(lambda: eng.run(state, 100)))
