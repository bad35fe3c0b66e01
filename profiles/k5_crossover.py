"""k-5 time of the pair kernel and the list-walk kernel over crowd density (1000 x 1000 su, eight directions, 7x7 fields):
where does the per-position walk overtake the per-event pairs?   python profiles/k5_crossover.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_04782_b200 import socfield as sf  # noqa: E402

for period in ("1..1", "1..3"):
    for rho in (0.02, 0.05, 0.1, 0.15, 0.2, 0.3, 0.5, 0.7, 0.9):
        row = []
        for path in ("pairs", "listwalk"):
            os.environ["SFC_K5_PATH"] = path
            cfg = sf.parse_scenario(f"grid = 1000x1000\ndensity = {rho}\ndirections = eight\nwalk_period = {period}\nseed = 42\nrebuild_interval = 0\n")
            eng = sf.Engine(cfg)
            P = eng.seed_resident(cfg)
            eng.step_resident(30)
            m = eng.step_resident(20, True)
            k5 = sum(x.phase_us[4] for x in m) / len(m)
            moved = sum(x.moved for x in m) / len(m)
            row.append((k5, moved))
            del eng
        print(f"period {period} rho {rho:4.2f} P {P:7d} moved/tick {row[0][1]:9.0f} ({row[0][1] / 1e6 * 2 * 49:5.2f} events per window)  "
              f"pairs {row[0][0]:7.1f} us  listwalk {row[1][0]:7.1f} us", flush=True)
