"""Per-tick latency of a long (rps=1) trajectory alone vs. among many."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2506_19677_b200 as S
from helpers import sim_config
for mode, cap in [(1, 10), (0, 0)]:
    for count in (1, 32, 1024, 8192):
        cfgs = [sim_config("w1", 1.0, 100, 42 + i, mode=mode, cap=cap) for i in range(count)]
        best = 1e9
        for _ in range(3):
            r = S.run_batch(cfgs)
            best = min(best, r.device_ms)
        ticks = r.rows["ticks"].max()
        print(f"mode {'static' if mode else 'saber '} count {count:5d} device {best:8.2f} ms  max ticks {ticks}  "
              f"{1e6 * best / 1e3 / ticks:7.3f} us/tick (slowest)")
