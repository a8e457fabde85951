"""Diagnostic: leave a live device-merge run with chains in flight (objects
kept alive, as a failing pytest's traceback does), then run the Appendix-B
tee and print rows whose logits miss the oracle.
Usage: python tools/debug_contam.py <device_merges 0|1> <iterations> [runs]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from debug_tee_bad import run  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_live_parity import _live_run  # noqa: E402

dm = bool(int(sys.argv[1]))
iters = int(sys.argv[2])
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2

import paper_2603_12831_b200.live as live  # noqa: E402

orig = live.LiveEngine.run_live


def capped(self, *a, **k):
    k["max_iterations"] = iters
    return orig(self, *a, **k)


live.LiveEngine.run_live = capped
keep = _live_run(2, 1, device_merges=dm)
print("phase 1:", keep[4], "iterations, counters", {k: keep[2].counters[k] for k in
                                                      ("tokens_total", "merges")}, flush=True)
for k in range(runs):
    t = run()
    print(f"run {k}: max_rel={t.max_rel:.3e} bad={len(t.bad)} ties={t.ties} "
          f"n_bad_rows={len(t.rows)}", flush=True)
    for r in t.rows[:12]:
        print("   ", r, flush=True)
