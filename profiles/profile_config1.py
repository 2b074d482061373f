"""Host-side profile of config 1 (campaign CSV -> fit -> 16 predictions): where the wall time goes."""
import cProfile
import pstats
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1604_04997_b200 as kc  # noqa: E402

golden = ROOT / "tests" / "golden"
kc.fit_from_csv(golden / "meas_sigma0.csv", device="simdev-v1")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    kc.fit_from_csv(golden / "meas_sigma0.csv", device="simdev-v1")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
