"""The integer-sliced Gram on the int8 tensor cores (gram_sliced.cu, opt-in
through KCG_GRAM_SLICED=1): G within 1e-13 of sum_r |x_ri||x_rj| of torch's
fp64 product, X^T 1 within 1e-13 of sum |x|, exact column maxima -- on
tails, segment breaks (rising magnitudes), zero / signed / 1e+-140 columns,
and NaN propagation from a non-finite input. The knob is read once per
process, so the cases run in a subprocess."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_sliced_gram_parity():
    env = dict(os.environ, KCG_GRAM_SLICED="1")
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "gram_sliced_case.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["cases"] >= 30 and not out["bad"]
