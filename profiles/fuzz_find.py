import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import torch
import kc_oracle as ko
from fuzz_programs import random_bindings, random_program
import paper_1604_04997_b200 as kc
from conftest import load_golden
start, stop = int(sys.argv[1]), int(sys.argv[2])
alpha = [1e-12 * (1 + i % 7) for i in range(149)]
w = kc.ModelWeights(alpha=alpha, covered=[True] * 149)
for seed in range(start, stop):
    text = random_program(seed)
    p = kc.Program(text)
    bs = random_bindings(seed, p.params, 150)
    cols = {q: torch.tensor([b[q] for b in bs], dtype=torch.int64, device="cuda") for q in p.params}
    print("seed", seed, flush=True)
    bb = kc.evaluate_properties(p, cols, wide=True)
    pred, st = kc.predict(w, p, cols, with_status=True)
    torch.cuda.synchronize()
print("all ok")
