"""Repro of one random fuzz program on the GPU (evaluate, then predict)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import torch
from fuzz_programs import random_bindings, random_program
import paper_1604_04997_b200 as kc
seed = int(sys.argv[1])
p = kc.Program(random_program(seed))
if len(sys.argv) > 2:
    p.set_engine(sys.argv[2])
bs = random_bindings(seed, p.params, 150)
cols = {q: torch.tensor([b[q] for b in bs], dtype=torch.int64, device="cuda") for q in p.params}
bb = kc.evaluate_properties(p, cols, wide=True)
torch.cuda.synchronize()
print("evaluate ok", flush=True)
w = kc.ModelWeights(alpha=[1e-12 * (1 + i % 7) for i in range(149)], covered=[True] * 149)
pred, st = kc.predict(w, p, cols, with_status=True)
torch.cuda.synchronize()
print("predict ok", flush=True)
