import sys, torch
sys.path.insert(0, '.')
import paper_1604_04997_b200 as kc
F, n = int(sys.argv[1]), int(sys.argv[2])
X = torch.rand((n, F), dtype=torch.float64, device='cuda') * 9999 + 1
st = kc.gram_accumulate(X); torch.cuda.synchronize()
print(F, n, float(((st.G - X.T @ X).abs() / (X.T @ X)).max()))
