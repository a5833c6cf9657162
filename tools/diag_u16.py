import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2011_11082_b200 import libccm, synth
data = synth.make_config("c2", N=70, L=400).astype(np.float64)
j = 33
data[:, j] = 1.0 + 1e-7 * np.sin(np.arange(400) * 0.7)
data[0, j] = 5.0
data = data.astype(np.float32)
E = (1 + np.arange(70) % 4).astype(np.int32); E[j] = 3
d = torch.as_tensor(data).cuda(); Ed = torch.as_tensor(E).cuda()
q = libccm.ccm_all_pairs(d, Ed, 1, 1, "target", True, lookup="u16").cpu().numpy()
f = libccm.ccm_all_pairs(d, Ed, 1, 1, "target", True).cpu().numpy()
ref = O.ccm_rows(data, E, 1, 1, 0, True, 0, 70)
for name, g in (("u16", q), ("fp32", f)):
    e = np.abs(g - ref); e[np.isnan(e)] = 0
    idx = np.argwhere(e > 1e-4)
    print(name, "max", e.max(), "bad count", len(idx), idx[:10].tolist())
    print(" nan mismatch", np.argwhere(np.isnan(g) != np.isnan(ref))[:5].tolist())
print("vals", q[idx[:3,0], idx[:3,1]] if len(idx) else None)
print(np.unique(data[:, j])[:10], len(np.unique(data[:, j])))
