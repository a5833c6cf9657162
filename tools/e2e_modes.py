import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2011_11082_b200 import libccm, synth
data = synth.make_config("c3")
N = data.shape[1]
pinned = torch.empty((N, N), dtype=torch.float32).pin_memory().numpy()
page = np.empty((N, N), np.float32)
for mode in ("library", "target"):
    for name, buf in (("pinned", pinned), ("pageable", page), ("pinned", pinned)):
        t = time.perf_counter(); libccm.causal_map_host(data, 20, 1, 1, mode, True, rho_out=buf); print(mode, name, time.perf_counter() - t, flush=True)
