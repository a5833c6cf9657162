"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):

* every kernel variant (E-sequential and sweep kNN, SIMPLEX / CCM / EMBED modes, library mode,
  padded global series, library-set masks, lags, smem and global lookups, table readback, the
  exact-tie fallback and a tie flood) runs under the CHECKED build (lib/libccm_checked.so,
  -DCCM_CHECKS: device-side bounds and invariant checks that trap) -- tools/sanitize_cases.py;
* scratch initialisation: results are byte-identical whether the workspace starts as 0x00 or
  0xFF bytes (no kernel reads scratch it did not write first; the initcheck question);
* determinism across repeated launches (no racy reductions)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2011_11082_b200 import build, libccm, synth
from tests.test_gpu_parity import dev

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_variant_under_device_checks():
    lib = build.build(checked=True)
    env = dict(os.environ, LIBCCM_PATH=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                         capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "sanitize cases done" in out.stdout
    assert "CCM_CHECK failed" not in out.stdout + out.stderr


def _poisoned(fn, kind, fill):
    libccm.release_workspaces()
    fn()  # allocates and caches the workspace
    torch.cuda.synchronize()
    for key, ws in libccm._ws_cache.items():
        ws.fill_(fill)
    r = fn()
    torch.cuda.synchronize()
    return r.cpu().numpy()


def test_results_independent_of_workspace_contents():
    build.build()
    libccm.load()
    data = synth.random_dataset(70, 300, 9)
    data[:, 3] = 1.25
    d = dev(data)
    E = libccm.simplex_optimal_E(d, 12)
    cases = [
        ("simplex", lambda: libccm.simplex_optimal_E(d, 12)),
        ("target", lambda: libccm.ccm_all_pairs(d, E, 1, 1, "target")),
        ("library", lambda: libccm.ccm_all_pairs(d, E, 1, 1, "library")),
        ("lagged", lambda: libccm.ccm_lagged(d, E, 1, -2, 1)),
        ("convergence", lambda: libccm.ccm_convergence(d, E, [20, 120], synth.library_orders(2, 300, 4))),
    ]
    for name, fn in cases:
        a = _poisoned(fn, name, 0)
        b = _poisoned(fn, name, 255)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), name
        c = fn().cpu().numpy()
        assert np.array_equal(a.view(np.uint32), c.view(np.uint32)), name
