"""Full-N optimal-E parity at BASELINE sizes (north_star: "bit-exact indices and E"): the GPU's
phase 1 (edm_simplex_optimal_E, Alg. 1 lines 2-10; argmax P:328) over EVERY
series of c3 (53,053 x 1,450) against the oracle's optE of every series, stored in
tests/golden/c3_optE_oracle.npz by tools/oracle_full_optE.py (which calls only oracle/; about
20 min on 8 host cores, so it is precomputed rather than run inside the test)."""
import os

import numpy as np
import pytest

from paper_2011_11082_b200 import libccm, synth
from tests.test_gpu_parity import dev

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2011_11082_b200 import build
    build.build()
    libccm.load()
    yield
    libccm.release_workspaces()


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_full_optE_bit_exact(config):
    path = os.path.join(GOLDEN, f"{config}_optE_oracle.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/oracle_full_optE.py --config {config})")
    z = np.load(path)
    cfg = synth.CONFIGS[config]
    data = synth.make_config(config)
    L, N = data.shape
    assert int(z["N"]) == N and int(z["L"]) == L and int(z["seed"]) == synth.SEED_BASE + int(config[1:])
    optE = libccm.simplex_optimal_E(dev(data), cfg["E_max"], cfg["tau"]).cpu().numpy()
    ref = z["optE"].astype(np.int32)
    bad = np.flatnonzero(optE != ref)
    assert bad.size == 0, f"{bad.size} of {N} series differ, e.g. {[(int(i), int(optE[i]), int(ref[i])) for i in bad[:5]]}"
