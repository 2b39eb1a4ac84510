"""GPU: the device generators against cuRAND (KAT) and against the oracle, bit for bit."""
import ctypes
import os

import numpy as np
import pytest

from oracle import omega
from oracle.philox import philox4x32_10

pytestmark = pytest.mark.gpu

PROBE = os.path.join(os.path.dirname(__file__), "librngprobe.so")


@pytest.fixture(scope="module")
def probe():
    if not os.path.exists(PROBE):
        pytest.fail("tests/librngprobe.so missing (python -m paper_2104_05877_b200.build)")
    lib = ctypes.CDLL(PROBE)
    lib.probe_philox.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.probe_gauss.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]
    lib.probe_sparse.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_void_p]
    return lib


def test_philox_matches_curand_and_oracle(probe):
    rng = np.random.default_rng(0)
    n = 4096
    inp = rng.integers(0, 2**32, size=(n, 6), dtype=np.uint64).astype(np.uint32)
    inp[0] = 0
    inp[1] = 0xFFFFFFFF
    out_cu = np.zeros((n, 4), dtype=np.uint32)
    out_sk = np.zeros((n, 4), dtype=np.uint32)
    assert probe.probe_philox(0, inp.ctypes.data, out_cu.ctypes.data, n) == 0
    assert probe.probe_philox(1, inp.ctypes.data, out_sk.ctypes.data, n) == 0
    np.testing.assert_array_equal(out_sk, out_cu)                     # library == cuRAND
    for r in range(16):
        o = philox4x32_10(*[int(inp[r, j]) for j in range(4)], int(inp[r, 4]), int(inp[r, 5]))
        assert [int(x) for x in o] == out_cu[r].tolist()              # oracle == cuRAND


@pytest.mark.parametrize("seed,l", [(2001, 40), (7, 13), (2**63 + 5, 522)])
def test_gaussian_omega_matches_oracle(probe, seed, l):
    m = 777
    z = np.zeros((l, m))
    assert probe.probe_gauss(seed, l, m, z.ctypes.data) == 0
    ref = omega.gaussian_z(seed, l, np.arange(m))
    np.testing.assert_allclose(z, ref, rtol=4e-16 * 8, atol=2e-15)


@pytest.mark.parametrize("l,zeta", [(510, 8), (16, 8), (40, 33), (9, 2)])
def test_sparse_structure_bitwise(probe, l, zeta):
    m = 3000
    rows = np.zeros((m, zeta), dtype=np.int32)
    sbits = np.zeros(m, dtype=np.uint64)
    assert probe.probe_sparse(2003, l, m, zeta, rows.ctypes.data, sbits.ctypes.data) == 0
    ref_rows, ref_signs = omega.sparse_sign_structure(2003, l, m, zeta)
    np.testing.assert_array_equal(rows, ref_rows)
    neg = ((sbits[:, None] >> np.arange(zeta, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(bool)
    np.testing.assert_array_equal(neg, ref_signs < 0)
