"""Parity helpers shared by the GPU tests (test infrastructure; imports the oracle).

Near-tie rule: GPU and oracle pivot sequences must be identical,
except that a divergence at step t is *documented* when the oracle's relative top-2 gap
there is below tau_t = max(1e-12, 4 (t+1) u max|U[0:t,:]| / a1).  The harness then forces
the oracle onto the GPU's pivot and keeps comparing from step t+1.
"""
import numpy as np

U_RND = 2.0 ** -53


def lupp_parity(gpu_piv, oracle_run, max_divergences=8):
    """oracle_run(forced) -> (piv, Lf, U, gaps).  Returns (oracle result, #documented near-ties).

    Raises AssertionError on an undocumented divergence."""
    gpu_piv = [int(x) for x in gpu_piv]
    forced = {}
    for _ in range(max_divergences + 1):
        piv, Lf, U, gaps = oracle_run(forced)
        diff = [t for t in range(len(gpu_piv)) if int(piv[t]) != gpu_piv[t] and t not in forced]
        if not diff:
            return (piv, Lf, U, gaps), len(forced)
        t = diff[0]
        a1 = abs(U[t, t]) if abs(U[t, t]) > 0 else 1.0
        umax = float(np.max(np.abs(U[:t]))) if t > 0 else 0.0
        tau = max(1e-12, 4 * (t + 1) * U_RND * umax / a1)
        assert gaps[t] < tau, (
            f"pivot divergence at step {t}: gpu {gpu_piv[t]} vs oracle {int(piv[t])}, "
            f"oracle gap {gaps[t]:.3e} >= tau {tau:.3e}")
        forced[t] = gpu_piv[t]
    raise AssertionError("too many near-tie divergences")


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
