"""Philox4x32-10 counter-based RNG, plain numpy (TEST INFRASTRUCTURE ONLY).

Definition: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as
1, 2, 3" (SC'11), Philox-4x32 with R = 10 rounds.  One round maps the counter
(c0, c1, c2, c3) under key (k0, k1) to

    (hi(M1*c2) ^ c1 ^ k0,  lo(M1*c2),  hi(M0*c0) ^ c3 ^ k1,  lo(M0*c0))

with M0 = 0xD2511F53, M1 = 0xCD9E8D57; between rounds the key is bumped by the
Weyl constants (0x9E3779B9, 0xBB67AE85).  The paper only asks for i.i.d. draws
(P:176); the counter-based generator is the reading DESIGN.md §3 (R1)
takes so that Omega can be regenerated anywhere without being stored.

Pins: the Random123 known-answer vectors (tests/golden/philox_kat.txt) and, on
the GPU box, cuRAND's device ``curand_Philox4x32_10`` (tests/test_gpu_rng.py).
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Return the four 32-bit output words (as uint64 arrays) for the given counters.

    c0..c3 are broadcastable integer arrays (values < 2**32); k0, k1 python ints.
    """
    c = [np.asarray(x, dtype=np.uint64) & MASK32 for x in (c0, c1, c2, c3)]
    c = np.broadcast_arrays(*c)
    c = [x.copy() for x in c]
    key0, key1 = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for rnd in range(10):
        if rnd > 0:
            key0 = (key0 + W0) & 0xFFFFFFFF
            key1 = (key1 + W1) & 0xFFFFFFFF
        p0 = M0 * c[0]            # < 2**64, exact in uint64
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c = [hi1 ^ c[1] ^ np.uint64(key0), lo1, hi0 ^ c[3] ^ np.uint64(key1), lo0]
    return c


def uniform53(w_hi, w_lo):
    """Two 32-bit words -> a double in (0, 1] with 53 random bits (R2).

    u = ((w_hi >> 5) * 2**26 + (w_lo >> 6) + 0.5) * 2**-53.  The integer part is exact;
    adding 0.5 rounds to nearest-even once the integer exceeds 2**52, so the largest
    value is exactly 1.0 and the smallest 2**-54 (never 0, so log(u) is finite).
    """
    a = (np.asarray(w_hi, dtype=np.uint64) >> np.uint64(5)).astype(np.float64)
    b = (np.asarray(w_lo, dtype=np.uint64) >> np.uint64(6)).astype(np.float64)
    return (a * 67108864.0 + b + 0.5) * (1.0 / 9007199254740992.0)
