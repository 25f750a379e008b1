"""Philox4x32-10 counter-based generator, plain numpy (TEST INFRASTRUCTURE ONLY).

The paper says only "randomly sample" the negative class centres (§3.2.2 step 3) and
names no generator. DESIGN.md reading R2 fixes it to Philox4x32-10 (Salmon et al., "Parallel random
numbers: as easy as 1, 2, 3", SC'11 — the Random123 definition) so that the sampled index set is a
pure function of (seed, step, global class id) and is reproducible on any partition.

Definition (Random123, 10 rounds):
    round:  (hi0, lo0) = mulhilo32(M0, c0);  (hi1, lo1) = mulhilo32(M1, c2)
            c = (hi1 ^ c1 ^ k0,  lo1,  hi0 ^ c3 ^ k1,  lo0)
    key bump between rounds:  k0 += W0;  k1 += W1   (mod 2^32)
with M0 = 0xD2511F53, M1 = 0xCD9E8D57, W0 = 0x9E3779B9, W1 = 0xBB67AE85.

Pinned by the Random123 known-answer vectors in tests/golden/philox_kat.txt (tests/test_oracle_pins.py).
"""
import numpy as np

_MASK = np.uint64(0xFFFFFFFF)
_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10. Every argument is an array (or scalar) of 32-bit values; returns 4
    uint64 arrays holding the 32-bit output words (x, y, z, w)."""
    c0, c1, c2, c3, k0, k1 = (np.asarray(v, dtype=np.uint64) & _MASK for v in (c0, c1, c2, c3, k0, k1))
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0 = _M0 * c0          # < 2^64: exact in uint64
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def class_key(global_ids, seed, step):
    """h_j of DESIGN.md reading R2/R3: the first output word of
    Philox4x32-10(ctr = {j mod 2^32, j >> 32, step mod 2^32, 0}, key = {seed mod 2^32, seed >> 32}).
    Depends only on (seed, step, j): never on the partition."""
    j = np.asarray(global_ids, dtype=np.uint64)
    seed = int(seed)
    x, _, _, _ = philox4x32_10(j & _MASK, j >> _S32, np.uint64(int(step) & 0xFFFFFFFF), np.uint64(0),
                               np.uint64(seed & 0xFFFFFFFF), np.uint64((seed >> 32) & 0xFFFFFFFF))
    return x
