"""Order-independent 64-bit fingerprint of each box's skeleton set.

Test infrastructure: lets the full-size fixtures carry one uint64 per box
instead of the skeleton index lists, while the count of boxes whose skeleton
sets differ from the reference stays exact (up to 2^-64 collisions).
"""

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(x):
    """splitmix64 finaliser, vectorised (uint64 arithmetic wraps)."""
    z = x.astype(np.uint64) + _G
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def skel_set_hash(idx, counts):
    """Per segment (``counts`` consecutive entries of ``idx``) the wrapped sum
    of mixed indices: equal sets give equal hashes regardless of order."""
    idx = np.asarray(idx, dtype=np.int64)
    counts = np.asarray(counts, dtype=np.int64)
    with np.errstate(over="ignore"):
        h = _mix(idx)
        cs = np.zeros(idx.size + 1, dtype=np.uint64)
        np.cumsum(h, dtype=np.uint64, out=cs[1:])
        off = np.concatenate([[0], np.cumsum(counts)])
        return cs[off[1:]] - cs[off[:-1]]
