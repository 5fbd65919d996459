"""Size-independent digest of a full-size state, shared by the reference-run
generator (tests/golden/make_fullsize_refs.py) and the GPU test
(tests/test_gpu_fullsize.py)."""
import hashlib

import numpy as np

N_SAMPLE = 65536
N_BLOCKS = 1024
SAMPLE_SEED = 20251025


def sample_cells(n):
    """A seeded sample of cell ids whose final states are stored verbatim."""
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.sort(rng.choice(n, size=min(N_SAMPLE, n), replace=False)).astype(np.int64)


def sha256(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


def summarise(u):
    """SHA-256, per-variable L1 norm (sum |U_v| in cell order) and per-variable
    sums of U and |U| over N_BLOCKS contiguous cell blocks."""
    blocks = np.array_split(np.arange(u.shape[0]), N_BLOCKS)
    return dict(sha256=sha256(u), l1=np.abs(u).sum(0),
                block_sum=np.array([u[b].sum(0) for b in blocks]),
                block_abs=np.array([np.abs(u[b]).sum(0) for b in blocks]))
