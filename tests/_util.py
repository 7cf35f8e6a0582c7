"""Shared test helpers (hashing, small graph builders via the oracle)."""

import hashlib

import numpy as np

import oracle


def sha(a, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()[:32]


def pairs_arrays(pairs):
    arr = np.array(pairs, dtype=np.uint32).reshape(-1, 2)
    return arr[:, 0].copy(), arr[:, 1].copy()


def oracle_csr_from_pairs(pairs, n, symmetrize=True, dedup=True):
    s, d = pairs_arrays(pairs)
    return oracle.build_csr(n, s, d, symmetrize, dedup)


def layers_tuples(layers):
    return [tuple(x) if not hasattr(x, "input") else (x.input, x.edges, x.discovered) for x in layers]
