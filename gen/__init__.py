"""Seeded synthetic SPS workload generator (inputs only; see gen/gen.c).

Shared by the oracle side and the CUDA side.  Holds none of the method's
arithmetic.  Configs mirror BASELINE.json ``configs``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STORE_SEED = 251218674  # the arXiv id (SURVEY.md §8(d) "Seeds")


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build()) first")
        lib = ctypes.CDLL(path)
        i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        vp = ctypes.c_void_p
        lib.gen_store_emb.argtypes = [u64, i64, i64, i64, i32, vp, i32]
        lib.gen_store_act.argtypes = [u64, i64, i64, i64, i32, i32, i32, vp, i32]
        lib.gen_queries.argtypes = [u64, u64, i64, i32, i64, i32, vp, i32]
        lib.gen_query_source_row.argtypes = [u64, i64, i64, i32]
        lib.gen_query_source_row.restype = i64
        lib.gen_cluster_of.argtypes = [u64, i64, i64]
        lib.gen_cluster_of.restype = i64
        lib.gen_num_clusters.argtypes = [i64]
        lib.gen_num_clusters.restype = i64
        _LIB = lib
    return _LIB


def _threads() -> int:
    return max(1, os.cpu_count() or 1)


@dataclass(frozen=True)
class Config:
    """One workload shape (BASELINE.json configs; SURVEY.md §8 'Configs')."""
    name: str
    n: int          # N, stored prompts
    dim: int        # D
    layers: int     # L (MoE layers)
    experts: int    # E (routed experts per layer; shared experts excluded)
    moe_topk: int   # N^topk
    batch: int      # default B
    k: int          # alpha
    index: int      # seed offset

    @property
    def store_seed(self) -> int:
        return STORE_SEED + self.index

    @property
    def query_seed(self) -> int:
        return self.store_seed + 1


CONFIGS = {
    "tiny": Config("tiny", 1_000, 384, 32, 8, 2, 16, 5, 0),
    "c2": Config("c2", 100_000, 768, 27, 64, 6, 64, 10, 1),
    "c3": Config("c3", 1_000_000, 1024, 24, 60, 4, 64, 16, 2),
    "c4": Config("c4", 10_000_000, 1024, 32, 8, 2, 1, 32, 3),
    "c5": Config("c5", 1_000_000, 1024, 24, 60, 4, 256, 16, 2),  # the c3 store
    # p0: the paper's own SPS scale (PAPER.md:675, 5,000 history, alpha=15); context only
    "p0_gpt2": Config("p0_gpt2", 5_000, 768, 12, 8, 2, 1, 15, 5),
    "p0_dsv2": Config("p0_dsv2", 5_000, 2048, 26, 64, 6, 1, 15, 6),
}


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard of rank: [offset, offset+n_local), the
    balanced split offset_g = floor(n_total * g / world): no shard is empty for n >= world."""
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def num_clusters(n_total: int) -> int:
    return int(_lib().gen_num_clusters(n_total))


def cluster_of(seed: int, n_total: int, row: int) -> int:
    return int(_lib().gen_cluster_of(seed, n_total, row))


def store_emb(seed: int, n_total: int, dim: int, row0: int = 0, nrows: int | None = None,
              out: np.ndarray | None = None) -> np.ndarray:
    """bf16 bits (uint16) [nrows, dim] of rows [row0, row0+nrows)."""
    if nrows is None:
        nrows = n_total - row0
    if out is None:
        out = np.empty((nrows, dim), dtype=np.uint16)
    assert out.dtype == np.uint16 and out.flags.c_contiguous and out.shape == (nrows, dim)
    rc = _lib().gen_store_emb(seed, n_total, row0, nrows, dim, out.ctypes.data, _threads())
    if rc:
        raise ValueError(f"gen_store_emb failed ({rc})")
    return out


def store_act(seed: int, n_total: int, layers: int, experts: int, moe_topk: int,
              row0: int = 0, nrows: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """fp32 [nrows, L, E] activation tables, rows sum to 1 per (prompt, layer)."""
    if nrows is None:
        nrows = n_total - row0
    if out is None:
        out = np.empty((nrows, layers, experts), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous
    rc = _lib().gen_store_act(seed, n_total, row0, nrows, layers, experts, moe_topk,
                              out.ctypes.data, _threads())
    if rc:
        raise ValueError(f"gen_store_act failed ({rc})")
    return out


def queries(store_seed: int, query_seed: int, n_total: int, dim: int, batch: int,
            mode: int = 0) -> np.ndarray:
    """bf16 bits [B, dim]; mode 0 = fresh cluster members, 1 = correctness mix."""
    out = np.empty((batch, dim), dtype=np.uint16)
    rc = _lib().gen_queries(store_seed, query_seed, n_total, dim, batch, mode,
                            out.ctypes.data, _threads())
    if rc:
        raise ValueError(f"gen_queries failed ({rc})")
    return out


def query_source_row(query_seed: int, n_total: int, i: int, mode: int = 1) -> int:
    return int(_lib().gen_query_source_row(query_seed, n_total, i, mode))


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float32 (shift into the high half)."""
    return (bits.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bits (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


def token_prompts(seed: int, n_prompts: int, dim: int, min_len: int = 1, max_len: int = 64,
                  n_topics: int = 8, zero_token_every: int = 0):
    """Synthetic token-embedding matrices for the Eq. 11 front end (NEXT-N1).

    Prompt p draws a topic; its tokens are topic centroid + unit noise, so prompts of a
    topic have high SCS.  Returns (tokens bf16 bits [T, dim], offsets int64 [P+1], topic [P]).
    Host-only numpy (PCG64 seeded): inputs, no method arithmetic."""
    rng = np.random.default_rng(seed)
    cent = rng.standard_normal((n_topics, dim))
    lens = rng.integers(min_len, max_len + 1, size=n_prompts)
    topic = rng.integers(0, n_topics, size=n_prompts)
    offsets = np.zeros(n_prompts + 1, np.int64)
    offsets[1:] = np.cumsum(lens)
    tok = np.empty((int(offsets[-1]), dim), np.float32)
    for p in range(n_prompts):
        a, b = offsets[p], offsets[p + 1]
        tok[a:b] = cent[topic[p]] + rng.standard_normal((b - a, dim))
    if zero_token_every:
        tok[::zero_token_every] = 0.0
    return f32_to_bf16_bits(tok), offsets, topic
