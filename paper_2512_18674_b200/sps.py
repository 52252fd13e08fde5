"""Thin ctypes binding of include/remoe.h (argument marshalling only).

Every step of the SPS path runs in libremoe.so's CUDA kernels; this module only
turns torch tensors / numpy arrays into pointers, picks the current CUDA stream,
and raises on non-OK status.  There is no CPU fallback: if libremoe.so is
missing or no GPU is visible, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libremoe.so")

REMOE_OK = 0
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "CUDA", 3: "NCCL", 4: "OOM", 5: "UNSUPPORTED", 6: "STATE"}
KERNEL_AUTO, KERNEL_STREAM, KERNEL_TC, KERNEL_PAIR = 0, 1, 2, 3

# every function declared in include/remoe.h
ABI_FUNCTIONS = (
    "remoe_sps_config_default", "remoe_sps_build", "remoe_sps_query", "remoe_sps_query_host",
    "remoe_expert_plan", "remoe_nccl_unique_id", "remoe_sps_sync", "remoe_sps_get_info",
    "remoe_sps_set_kernel", "remoe_sps_profile", "remoe_sps_destroy", "remoe_status_string",
    "remoe_last_error", "remoe_sps_embed", "remoe_js_divergence",
    "remoe_sps_tree_build", "remoe_sps_tree_info", "remoe_sps_tree_export", "remoe_sps_tree_query",
    "remoe_loopback_group_create", "remoe_loopback_group_destroy", "remoe_sps_query_group",
)


class RemoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class TreeInfo(ctypes.Structure):
    _fields_ = [
        ("n_nodes", ctypes.c_int32),
        ("n_leaves", ctypes.c_int32),
        ("depth", ctypes.c_int32),
        ("max_leaf", ctypes.c_int32),
        ("beta", ctypes.c_int32),
        ("branching", ctypes.c_int32),
        ("build_ms", ctypes.c_double),
    ]


class SpsConfig(ctypes.Structure):
    _fields_ = [
        ("n_local", ctypes.c_int64),
        ("global_offset", ctypes.c_int64),
        ("dim", ctypes.c_int32),
        ("n_layers", ctypes.c_int32),
        ("n_experts", ctypes.c_int32),
        ("sigma", ctypes.c_float),
        ("temperature", ctypes.c_float),
        ("max_batch", ctypes.c_int32),
        ("max_k", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
        ("inputs_on_device", ctypes.c_int32),
        ("validate", ctypes.c_int32),
        ("loopback_group", ctypes.c_void_p),
    ]


class SpsInfo(ctypes.Structure):
    _fields_ = [
        ("n_total", ctypes.c_int64),
        ("n_local", ctypes.c_int64),
        ("global_offset", ctypes.c_int64),
        ("dim", ctypes.c_int32),
        ("n_layers", ctypes.c_int32),
        ("n_experts", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("last_scan_kernel", ctypes.c_int32),
        ("last_launches", ctypes.c_int32),
        ("scan_ctas", ctypes.c_int32),
        ("device_bytes", ctypes.c_int64),
        ("fused_exchange", ctypes.c_int32),
        ("reserved_", ctypes.c_int32),
    ]


_LIB = None


def lib():
    """Load libremoe.so (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or "
                               "__graft_entry__.build(); there is no fallback path")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.remoe_sps_config_default.argtypes = [ctypes.POINTER(SpsConfig)]
        L.remoe_sps_config_default.restype = None
        L.remoe_sps_build.argtypes = [ctypes.POINTER(SpsConfig), vp, vp, ctypes.POINTER(vp)]
        L.remoe_sps_query.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp]
        L.remoe_sps_query_host.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp]
        L.remoe_expert_plan.argtypes = [vp, i32, i32, i32, i32, vp, vp]
        L.remoe_nccl_unique_id.argtypes = [vp]
        L.remoe_sps_sync.argtypes = [vp]
        L.remoe_sps_get_info.argtypes = [vp, ctypes.POINTER(SpsInfo)]
        L.remoe_sps_set_kernel.argtypes = [vp, i32]
        L.remoe_sps_profile.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_int64)]
        L.remoe_sps_embed.argtypes = [vp, vp, i32, i32, vp, vp, vp]
        L.remoe_js_divergence.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp]
        L.remoe_sps_tree_build.argtypes = [vp, i32, i32, i32, ctypes.c_uint64]
        L.remoe_sps_tree_info.argtypes = [vp, ctypes.POINTER(TreeInfo)]
        L.remoe_sps_tree_export.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.remoe_sps_tree_query.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp]
        L.remoe_loopback_group_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.remoe_loopback_group_destroy.argtypes = [vp]
        L.remoe_sps_query_group.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp]
        L.remoe_sps_destroy.argtypes = [vp]
        L.remoe_sps_destroy.restype = None
        L.remoe_status_string.argtypes = [i32]
        L.remoe_status_string.restype = ctypes.c_char_p
        L.remoe_last_error.argtypes = []
        L.remoe_last_error.restype = ctypes.c_char_p
        for f in ("remoe_sps_build", "remoe_sps_query", "remoe_sps_query_host", "remoe_expert_plan",
                  "remoe_nccl_unique_id", "remoe_sps_sync", "remoe_sps_get_info",
                  "remoe_sps_set_kernel", "remoe_sps_profile", "remoe_sps_embed",
                  "remoe_js_divergence", "remoe_sps_tree_build", "remoe_sps_tree_info",
                  "remoe_sps_tree_export", "remoe_sps_tree_query", "remoe_loopback_group_create",
                  "remoe_loopback_group_destroy", "remoe_sps_query_group"):
            getattr(L, f).restype = i32
        _LIB = L
    return _LIB


def _check(status: int):
    if status != REMOE_OK:
        raise RemoeError(status, lib().remoe_last_error().decode(errors="replace"))


def _ptr(t) -> int | None:
    """Raw pointer of a torch tensor or numpy array (None passes through)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags.c_contiguous, "array must be C-contiguous"
        return t.ctypes.data
    assert t.is_contiguous(), "tensor must be contiguous"
    return t.data_ptr()


def _stream(stream, device=None) -> int | None:
    """The stream to enqueue on: the given one, else torch's current stream of `device`
    (the handle's device -- not the current device, which may be another GPU)."""
    if stream is not None:
        return int(stream) if isinstance(stream, int) else stream.cuda_stream
    import torch
    return torch.cuda.current_stream(device).cuda_stream


# ------------------------------------------------------------------ C-ABI-named calls

def remoe_sps_config_default() -> SpsConfig:
    c = SpsConfig()
    lib().remoe_sps_config_default(ctypes.byref(c))
    return c


def remoe_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().remoe_nccl_unique_id(buf))
    return bytes(buf)


def remoe_sps_build(cfg: SpsConfig, emb_bf16, act, nccl_unique_id: bytes | None = None) -> int:
    """S0.  emb_bf16: uint16/int16/bfloat16 [n_local, D]; act: float32 [n_local, L, E]."""
    idbuf = None
    if nccl_unique_id is not None:
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_unique_id)
        cfg.nccl_unique_id = ctypes.cast(idbuf, ctypes.c_void_p)
    h = ctypes.c_void_p()
    _check(lib().remoe_sps_build(ctypes.byref(cfg), _ptr(emb_bf16), _ptr(act), ctypes.byref(h)))
    cfg.nccl_unique_id = None
    return h.value


def _dev(t):
    return t.device if getattr(t, "is_cuda", False) else None


def remoe_sps_query(h: int, q_bf16, B: int, k: int, ids, scores, pred=None, stream=None):
    """S1-S7 on device buffers (torch CUDA tensors)."""
    _check(lib().remoe_sps_query(h, _ptr(q_bf16), B, k, _ptr(ids), _ptr(scores), _ptr(pred),
                                 _stream(stream, _dev(ids))))


def remoe_loopback_group_create(world: int) -> int:
    """An empty loopback group of `world` ranks (one process, one device; test harness of
    the multi-rank exchange, include/remoe.h)."""
    g = ctypes.c_void_p()
    _check(lib().remoe_loopback_group_create(world, ctypes.byref(g)))
    return g.value


def remoe_loopback_group_destroy(g: int):
    _check(lib().remoe_loopback_group_destroy(g))


def remoe_sps_query_group(g: int, q_bf16, B: int, k: int, ids, scores, pred=None, stream=None):
    """remoe_sps_query for every rank of a loopback group: ids/scores/pred are lists with
    one device tensor per rank (pred None: S6-S7 skipped)."""
    n = len(ids)
    arr = lambda ts: (ctypes.c_void_p * n)(*[_ptr(t) for t in ts])  # noqa: E731
    _check(lib().remoe_sps_query_group(g, _ptr(q_bf16), B, k, arr(ids), arr(scores),
                                       arr(pred) if pred is not None else None,
                                       _stream(stream, _dev(ids[0]))))


def remoe_sps_query_host(h: int, q_bf16, B: int, k: int, ids, scores, pred=None, stream=None, device=None):
    """S1-S7 on host buffers (numpy or pinned CPU tensors); synchronous."""
    _check(lib().remoe_sps_query_host(h, _ptr(q_bf16), B, k, _ptr(ids), _ptr(scores), _ptr(pred),
                                      _stream(stream, device)))


def remoe_expert_plan(pred, B: int, L: int, E: int, n_cold: int, cold_mask, stream=None):
    """S8 on device buffers."""
    _check(lib().remoe_expert_plan(_ptr(pred), B, L, E, n_cold, _ptr(cold_mask), _stream(stream, _dev(pred))))


def remoe_sps_sync(h: int):
    _check(lib().remoe_sps_sync(h))


def remoe_sps_get_info(h: int) -> SpsInfo:
    info = SpsInfo()
    _check(lib().remoe_sps_get_info(h, ctypes.byref(info)))
    return info


def remoe_sps_set_kernel(h: int, which: int):
    _check(lib().remoe_sps_set_kernel(h, which))


def remoe_sps_profile(h: int, enable: bool) -> tuple[float, int]:
    """Scan-kernel time (ms) and launches since the previous call; toggles recording."""
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    _check(lib().remoe_sps_profile(h, 1 if enable else 0, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def remoe_sps_embed(tokens_bf16, offsets, n_prompts: int, dim: int, out_bf16=None, out_f32=None,
                    stream=None):
    """NEXT-N1: prompt vectors a_p = sum_t x_t / |x_t| from token embeddings (device buffers)."""
    _check(lib().remoe_sps_embed(_ptr(tokens_bf16), _ptr(offsets), n_prompts, dim, _ptr(out_bf16),
                                 _ptr(out_f32), _stream(stream, _dev(tokens_bf16))))


def embed(tokens_bf16, offsets, want_f32=False, stream=None):
    """Torch convenience: tokens [T, D] (int16/uint16 bf16 bits, CUDA), offsets [P+1] int64 (CUDA).
    Returns (bf16 bits [P, D] as int16, fp32 [P, D] or None)."""
    import torch
    P = offsets.shape[0] - 1
    D = tokens_bf16.shape[1]
    ob = torch.empty((P, D), dtype=torch.int16, device=tokens_bf16.device)
    of = torch.empty((P, D), dtype=torch.float32, device=tokens_bf16.device) if want_f32 else None
    remoe_sps_embed(tokens_bf16, offsets, P, D, ob, of, stream)
    return ob, of


def remoe_js_divergence(P, Q, shared_q: bool, B: int, L: int, E: int, out, stream=None):
    """NEXT-N4: out[b] = mean_l JS_2(P[b,l], Q[b,l] or Q[l]) on device buffers."""
    _check(lib().remoe_js_divergence(_ptr(P), _ptr(Q), 1 if shared_q else 0, B, L, E, _ptr(out),
                                     _stream(stream, _dev(P))))


def js_divergence(P, Q, stream=None):
    """Torch convenience: P [B, L, E], Q [B, L, E] or [L, E] (CUDA fp32) -> [B] fp32."""
    import torch
    B, L, E = P.shape
    out = torch.empty(B, dtype=torch.float32, device=P.device)
    remoe_js_divergence(P, Q, Q.dim() == 2, B, L, E, out, stream)
    return out


def remoe_sps_tree_build(h: int, beta: int, branching: int, max_iter: int, seed: int):
    """NEXT-N2: build the clustering tree over the handle's shard (synchronous)."""
    _check(lib().remoe_sps_tree_build(h, beta, branching, max_iter, seed & ((1 << 64) - 1)))


def remoe_sps_tree_info(h: int) -> TreeInfo:
    info = TreeInfo()
    _check(lib().remoe_sps_tree_info(h, ctypes.byref(info)))
    return info


def remoe_sps_tree_export(h: int, n_local: int) -> dict:
    """The tree as numpy arrays (host copies)."""
    n = remoe_sps_tree_info(h).n_nodes
    out = dict(perm=np.empty(n_local, np.int64), begin=np.empty(n, np.int64), end=np.empty(n, np.int64),
               parent=np.empty(n, np.int32), child0=np.empty(n, np.int32), nchild=np.empty(n, np.int32),
               medoid=np.empty(n, np.int64))
    _check(lib().remoe_sps_tree_export(h, *(out[f].ctypes.data for f in
                                             ("perm", "begin", "end", "parent", "child0", "nchild", "medoid"))))
    return out


def remoe_sps_tree_query(h: int, q_bf16, B: int, k: int, ids, scores, pred=None, leaf=None, n_eval=None,
                         stream=None):
    """NEXT-N2: Algorithm 1 + S6/S7 on device buffers."""
    _check(lib().remoe_sps_tree_query(h, _ptr(q_bf16), B, k, _ptr(ids), _ptr(scores), _ptr(pred), _ptr(leaf),
                                      _ptr(n_eval), _stream(stream, _dev(ids))))


def remoe_sps_destroy(h: int):
    if h:
        lib().remoe_sps_destroy(h)


# ------------------------------------------------------------------ convenience wrapper

class Sps:
    """Owns one handle.  Tensors in, tensors out (torch on the handle's device)."""

    def __init__(self, emb_bf16, act, *, sigma=1e-6, temperature=1.0, max_batch=256, max_k=128,
                 device=0, rank=0, world=1, global_offset=0, nccl_unique_id=None, validate=True,
                 loopback_group=None):
        import torch
        cfg = remoe_sps_config_default()
        n, d = emb_bf16.shape
        cfg.n_local, cfg.global_offset, cfg.dim = n, global_offset, d
        cfg.n_layers, cfg.n_experts = act.shape[1], act.shape[2]
        cfg.sigma, cfg.temperature = sigma, temperature
        cfg.max_batch, cfg.max_k = max_batch, max_k
        cfg.device, cfg.rank, cfg.world = device, rank, world
        cfg.validate = 1 if validate else 0
        cfg.loopback_group = loopback_group
        on_dev = isinstance(emb_bf16, torch.Tensor) and emb_bf16.is_cuda
        cfg.inputs_on_device = 1 if on_dev else 0
        self.device = torch.device("cuda", device)
        self.dim, self.layers, self.experts = d, act.shape[1], act.shape[2]
        self.n_local = n
        self.handle = remoe_sps_build(cfg, emb_bf16, act, nccl_unique_id)

    def query(self, q_bf16, k, want_pred=True, stream=None):
        import torch
        B = q_bf16.shape[0]
        ids = torch.empty((B, k), dtype=torch.int64, device=self.device)
        scores = torch.empty((B, k), dtype=torch.float32, device=self.device)
        pred = (torch.empty((B, self.layers, self.experts), dtype=torch.float32, device=self.device)
                if want_pred else None)
        remoe_sps_query(self.handle, q_bf16, B, k, ids, scores, pred, stream)
        return ids, scores, pred

    def query_host(self, q_bf16: np.ndarray, k: int, want_pred=True, stream=None):
        B = q_bf16.shape[0]
        ids = np.empty((B, k), np.int64)
        scores = np.empty((B, k), np.float32)
        pred = np.empty((B, self.layers, self.experts), np.float32) if want_pred else None
        remoe_sps_query_host(self.handle, q_bf16, B, k, ids, scores, pred, stream, self.device)
        return ids, scores, pred

    def tree_build(self, beta=150, branching=8, max_iter=10, seed=0):
        """NEXT-N2: the clustering tree; alpha = k of tree_query."""
        remoe_sps_tree_build(self.handle, beta, branching, max_iter, seed)
        return remoe_sps_tree_info(self.handle)

    def tree_info(self) -> TreeInfo:
        return remoe_sps_tree_info(self.handle)

    def tree_export(self) -> dict:
        return remoe_sps_tree_export(self.handle, self.n_local)

    def tree_query(self, q_bf16, k, want_pred=True, stream=None):
        """Algorithm 1: returns ids, scores, pred (or None), leaf [B], n_eval [B]."""
        import torch
        B = q_bf16.shape[0]
        ids = torch.empty((B, k), dtype=torch.int64, device=self.device)
        scores = torch.empty((B, k), dtype=torch.float32, device=self.device)
        pred = (torch.empty((B, self.layers, self.experts), dtype=torch.float32, device=self.device)
                if want_pred else None)
        leaf = torch.empty(B, dtype=torch.int32, device=self.device)
        n_eval = torch.empty(B, dtype=torch.int32, device=self.device)
        remoe_sps_tree_query(self.handle, q_bf16, B, k, ids, scores, pred, leaf, n_eval, stream)
        return ids, scores, pred, leaf, n_eval

    def plan(self, pred, n_cold, stream=None):
        import torch
        B, L, E = pred.shape
        mask = torch.empty((B, L, E), dtype=torch.uint8, device=pred.device)
        remoe_expert_plan(pred, B, L, E, n_cold, mask, stream)
        return mask

    def set_kernel(self, which: int):
        remoe_sps_set_kernel(self.handle, which)

    def info(self) -> SpsInfo:
        return remoe_sps_get_info(self.handle)

    def profile(self, enable: bool) -> tuple[float, int]:
        return remoe_sps_profile(self.handle, enable)

    def sync(self):
        remoe_sps_sync(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            remoe_sps_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """G ranks of one row-sharded store in ONE process on ONE device: the multi-rank path
    (key all-gather + merge, owner-side partial prediction, partial exchange) with device
    copies in place of NCCL (include/remoe.h "Loopback groups")."""

    def __init__(self, shards, acts, n_total: int, *, device=0, **kw):
        from .dist import shard_range
        self.world = len(shards)
        self.group = remoe_loopback_group_create(self.world)
        self.ranks = []
        try:
            for r, (x, a) in enumerate(zip(shards, acts)):
                off, n = shard_range(n_total, self.world, r)
                assert x.shape[0] == n, f"rank {r}: expected {n} rows, got {x.shape[0]}"
                self.ranks.append(Sps(x, a, device=device, rank=r, world=self.world, global_offset=off,
                                      loopback_group=self.group, **kw))
        except Exception:
            self.close()
            raise
        s0 = self.ranks[0]
        self.device, self.layers, self.experts = s0.device, s0.layers, s0.experts

    def query(self, q_bf16, k, want_pred=True, stream=None):
        """Every rank's (ids, scores, pred) as lists of device tensors (identical values)."""
        import torch
        B = q_bf16.shape[0]
        ids = [torch.empty((B, k), dtype=torch.int64, device=self.device) for _ in range(self.world)]
        scores = [torch.empty((B, k), dtype=torch.float32, device=self.device) for _ in range(self.world)]
        pred = ([torch.empty((B, self.layers, self.experts), dtype=torch.float32, device=self.device)
                 for _ in range(self.world)] if want_pred else None)
        remoe_sps_query_group(self.group, q_bf16, B, k, ids, scores, pred, stream)
        return ids, scores, pred

    def close(self):
        for s in getattr(self, "ranks", []):
            s.close()
        self.ranks = []
        if getattr(self, "group", None):
            remoe_loopback_group_destroy(self.group)
            self.group = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
