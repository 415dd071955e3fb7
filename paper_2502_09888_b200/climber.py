"""Thin ctypes binding of libclimber.so (include/climber.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  PyTorch provides device memory (the arena, inputs, outputs) and
the CUDA stream.  If the library is missing this module raises — there is no
CPU or eager fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CLIMBER_LIB: another build of the library (A/B measurements); default in-tree
LIB_PATH = os.environ.get("CLIMBER_LIB") or os.path.join(_HERE, "lib", "libclimber.so")

ABI_VERSION = 2
BF16, FP32 = 0, 1
STATUS = {0: "OK", 1: "E_INVALID_ARG", 2: "E_CONFIG", 3: "E_OUT_OF_RANGE", 4: "E_UNSORTED",
          5: "E_CAPACITY", 6: "E_STALE", 7: "E_CUDA", 8: "E_NCCL", 9: "E_NUMERIC", 10: "E_UNSUPPORTED"}


class ClimberError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "abi_version", "d", "n_heads", "n_layers", "n_blocks", "n_k", "ffn_mult", "se_reduction", "vocab",
        "n_actions", "n_scenarios", "max_candidates", "hist_causal", "dtype", "page_tokens")] + [
        ("rms_eps", C.c_float), ("max_batch_users", C.c_int32), ("max_wave_users", C.c_int32),
        ("max_wave_pairs", C.c_int32), ("kv_pages", C.c_int64), ("rel_bias", C.c_int32)]


class _Strategy(C.Structure):
    _fields_ = [("action_mask", C.c_uint64), ("scenario_mask", C.c_uint64)]


class _Events(C.Structure):
    _fields_ = [("item", C.c_void_p), ("action", C.c_void_p), ("scenario", C.c_void_p), ("ts", C.c_void_p)]


WEIGHT_NAMES = ("emb_item", "emb_act", "emb_scn", "g1", "w_qkv", "w_o", "g2", "w1", "w2", "tau", "f_g1", "f_w_qkv",
                "f_w_o", "f_g2", "f_w1", "f_w2", "tau_f", "w_se1", "b_se1", "w_se2", "b_se2", "w_head")


class _Weights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in WEIGHT_NAMES] + [("b_head", C.c_float), ("b_pos", C.c_void_p),
                                                          ("b_time", C.c_void_p)]


_LIB = None


def lib() -> C.CDLL:
    """Load libclimber.so (raises if it has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, VP = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p
        sig = {
            "climber_arena_bytes": (C.c_size_t, [P]),
            "climber_create": (I32, [P, P, P, VP, C.c_size_t, I32, I32, VP, P]),
            "climber_destroy": (I32, [VP]),
            "climber_encode_user": (I32, [VP, P, I64, I32, VP, P]),
            "climber_encode_users": (I32, [VP, I32, P, P, P, VP, P]),
            "climber_score_items": (I32, [VP, VP, VP, I32, VP, VP]),
            "climber_score_items_batched": (I32, [VP, I32, P, P, VP, VP, VP]),
            "climber_rank_host": (I32, [VP, I32, P, P, P, P, P, P, P, P, P, VP]),
            "climber_kv_release": (I32, [VP, VP]),
            "climber_kv_broadcast": (I32, [VP, P, I32, VP]),
            "climber_stream_status": (I32, [VP, VP]),
            "climber_last_error": (C.c_char_p, []),
            "climber_debug_extract": (I32, [VP, VP, P, P]),
            "climber_debug_mask": (I32, [VP, VP, I32, P]),
            "climber_debug_kv": (I32, [VP, VP, I32, I32, P, P]),
            "climber_debug_attn_probe": (I32, [VP, VP, I32, I32, I32, I32, I32, P]),
            "climber_launch_count": (I64, [VP]),
            "climber_debug_gemm": (I32, [VP, VP, VP, I64, I32, I32, I32, I32, VP]),
            "climber_profile": (I32, [VP, I32]),
            "climber_kv_slab_bytes": (C.c_size_t, [VP]),
            "climber_kv_export": (I32, [VP, VP, VP, VP]),
            "climber_kv_import": (I32, [VP, VP, I32, VP, P]),
            "climber_profile_read": (I32, [VP, P]),
            "climber_encode_users_blocks": (I32, [VP, I32, P, P, P, I32, I32, VP, P]),
            "climber_score_blocks": (I32, [VP, I32, P, P, VP, I32, I32, VP, VP]),
            "climber_fuse_scores": (I32, [VP, I32, P, P, I32, VP, VP, VP]),
            "climber_forward": (I32, [VP, I32, P, P, P, P, VP, VP, VP]),
            "climber_cache_acquire": (I32, [VP, C.c_uint64, I32, C.c_uint64, P, I64, VP, P, P]),
            "climber_cache_release": (I32, [VP, VP]),
            "climber_cache_append": (I32, [VP, C.c_uint64, I32, C.c_uint64, C.c_uint64, P, I64, VP, P, P, P]),
            "climber_nccl_unique_id": (I32, [P]),
            "climber_encode_user_bcast": (I32, [VP, P, I64, I32, I32, VP, P]),
            "climber_cache_stats": (I32, [VP, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


EXPORTED_SYMBOLS = ("climber_arena_bytes", "climber_create", "climber_destroy", "climber_encode_user",
                    "climber_encode_users", "climber_score_items", "climber_score_items_batched",
                    "climber_rank_host", "climber_kv_release", "climber_kv_broadcast", "climber_stream_status",
                    "climber_last_error", "climber_debug_extract", "climber_debug_mask", "climber_debug_kv",
                    "climber_debug_attn_probe",
                    "climber_launch_count", "climber_debug_gemm", "climber_profile", "climber_profile_read",
                    "climber_kv_slab_bytes", "climber_kv_export", "climber_kv_import",
                    "climber_encode_users_blocks", "climber_score_blocks", "climber_fuse_scores", "climber_forward",
                    "climber_cache_acquire", "climber_cache_release", "climber_cache_stats",
                    "climber_cache_append", "climber_nccl_unique_id", "climber_encode_user_bcast")

KERNEL_CLASSES = ("extract", "embed", "rmsnorm", "gemm_qkv", "gemm_o", "gemm_ffn_up", "gemm_ffn_down", "gemm_se",
                  "attn_hist", "attn_sumi", "attn_fusion", "head", "other")


def _check(st: int):
    if st != 0:
        raise ClimberError(st, lib().climber_last_error().decode())


def debug_gemm(A, B, D, use_tc: bool = True, stream=None, epi: int = 0):
    """The library's bf16 GEMM C = A @ B^T (A [M][K], B [N][K] bf16; CUDA tensors):
    epi 0: D(fp32) += C; epi 1: D(bf16) = C; epi 2: D(bf16) = SiLU(C)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    M, K = A.shape
    N = B.shape[0]
    if epi == 3:  # grouped interleaved test mode: A [M][2K], B [2N][K]
        K //= 2
        N //= 2
    _check(lib().climber_debug_gemm(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(D.data_ptr()),
                                    M, N, K, int(use_tc), int(epi), C.c_void_p(s.cuda_stream)))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for Climber(..., rank, world, nccl_uid)."""
    buf = (C.c_char * 128)()
    _check(lib().climber_nccl_unique_id(buf))
    return bytes(buf)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class ModelConfig:
    """Mirror of climber_config's model fields (PAPER.md notation)."""
    d: int
    h: int
    L: int
    N_b: int
    n_k: int
    V: int
    R: int
    M_max: int
    n_actions: int = 6
    ffn_mult: int = 4
    se_reduction: int = 4
    hist_causal: int = 1
    dtype: str = "bf16"
    rms_eps: float = 1e-6
    rel_bias: int = 0

    @classmethod
    def from_any(cls, cfg, M_max: Optional[int] = None) -> "ModelConfig":
        return cls(d=cfg.d, h=cfg.h, L=cfg.L, N_b=cfg.N_b, n_k=cfg.n_k, V=cfg.V, R=cfg.R,
                   M_max=M_max or cfg.M, n_actions=getattr(cfg, "n_actions", 6), ffn_mult=cfg.ffn_mult,
                   se_reduction=cfg.se_reduction, hist_causal=cfg.hist_causal, dtype=cfg.dtype,
                   rms_eps=cfg.rms_eps, rel_bias=getattr(cfg, "rel_bias", 0))


class Climber:
    """One libclimber context on the current CUDA device.

    weights: object with the attributes of climber_weights (fp32 numpy arrays,
    [in][out] layout); strategies: list of (action_mask, scenario_mask).
    """

    def __init__(self, cfg: ModelConfig, weights, strategies: Sequence[tuple], *, max_users: int = 64,
                 max_wave_users: int = 64, max_wave_pairs: Optional[int] = None, kv_users: Optional[int] = None,
                 device=None, rank: int = 0, world: int = 1, nccl_uid: Optional[bytes] = None):
        import torch
        self.torch = torch
        self.cfg = cfg
        ppb = (cfg.n_k + 63) // 64
        per_user = cfg.N_b * cfg.L * ppb
        kv_users = kv_users or max_users
        c = _Config()
        c.abi_version = ABI_VERSION
        c.d, c.n_heads, c.n_layers, c.n_blocks, c.n_k = cfg.d, cfg.h, cfg.L, cfg.N_b, cfg.n_k
        c.ffn_mult, c.se_reduction, c.vocab, c.n_actions, c.n_scenarios = (
            cfg.ffn_mult, cfg.se_reduction, cfg.V, cfg.n_actions, cfg.R)
        c.max_candidates, c.hist_causal = cfg.M_max, cfg.hist_causal
        c.dtype = BF16 if cfg.dtype == "bf16" else FP32
        c.page_tokens = 64
        c.rms_eps = cfg.rms_eps
        c.max_batch_users = max_users
        c.max_wave_users = max_wave_users
        c.max_wave_pairs = max_wave_pairs or max(cfg.M_max, min(max_users * cfg.M_max, 65536))
        c.kv_pages = kv_users * per_user
        c.rel_bias = int(cfg.rel_bias)
        self._c = c
        L = lib()
        nbytes = L.climber_arena_bytes(C.byref(c))
        if nbytes == 0:
            raise ClimberError(2, "invalid config")
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.arena = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        self._keep = []
        w = _Weights()
        for n in WEIGHT_NAMES:
            a = np.ascontiguousarray(getattr(weights, n), dtype=np.float32)
            self._keep.append(a)
            setattr(w, n, a.ctypes.data)
        w.b_head = float(np.asarray(weights.b_head).reshape(-1)[0])
        for n in ("b_pos", "b_time"):
            t = getattr(weights, n, None)
            if cfg.rel_bias and t is not None:
                a = np.ascontiguousarray(t, dtype=np.float32)
                self._keep.append(a)
                setattr(w, n, a.ctypes.data)
        st = (_Strategy * cfg.N_b)(*[_Strategy(int(a), int(s)) for a, s in strategies])
        h = C.c_void_p()
        uid = C.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
        _check(L.climber_create(C.byref(c), st, C.byref(w), C.c_void_p(self.arena.data_ptr()), nbytes, int(rank),
                                int(world), uid, C.byref(h)))
        self._keep = []
        self.h = h

    # -- plumbing ---------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            _check(lib().climber_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self, stream=None):
        s = stream if stream is not None else self.torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def profile(self, enable: bool):
        _check(lib().climber_profile(self.h, int(bool(enable))))

    def profile_read(self) -> dict:
        """{class: {launches, ms, flops, bytes}} accumulated since the last read."""
        out = np.zeros(4 * len(KERNEL_CLASSES), np.float64)
        _check(lib().climber_profile_read(self.h, _ptr(out)))
        return {n: dict(zip(("launches", "ms", "flops", "bytes"), out[4 * i:4 * i + 4].tolist()))
                for i, n in enumerate(KERNEL_CLASSES)}

    @property
    def launch_count(self) -> int:
        return int(lib().climber_launch_count(self.h))

    # -- the hot path -------------------------------------------------------
    def encode_users(self, ev_offsets: np.ndarray, item, action, scenario, ts, r: np.ndarray, stream=None) -> List[int]:
        """item/action/scenario/ts: CUDA tensors (int32/uint8/uint8/int64);
        ev_offsets int64[B+1], r int32[B]: numpy (host)."""
        ev_offsets = np.ascontiguousarray(ev_offsets, np.int64)
        r = np.ascontiguousarray(r, np.int32)
        B = len(r)
        ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        out = (C.c_void_p * B)()
        _check(lib().climber_encode_users(self.h, B, _ptr(ev_offsets), C.byref(ev), _ptr(r), self._stream(stream), out))
        return [out[i] for i in range(B)]

    def score_batched(self, handles: Sequence[int], cand_offsets: np.ndarray, items, scores=None, stream=None):
        """items: CUDA int32 tensor; returns (or fills) a CUDA float32 tensor."""
        cand_offsets = np.ascontiguousarray(cand_offsets, np.int64)
        B = len(handles)
        if scores is None:
            scores = self.torch.empty(int(cand_offsets[-1]), dtype=self.torch.float32, device=items.device)
        hs = (C.c_void_p * B)(*handles)
        _check(lib().climber_score_items_batched(self.h, B, hs, _ptr(cand_offsets), C.c_void_p(items.data_ptr()),
                                                 C.c_void_p(scores.data_ptr()), self._stream(stream)))
        return scores

    def encode_user(self, item, action, scenario, ts, r: int, stream=None) -> int:
        ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        out = C.c_void_p()
        _check(lib().climber_encode_user(self.h, C.byref(ev), int(item.numel()), int(r), self._stream(stream),
                                         C.byref(out)))
        return out.value

    def score_items(self, handle: int, items, scores=None, stream=None):
        if scores is None:
            scores = self.torch.empty(items.numel(), dtype=self.torch.float32, device=items.device)
        _check(lib().climber_score_items(self.h, C.c_void_p(handle), C.c_void_p(items.data_ptr()), int(items.numel()),
                                         C.c_void_p(scores.data_ptr()), self._stream(stream)))
        return scores

    def forward(self, ev_offsets, item, action, scenario, ts, r, cand_offsets, items, scores=None, stream=None):
        """SUMI forward of compressed training records (no cache kept): CUDA
        tensors for events / items, numpy offsets and scenarios."""
        ev_offsets = np.ascontiguousarray(ev_offsets, np.int64)
        cand_offsets = np.ascontiguousarray(cand_offsets, np.int64)
        r = np.ascontiguousarray(r, np.int32)
        if scores is None:
            scores = self.torch.empty(int(cand_offsets[-1]), dtype=self.torch.float32, device=items.device)
        ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        _check(lib().climber_forward(self.h, len(r), _ptr(ev_offsets), C.byref(ev), _ptr(r), _ptr(cand_offsets),
                                     C.c_void_p(items.data_ptr()), C.c_void_p(scores.data_ptr()),
                                     self._stream(stream)))
        return scores

    # -- serving cache store (NEXT-4) ---------------------------------------
    CACHE_RESULT = {0: "hit", 1: "encoded", 2: "uncached", 3: "appended"}

    def cache_acquire(self, user_key: int, r: int, digest: int, item, action, scenario, ts, stream=None):
        """(handle, "hit" | "encoded" | "uncached"); events are CUDA tensors."""
        ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        out, res = C.c_void_p(), C.c_int32()
        _check(lib().climber_cache_acquire(self.h, C.c_uint64(user_key), int(r), C.c_uint64(digest), C.byref(ev),
                                           int(item.numel()), self._stream(stream), C.byref(out), C.byref(res)))
        return out.value, self.CACHE_RESULT[res.value]

    def cache_append(self, user_key: int, r: int, digest_prefix: int, digest: int, item, action, scenario, ts,
                     stream=None):
        """(handle, result, blocks recomputed) after the user's log grew by appending."""
        ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        out, res, nb = C.c_void_p(), C.c_int32(), C.c_int32()
        _check(lib().climber_cache_append(self.h, C.c_uint64(user_key), int(r), C.c_uint64(digest_prefix),
                                          C.c_uint64(digest), C.byref(ev), int(item.numel()), self._stream(stream),
                                          C.byref(out), C.byref(res), C.byref(nb)))
        return out.value, self.CACHE_RESULT[res.value], nb.value

    def cache_release(self, handle):
        _check(lib().climber_cache_release(self.h, C.c_void_p(handle)))

    def cache_stats(self) -> dict:
        st = np.zeros(5, np.int64)
        _check(lib().climber_cache_stats(self.h, _ptr(st)))
        return dict(zip(("entries", "pinned", "hits", "misses", "evictions"), map(int, st)))

    # -- block-parallel serving (NEXT-2): blocks [k0, k1) per process --------
    def encode_users_blocks(self, ev_offsets, item, action, scenario, ts, r, k0: int, k1: int,
                            stream=None) -> List[int]:
        ev_offsets = np.ascontiguousarray(ev_offsets, np.int64)
        r = np.ascontiguousarray(r, np.int32)
        B = len(r)
        ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        out = (C.c_void_p * B)()
        _check(lib().climber_encode_users_blocks(self.h, B, _ptr(ev_offsets), C.byref(ev), _ptr(r), int(k0), int(k1),
                                                 self._stream(stream), out))
        return [out[i] for i in range(B)]

    def score_blocks(self, handles, cand_offsets, items, k0: int, k1: int, E=None, stream=None):
        """Block outputs E [P][k1 - k0][d] (fp32 CUDA tensor) of blocks [k0, k1)."""
        cand_offsets = np.ascontiguousarray(cand_offsets, np.int64)
        B = len(handles)
        P = int(cand_offsets[-1] - cand_offsets[0])
        if E is None:
            E = self.torch.empty((P, k1 - k0, self.cfg.d), dtype=self.torch.float32, device=items.device)
        hs = (C.c_void_p * B)(*handles)
        _check(lib().climber_score_blocks(self.h, B, hs, _ptr(cand_offsets), C.c_void_p(items.data_ptr()), int(k0),
                                          int(k1), C.c_void_p(E.data_ptr()), self._stream(stream)))
        return E

    def fuse_scores(self, cand_offsets, r, E, n_slices: int = 1, scores=None, stream=None):
        """BGF + head from E [n_slices][P][N_b / n_slices][d] (fp32 CUDA tensor)."""
        cand_offsets = np.ascontiguousarray(cand_offsets, np.int64)
        r = np.ascontiguousarray(r, np.int32)
        P = int(cand_offsets[-1] - cand_offsets[0])
        if scores is None:
            scores = self.torch.empty(P, dtype=self.torch.float32, device=E.device)
        _check(lib().climber_fuse_scores(self.h, len(r), _ptr(cand_offsets), _ptr(r), int(n_slices),
                                         C.c_void_p(E.data_ptr()), C.c_void_p(scores.data_ptr()),
                                         self._stream(stream)))
        return scores

    def release(self, handles):
        for hd in (handles if isinstance(handles, (list, tuple)) else [handles]):
            _check(lib().climber_kv_release(self.h, C.c_void_p(hd)))

    def rank_host(self, ev_offsets, item, action, scenario, ts, r, cand_offsets, items, stream=None) -> np.ndarray:
        """End-to-end with HOST numpy buffers (H2D, encode, score, D2H inside the call)."""
        arrs = [np.ascontiguousarray(a, dt) for a, dt in (
            (ev_offsets, np.int64), (item, np.int32), (action, np.uint8), (scenario, np.uint8), (ts, np.int64),
            (r, np.int32), (cand_offsets, np.int64), (items, np.int32))]
        scores = np.empty(int(arrs[6][-1]), np.float32)
        B = len(arrs[5])
        _check(lib().climber_rank_host(self.h, B, *[_ptr(a) for a in arrs], _ptr(scores), self._stream(stream)))
        return scores

    # -- multi-GPU candidate sharding: K/V slab exchange ---------------------
    @property
    def slab_bytes(self) -> int:
        return int(lib().climber_kv_slab_bytes(self.h))

    def kv_export(self, handle, slab=None, stream=None):
        """Gather the handle's K/V pages into a CUDA uint8 tensor (the slab)."""
        if slab is None:
            slab = self.torch.empty(self.slab_bytes, dtype=self.torch.uint8, device=self.arena.device)
        _check(lib().climber_kv_export(self.h, C.c_void_p(handle), C.c_void_p(slab.data_ptr()), self._stream(stream)))
        return slab

    def kv_broadcast(self, handle: Optional[int], root: int = 0, stream=None) -> int:
        """Collective: replicate root's handle to every rank (NCCL inside the library)."""
        kv = C.c_void_p(handle or 0)
        _check(lib().climber_kv_broadcast(self.h, C.byref(kv), int(root), self._stream(stream)))
        return kv.value

    def encode_user_bcast(self, events, r: int, root: int = 0, stream=None) -> int:
        """Collective: encode on root and replicate the K/V layer by layer while
        it is encoded (climber_encode_user_bcast).  events = (item, action,
        scenario, ts) CUDA tensors on root, None elsewhere."""
        ev, n_s = None, 0
        if events is not None:
            item, action, scenario, ts = events
            n_s = int(item.numel())
            ev = _Events(item.data_ptr(), action.data_ptr(), scenario.data_ptr(), ts.data_ptr())
        out = C.c_void_p()
        _check(lib().climber_encode_user_bcast(self.h, C.byref(ev) if ev is not None else None, n_s, int(r),
                                               int(root), self._stream(stream), C.byref(out)))
        return out.value

    def kv_import(self, slab, r: int, stream=None) -> int:
        out = C.c_void_p()
        _check(lib().climber_kv_import(self.h, C.c_void_p(slab.data_ptr()), int(r), self._stream(stream), C.byref(out)))
        return out.value

    def stream_status(self, stream=None):
        _check(lib().climber_stream_status(self.h, self._stream(stream)))

    # -- debug exports (synchronous) ---------------------------------------
    def debug_extract(self, handle):
        idx = np.empty((self.cfg.N_b, self.cfg.n_k), np.int32)
        vlen = np.empty(self.cfg.N_b, np.int32)
        _check(lib().climber_debug_extract(self.h, C.c_void_p(handle), _ptr(idx), _ptr(vlen)))
        return idx, vlen

    def debug_mask(self, handle, M: int):
        T = self.cfg.n_k + M
        m = np.empty((self.cfg.N_b, T, T), np.uint8)
        _check(lib().climber_debug_mask(self.h, C.c_void_p(handle), int(M), _ptr(m)))
        return m

    def debug_attn_probe(self, handle, mode: int, layer: int, block: int, M: int, key_off: int):
        """climber_debug_attn_probe: float [rows][d] (rows = n_k for mode 0, M for mode 1)."""
        rows = self.cfg.n_k if mode == 0 else M
        out = np.zeros((rows, self.cfg.d), np.float32)
        _check(lib().climber_debug_attn_probe(self.h, C.c_void_p(handle), int(mode), int(layer), int(block),
                                              int(M), int(key_off), _ptr(out)))
        return out

    def debug_kv(self, handle, layer: int, block: int, v: int):
        dt = np.uint16 if self.cfg.dtype == "bf16" else np.float32
        K = np.zeros((v, self.cfg.d), dt)
        V = np.zeros((v, self.cfg.d), dt)
        _check(lib().climber_debug_kv(self.h, C.c_void_p(handle), int(layer), int(block), _ptr(K), _ptr(V)))
        if dt == np.uint16:
            K = (K.astype(np.uint32) << 16).view(np.float32)
            V = (V.astype(np.uint32) << 16).view(np.float32)
        return K, V
