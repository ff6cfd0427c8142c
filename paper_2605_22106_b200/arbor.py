"""Thin ctypes binding of libarbor.so (include/arbor.h) — argument marshalling only.

Every step of the ArborKV path runs in the library's CUDA kernels.  PyTorch is used
only to own device memory (the K/V/pos pools, the accumulated-attention array) and to
provide streams.  There is no CPU fallback: if the shared library is missing or no CUDA
device is present, constructing a context raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ARBOR_LIB: A/B experiments only (profiles/, tools/) — the default is the in-tree build
LIB_PATH = os.environ.get("ARBOR_LIB") or os.path.join(_HERE, "libarbor.so")

ARBOR_OK = 0
STATUS = {0: "OK", 2: "INVALID_ARG", 3: "INFEASIBLE_BUDGET", 4: "INVARIANT", 5: "IO",
          6: "OUT_OF_PAGES", 7: "STATE", 8: "CUDA", 9: "NCCL"}
ALLOC_MODES = {"waterfill": 0, "static": 1, "static_drain": 2, "stream": 3}
SELECT_MODES = {"heavy": 0, "tail": 1, "sinks_tail": 2}
FLAG_PROFILE = 1
FLAG_EXTERNAL_REDUCE = 2
FLAG_COLLECTIVE = 4
NUM_STAGES = 13
STAGES = ["geometry", "score_accum", "node_mass", "msve", "allocate", "evict_plan",
          "select_compact", "rehydrate", "attn", "attn_merge", "allreduce", "stash",
          "compact_move"]


class ArborError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"arbor status {status} ({STATUS.get(status, '?')}): {message}")
        self.status = status
        self.message = message


class ArborParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("gamma", C.c_double), ("lambda_d", C.c_double),
                ("lambda_delta", C.c_double), ("eta", C.c_double), ("r_min", C.c_double),
                ("k_min", C.c_int32), ("l_tail", C.c_int32), ("n_sinks", C.c_int32),
                ("alloc_mode", C.c_int32), ("theta", C.c_double * 4),
                ("select_mode", C.c_int32), ("no_rehydrate", C.c_int32),
                ("k_protect", C.c_int32), ("slice_layers", C.c_int32),
                ("slice_kv_heads", C.c_int32), ("select_shared", C.c_int32)]


class ArborConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_kv_heads", C.c_int32), ("num_q_heads", C.c_int32),
                ("head_dim", C.c_int32), ("layer_begin", C.c_int32), ("layer_count", C.c_int32),
                ("kv_head_begin", C.c_int32), ("kv_head_count", C.c_int32), ("kv_dtype", C.c_int32),
                ("page_size", C.c_int32), ("num_pages", C.c_int32), ("max_nodes", C.c_int32),
                ("max_node_tokens", C.c_int32), ("max_active", C.c_int32), ("max_tokens", C.c_int64),
                ("k_pool", C.c_void_p), ("v_pool", C.c_void_p), ("pos_pool", C.c_void_p),
                ("score", C.c_void_p), ("host_stash", C.c_void_p), ("host_stash_bytes", C.c_size_t),
                ("rank", C.c_int32), ("world_size", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("main_stream", C.c_void_p), ("side_stream", C.c_void_p), ("flags", C.c_uint32)]


class ArborTree(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("parent", C.c_void_p), ("span_start", C.c_void_p),
                ("span_len", C.c_void_p), ("is_open", C.c_void_p), ("search_value", C.c_void_p),
                ("uncertainty", C.c_void_p), ("num_active", C.c_int32), ("active", C.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libarbor.so and declare its signatures (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ArborError(8, f"{path} not built (run python -m paper_2605_22106_b200.build)")
    lib = C.CDLL(path)
    P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "arbor_init": ([C.POINTER(ArborConfig), C.POINTER(ArborParams), C.POINTER(C.c_void_p)], I32),
        "arbor_destroy": ([P], None),
        "arbor_last_error": ([P], C.c_char_p),
        "arbor_status_string": ([I32], C.c_char_p),
        "arbor_nccl_unique_id": ([P], I32),
        "arbor_open_node": ([P, I32, I64], I32),
        "arbor_append_kv": ([P, I32, P, P, I32], I32),
        "arbor_close_node": ([P, I32], I32),
        "arbor_score": ([P, C.POINTER(ArborTree), P, P, P], I32),
        "arbor_allocate": ([P, C.POINTER(ArborTree), P, I64, P, C.POINTER(C.c_int64)], I32),
        "arbor_evict": ([P, C.POINTER(ArborTree), P, C.POINTER(C.c_int64)], I32),
        "arbor_rehydrate": ([P, C.POINTER(ArborTree), P, I32], I32),
        "arbor_policy_event": ([P, C.POINTER(ArborTree), I32, I32, I64, P, C.POINTER(C.c_int64)], I32),
        "arbor_retained_tokens": ([P, C.POINTER(C.c_int64)], I32),
        "arbor_policy_waterline": ([P, C.POINTER(ArborTree), I64, I64, P], I32),
        "arbor_pressure_events": ([P, C.POINTER(C.c_int64)], I32),
        "arbor_boundary_uncertainty": ([P, P, I32, I32, I32, P], I32),
        "arbor_tree_decode_attn": ([P, C.POINTER(ArborTree), I32, I32, P, P, P], I32),
        "arbor_decode_step": ([P, C.POINTER(ArborTree), P, P, P, P], I32),
        "arbor_sync": ([P], I32),
        "arbor_read_node": ([P, I32, P, P, P, P], I32),
        "arbor_read_node_offset": ([P, I32, C.POINTER(C.c_int32)], I32),
        "arbor_read_free_list": ([P, P, P], I32),
        "arbor_read_scores": ([P, I32, P, P, P, P, P], I32),
        "arbor_read_counters": ([P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], I32),
        "arbor_mass_buffer": ([P, C.POINTER(C.c_void_p), C.POINTER(C.c_int32)], I32),
        "arbor_rehydrate_in_flight": ([P, C.POINTER(C.c_int32)], I32),
        "arbor_score_finish": ([P, P, P], I32),
        "arbor_save_state": ([P, I32], I32),
        "arbor_load_state": ([P, I32], I32),
        "arbor_launch_count": ([P], I64),
        "arbor_attn_tensor_cores": ([P], I32),
        "arbor_invalidate_masses": ([P], I32),
        "arbor_stage_times": ([P, P], I32),
        "arbor_reset_stage_times": ([P], I32),
        "arbor_set_profiling": ([P, I32], I32),
        "arbor_capture_begin": ([P], I32),
        "arbor_capture_end": ([P, C.POINTER(C.c_void_p)], I32),
        "arbor_graph_launch": ([P, P], I32),
        "arbor_graph_destroy": ([P], I32),
        "arbor_validate_tree": ([C.POINTER(ArborTree), I32, C.c_char_p, C.c_size_t], I32),
        "arbor_min_feasible_budget": ([C.POINTER(ArborParams), C.POINTER(ArborTree),
                                       C.POINTER(C.c_int64)], I32),
        "arbor_version": ([], C.c_char_p),
        "arbor_fit_theta": ([P, P, I32, I32, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)], I32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def make_params(alpha=1.0, gamma=2.0, lambda_d=0.0, lambda_delta=0.5, eta=0.8, r_min=0.05,
                k_min=4, l_tail=8, n_sinks=4, theta=(-1.0, 2.0, 1.0, 4.0),
                alloc_mode="waterfill", select_mode="heavy", no_rehydrate=False,
                k_protect=0, slice_layers=0, slice_kv_heads=0, select_shared=False) -> ArborParams:
    """Parameter bundle Π (Alg. 1 caption P:498); defaults are DESIGN.md's documented choices."""
    mode = ALLOC_MODES[alloc_mode] if isinstance(alloc_mode, str) else int(alloc_mode)
    sel = SELECT_MODES[select_mode] if isinstance(select_mode, str) else int(select_mode)
    p = ArborParams(alpha, gamma, lambda_d, lambda_delta, eta, r_min, int(k_min), int(l_tail),
                    int(n_sinks), mode)
    p.select_mode = sel
    p.no_rehydrate = 1 if no_rehydrate else 0
    p.k_protect = int(k_protect)
    p.slice_layers = int(slice_layers)
    p.slice_kv_heads = int(slice_kv_heads)
    p.select_shared = 1 if select_shared else 0
    for i, t in enumerate(theta):
        p.theta[i] = float(t)
    return p


def params_from_dict(d: dict) -> ArborParams:
    keys = ("alpha", "gamma", "lambda_d", "lambda_delta", "eta", "r_min", "k_min", "l_tail",
            "n_sinks", "theta", "alloc_mode", "select_mode", "no_rehydrate")
    return make_params(**{k: d[k] for k in keys if k in d})


@dataclass
class TreeArgs:
    """Host arrays of one ``arbor_tree`` snapshot, kept alive while the struct is used."""
    parent: np.ndarray
    span_start: np.ndarray
    span_len: np.ndarray
    is_open: np.ndarray
    v: np.ndarray
    u: np.ndarray
    active: np.ndarray
    struct: ArborTree = field(default=None)

    @classmethod
    def from_tree(cls, t) -> "TreeArgs":
        ta = cls(np.ascontiguousarray(t.parent, np.int32), np.ascontiguousarray(t.span_start, np.int64),
                 np.ascontiguousarray(t.span_len, np.int32), np.ascontiguousarray(t.is_open, np.uint8),
                 np.ascontiguousarray(t.v, np.float32), np.ascontiguousarray(t.u, np.float32),
                 np.ascontiguousarray(np.asarray(t.active, np.int32)))
        ta.struct = ArborTree(int(ta.parent.shape[0]), ta.parent.ctypes.data, ta.span_start.ctypes.data,
                              ta.span_len.ctypes.data, ta.is_open.ctypes.data, ta.v.ctypes.data,
                              ta.u.ctypes.data, int(ta.active.shape[0]), ta.active.ctypes.data)
        return ta


def _tree(t) -> TreeArgs:
    return t if isinstance(t, TreeArgs) else TreeArgs.from_tree(t)


def validate_tree(tree, n_sinks: int = 0):
    """Host-only tree validation (no device needed). Returns (status, message)."""
    lib = load_library()
    ta = _tree(tree)
    buf = C.create_string_buffer(512)
    st = lib.arbor_validate_tree(C.byref(ta.struct), int(n_sinks), buf, 512)
    return st, buf.value.decode()


def min_feasible_budget(params: ArborParams, tree) -> int:
    lib = load_library()
    ta = _tree(tree)
    out = C.c_int64(0)
    st = lib.arbor_min_feasible_budget(C.byref(params), C.byref(ta.struct), C.byref(out))
    if st != ARBOR_OK:
        raise ArborError(st, "arbor_min_feasible_budget")
    return int(out.value)


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    st = lib.arbor_nccl_unique_id(buf)
    if st != ARBOR_OK:
        raise ArborError(st, "arbor_nccl_unique_id")
    return buf.raw


class ArborKV:
    """One rank's ArborKV context: the caller-owned pools (torch tensors) + libarbor state.

    Shapes (this rank's shard of ``layer_count`` layers × ``kv_head_count`` KV heads):
      k_pool, v_pool [layer_count][num_pages][kv_head_count][page_size][head_dim]
      pos_pool       [layer_count][num_pages][kv_head_count][page_size] int16
      score (A)      [layer_count][kv_head_count][max_tokens] float32
    """

    def __init__(self, *, num_layers, num_kv_heads, num_q_heads, head_dim, dtype="bf16",
                 page_size=16, num_pages, max_nodes, max_node_tokens, max_active=16, max_tokens,
                 params: ArborParams, layer_begin=0, layer_count=None, kv_head_begin=0,
                 kv_head_count=None, rank=0, world_size=1, nccl_id: bytes = None,
                 profile=False, device=None, external_reduce=False, collective=False):
        import torch
        if not torch.cuda.is_available():
            raise ArborError(8, "no CUDA device: the ArborKV path has no CPU fallback")
        self.lib = load_library()
        self.torch = torch
        self.device = (torch.device(device) if device is not None
                       else torch.device("cuda", torch.cuda.current_device()))
        torch.cuda.set_device(self.device)
        self.dtype = dtype
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.tdtype = tdt
        L = layer_count if layer_count is not None else num_layers
        H = kv_head_count if kv_head_count is not None else num_kv_heads
        self.L, self.H, self.D, self.P, self.NP = L, H, head_dim, page_size, num_pages
        self.max_nodes = max_nodes
        self.G = num_q_heads // num_kv_heads
        self.Hq = H * self.G
        self.max_tokens = max_tokens
        dev = self.device
        self.k_pool = torch.zeros((L, num_pages, H, page_size, head_dim), dtype=tdt, device=dev)
        self.v_pool = torch.zeros_like(self.k_pool)
        self.pos_pool = torch.zeros((L, num_pages, H, page_size), dtype=torch.int16, device=dev)
        self.score = torch.zeros((L, H, max_tokens), dtype=torch.float32, device=dev)
        self.stream = torch.cuda.current_stream(dev)
        self.side = torch.cuda.Stream(dev)
        self._nccl = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        cfg = ArborConfig(num_layers, num_kv_heads, num_q_heads, head_dim, layer_begin, L,
                          kv_head_begin, H, 1 if dtype == "bf16" else 0, page_size, num_pages,
                          max_nodes, max_node_tokens, max_active, max_tokens,
                          self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.pos_pool.data_ptr(),
                          self.score.data_ptr(), None, 0, rank, world_size,
                          C.cast(self._nccl, C.c_void_p) if self._nccl is not None else None,
                          self.stream.cuda_stream, self.side.cuda_stream,
                          (FLAG_PROFILE if profile else 0) |
                          (FLAG_EXTERNAL_REDUCE if external_reduce else 0) |
                          (FLAG_COLLECTIVE if collective else 0))
        self.params = params
        self._ctx = C.c_void_p()
        st = self.lib.arbor_init(C.byref(cfg), C.byref(params), C.byref(self._ctx))
        if st != ARBOR_OK:
            raise ArborError(st, "arbor_init failed")
        self._tree_cache = None

    # ---------------------------------------------------------------- helpers
    def _check(self, st, what):
        if st != ARBOR_OK:
            msg = self.lib.arbor_last_error(self._ctx)
            raise ArborError(st, f"{what}: {msg.decode() if msg else ''}")

    @staticmethod
    def _ptr(t):
        return None if t is None else t.data_ptr()

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self.lib.arbor_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- plumbing
    def arbor_open_node(self, node: int, span_start: int):
        self._check(self.lib.arbor_open_node(self._ctx, int(node), int(span_start)), "arbor_open_node")

    def arbor_append_kv(self, node: int, k, v):
        """k, v: device [layer_count][kv_head_count][ntok][head_dim] contiguous."""
        assert k.is_contiguous() and v.is_contiguous() and k.dtype == self.tdtype
        self._check(self.lib.arbor_append_kv(self._ctx, int(node), k.data_ptr(), v.data_ptr(),
                                             int(k.shape[2])), "arbor_append_kv")

    def arbor_close_node(self, node: int):
        self._check(self.lib.arbor_close_node(self._ctx, int(node)), "arbor_close_node")

    # ---------------------------------------------------------------- hot path
    def arbor_score(self, tree, q, lse=None, s_out=None):
        ta = _tree(tree)
        self._check(self.lib.arbor_score(self._ctx, C.byref(ta.struct), q.data_ptr(), self._ptr(lse),
                                         self._ptr(s_out)), "arbor_score")
        return s_out

    def arbor_allocate(self, tree, s, budget: int, k_out):
        ta = _tree(tree)
        mf = C.c_int64(-1)
        st = self.lib.arbor_allocate(self._ctx, C.byref(ta.struct), self._ptr(s), int(budget),
                                     k_out.data_ptr(), C.byref(mf))
        if st == 3:
            e = ArborError(st, f"infeasible budget {budget}, min feasible {mf.value}")
            e.min_feasible = int(mf.value)
            raise e
        self._check(st, "arbor_allocate")
        return k_out

    def arbor_policy_event(self, tree, kind, node, budget: int, k_out):
        """f1: one policy update event of Alg. 2 (kind: 'boundary' | 'transition' | 'pressure'
        or the arbor_pue value); k_out receives the applied targets."""
        kinds = {"boundary": 0, "transition": 1, "pressure": 2}
        kd = kinds[kind] if isinstance(kind, str) else int(kind)
        ta = _tree(tree)
        mf = C.c_int64(-1)
        st = self.lib.arbor_policy_event(self._ctx, C.byref(ta.struct), kd, int(node), int(budget),
                                         k_out.data_ptr(), C.byref(mf))
        if st == 3:
            e = ArborError(st, f"infeasible budget {budget}, min feasible {mf.value}")
            e.min_feasible = int(mf.value)
            raise e
        self._check(st, "arbor_policy_event")
        return k_out

    def arbor_policy_waterline(self, tree, budget: int, delta: int, k_out):
        """f1: the waterline check + gated Pressure on the device (no host sync)."""
        ta = _tree(tree)
        self._check(self.lib.arbor_policy_waterline(self._ctx, C.byref(ta.struct), int(budget),
                                                    int(delta), k_out.data_ptr()),
                    "arbor_policy_waterline")

    def arbor_pressure_events(self) -> int:
        v = C.c_int64(0)
        self._check(self.lib.arbor_pressure_events(self._ctx, C.byref(v)), "arbor_pressure_events")
        return int(v.value)

    def arbor_boundary_uncertainty(self, logits, u_out):
        """f3: Eq. 1 uncertainty of each row of logits [batch][vocab] (f32 or bf16) → u_out."""
        import torch
        dt = {torch.float32: 0, torch.bfloat16: 1}[logits.dtype]
        b, v = logits.shape
        self._check(self.lib.arbor_boundary_uncertainty(self._ctx, logits.data_ptr(), dt, int(b),
                                                        int(v), u_out.data_ptr()),
                    "arbor_boundary_uncertainty")
        return u_out

    def arbor_retained_tokens(self) -> int:
        t = C.c_int64(0)
        self._check(self.lib.arbor_retained_tokens(self._ctx, C.byref(t)), "arbor_retained_tokens")
        return int(t.value)

    def arbor_evict(self, tree, k_target, want_count=False):
        ta = _tree(tree)
        ev = C.c_int64(0)
        self._check(self.lib.arbor_evict(self._ctx, C.byref(ta.struct), k_target.data_ptr(),
                                         C.byref(ev) if want_count else None), "arbor_evict")
        return int(ev.value) if want_count else None

    def arbor_rehydrate(self, tree, nodes):
        ta = _tree(tree)
        arr = np.ascontiguousarray(np.asarray(list(nodes), np.int32))
        self._check(self.lib.arbor_rehydrate(self._ctx, C.byref(ta.struct), arr.ctypes.data,
                                             int(arr.shape[0])), "arbor_rehydrate")

    def arbor_tree_decode_attn(self, tree, q, out, lse=None, layer_begin=0, layer_count=None):
        ta = _tree(tree)
        lc = self.L if layer_count is None else layer_count
        self._check(self.lib.arbor_tree_decode_attn(self._ctx, C.byref(ta.struct), int(layer_begin),
                                                    int(lc), q.data_ptr(), out.data_ptr(),
                                                    self._ptr(lse)), "arbor_tree_decode_attn")
        return out

    def arbor_decode_step(self, tree, q, out, lse=None, s_out=None):
        """f2: a9 + a2 + a3 fused (attention kernel, then merge + score in one launch)."""
        ta = _tree(tree)
        self._check(self.lib.arbor_decode_step(self._ctx, C.byref(ta.struct), q.data_ptr(),
                                               out.data_ptr(), self._ptr(lse), self._ptr(s_out)),
                    "arbor_decode_step")
        return out

    # ---------------------------------------------------------------- inspection
    def arbor_sync(self):
        self._check(self.lib.arbor_sync(self._ctx), "arbor_sync")

    def arbor_read_node(self, node: int):
        kc, n, npg = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        self._check(self.lib.arbor_read_node(self._ctx, int(node), C.byref(kc), C.byref(n), None,
                                             C.byref(npg)), "arbor_read_node")
        pages = np.zeros(max(1, npg.value), np.int32)
        cnt = C.c_int32(pages.shape[0])
        self._check(self.lib.arbor_read_node(self._ctx, int(node), None, None, pages.ctypes.data,
                                             C.byref(cnt)), "arbor_read_node")
        return int(kc.value), int(n.value), pages[:cnt.value].tolist()

    def arbor_read_node_offset(self, node: int) -> int:
        """Slot of the node's live page list holding its valid slot 0 (Q23*)."""
        v = C.c_int32(0)
        self._check(self.lib.arbor_read_node_offset(self._ctx, int(node), C.byref(v)),
                    "arbor_read_node_offset")
        return int(v.value)

    def arbor_read_free_list(self):
        cnt = C.c_int32(0)
        self._check(self.lib.arbor_read_free_list(self._ctx, None, C.byref(cnt)), "free list")
        buf = np.zeros(max(1, cnt.value), np.int32)
        cnt2 = C.c_int32(buf.shape[0])
        self._check(self.lib.arbor_read_free_list(self._ctx, buf.ctypes.data, C.byref(cnt2)), "free list")
        return buf[:cnt2.value].tolist()

    def arbor_read_scores(self, num_nodes: int):
        mass = np.zeros(num_nodes, np.int64)
        mclose = np.zeros(num_nodes, np.int64)
        nq = np.zeros(num_nodes, np.int64)
        a = np.zeros(num_nodes, np.float32)
        s = np.zeros(num_nodes, np.float32)
        self._check(self.lib.arbor_read_scores(self._ctx, int(num_nodes), mass.ctypes.data,
                                               mclose.ctypes.data, nq.ctypes.data, a.ctypes.data,
                                               s.ctypes.data), "arbor_read_scores")
        return dict(mass=mass, mclose=mclose, nq=nq, a=a, s=s)

    def arbor_rehydrate_in_flight(self) -> bool:
        """True while the last rehydration copy (side stream) is still running (no sync)."""
        v = C.c_int32(0)
        self._check(self.lib.arbor_rehydrate_in_flight(self._ctx, C.byref(v)), "arbor_rehydrate_in_flight")
        return bool(v.value)

    def arbor_mass_buffer(self):
        """a10's buffer: (device pointer, count) of this rank's int64 partial masses
        [Mass | Mclose] of the last score call (include/arbor.h)."""
        ptr, cnt = C.c_void_p(), C.c_int32(0)
        self._check(self.lib.arbor_mass_buffer(self._ctx, C.byref(ptr), C.byref(cnt)), "arbor_mass_buffer")
        return int(ptr.value or 0), int(cnt.value)

    def arbor_score_finish(self, reduced=None, s_out=None):
        """ARBOR_FLAG_EXTERNAL_REDUCE: MSVE on the reduced masses (a DEVICE int64 tensor
        [2N], or None when arbor_mass_buffer was reduced in place)."""
        self._check(self.lib.arbor_score_finish(self._ctx, self._ptr(reduced), self._ptr(s_out)),
                    "arbor_score_finish")

    def arbor_read_counters(self):
        r, p = C.c_int64(0), C.c_int64(0)
        self._check(self.lib.arbor_read_counters(self._ctx, C.byref(r), C.byref(p)), "counters")
        return int(r.value), int(p.value)

    def arbor_save_state(self, slot=0):
        self._check(self.lib.arbor_save_state(self._ctx, int(slot)), "arbor_save_state")

    def arbor_load_state(self, slot=0):
        self._check(self.lib.arbor_load_state(self._ctx, int(slot)), "arbor_load_state")

    def arbor_invalidate_masses(self):
        """Call after writing the score array (A) directly."""
        self._check(self.lib.arbor_invalidate_masses(self._ctx), "arbor_invalidate_masses")

    def arbor_launch_count(self) -> int:
        return int(self.lib.arbor_launch_count(self._ctx))

    def arbor_attn_tensor_cores(self) -> bool:
        return int(self.lib.arbor_attn_tensor_cores(self._ctx)) == 1

    def arbor_reset_stage_times(self):
        self._check(self.lib.arbor_reset_stage_times(self._ctx), "arbor_reset_stage_times")

    def arbor_set_profiling(self, on: bool):
        self._check(self.lib.arbor_set_profiling(self._ctx, 1 if on else 0), "arbor_set_profiling")

    def arbor_capture_begin(self):
        self._check(self.lib.arbor_capture_begin(self._ctx), "arbor_capture_begin")

    def arbor_capture_end(self):
        """Ends the capture; returns the graph handle (an int)."""
        g = C.c_void_p()
        self._check(self.lib.arbor_capture_end(self._ctx, C.byref(g)), "arbor_capture_end")
        return g.value

    def arbor_graph_launch(self, graph):
        self._check(self.lib.arbor_graph_launch(self._ctx, C.c_void_p(graph)), "arbor_graph_launch")

    def arbor_graph_destroy(self, graph):
        self._check(self.lib.arbor_graph_destroy(C.c_void_p(graph)), "arbor_graph_destroy")

    def arbor_stage_times(self) -> dict:
        ms = (C.c_float * NUM_STAGES)()
        self._check(self.lib.arbor_stage_times(self._ctx, ms), "arbor_stage_times")
        return {STAGES[i]: float(ms[i]) for i in range(NUM_STAGES)}

    # ---------------------------------------------------------------- views for tests
    def slot_rows(self, node: int):
        """(k_cur, n, pages) of a node (sync)."""
        return self.arbor_read_node(node)


def fit_theta(phi, target, theta0=(0.0, 0.0, 0.0, 0.0), epochs=200, lr=4.0):
    """f3: MSVE θ calibration on the device (include/arbor.h arbor_fit_theta).
    phi: DEVICE f32 tensor [n][3] (v, u, a); target: DEVICE f32 [n].  Returns (θ, (L0, L1))."""
    lib = load_library()
    th = (C.c_double * 4)(*[float(x) for x in theta0])
    ls = (C.c_double * 2)()
    st = lib.arbor_fit_theta(phi.data_ptr(), target.data_ptr(), int(target.numel()), int(epochs),
                             float(lr), th, ls)
    if st != ARBOR_OK:
        raise ArborError(st, "arbor_fit_theta failed")
    return [th[i] for i in range(4)], (ls[0], ls[1])
