"""Thin ctypes binding of libbingo.so (include/bingo.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of ``csrc/``.  PyTorch provides device memory (the graph's pools come from the
caching allocator through the ABI's allocator hooks), streams and tensors.
There is no CPU fallback: without the compiled library or a CUDA device every
entry point raises.
"""
from __future__ import annotations

import contextlib
import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BINGO_LIB_OVERRIDE") or os.path.join(HERE, "libbingo.so")   # override: A/B experiments only

OK, E_INVAL, E_NOMEM, E_CUDA, E_OVERFLOW, E_STATE = 0, 1, 2, 3, 4, 5
EMPTY, ONE, DENSE, SPARSE, REGULAR = 0, 1, 2, 3, 4
DEEPWALK, NODE2VEC, PPR = 0, 1, 2
BUILD_BS_MODE = 1
BUILD_NEIGHBOR_INDEX = 2
BUILD_FLOAT_BIAS = 4
UPD_HOST_BATCH = 1
WALK_HOST_OUTPUT = 1
WALK_WALKER_MAJOR = 2
COUNTS_HOST = 1
NO_CAP = 0xFFFFFFFF

# every symbol include/bingo.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ("bingo_build", "bingo_destroy", "bingo_apply_updates", "bingo_apply_updates_f64", "bingo_walk",
               "bingo_visit_counts",
               "bingo_export", "bingo_digests", "bingo_get_info", "bingo_status_str", "bingo_walk_profile",
               "bingo_walk_trace", "bingo_walk_replay", "bingo_stream_update", "bingo_walk_partition",
               "bingo_export_vertices", "bingo_import_vertices")


class BingoError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib().bingo_status_str(status).decode() if _LIB is not None else str(status)
        super().__init__(f"{where}: {msg} (status {status})")


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class BuildDesc(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_uint32), ("num_arcs", ctypes.c_uint64),
                ("row_offsets", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("bias", ctypes.c_void_p),
                ("alpha_pct", ctypes.c_uint32), ("beta_pct", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("arc_slack", ctypes.c_double), ("member_slack", ctypes.c_double),
                ("pool_reserve", ctypes.c_double), ("alloc", ALLOC_FN), ("free", FREE_FN),
                ("alloc_ctx", ctypes.c_void_p), ("bias_f64", ctypes.c_void_p)]


class UpdateStats(ctypes.Structure):
    _fields_ = [("inserted", ctypes.c_uint64), ("deleted", ctypes.c_uint64),
                ("missing_deletes", ctypes.c_uint64), ("touched_vertices", ctypes.c_uint64),
                ("kind_transitions", ctypes.c_uint64 * 25), ("epoch", ctypes.c_uint64)]


class WalkDesc(ctypes.Structure):
    _fields_ = [("app", ctypes.c_uint32), ("length", ctypes.c_uint32), ("p", ctypes.c_double),
                ("q", ctypes.c_double), ("stop_num", ctypes.c_uint32), ("stop_den", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("first_walker_id", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


class Info(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_uint32), ("epoch", ctypes.c_uint32), ("num_arcs", ctypes.c_uint64),
                ("arc_pool_used", ctypes.c_uint64), ("arc_pool_cap", ctypes.c_uint64),
                ("bucket_pool_used", ctypes.c_uint64), ("bucket_pool_cap", ctypes.c_uint64),
                ("member_pool_used", ctypes.c_uint64), ("member_pool_cap", ctypes.c_uint64),
                ("device_bytes", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("l2_persist_bytes", ctypes.c_uint64), ("hot_degree", ctypes.c_uint64),
                ("update_reruns", ctypes.c_uint64)]


_LIB = None


def _lib():
    """Load libbingo.so (built by ``python -m paper_2504_10233_b200._build``).  Raises if missing."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libbingo.so not built at {LIB_PATH}: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        L.bingo_build.argtypes = [ctypes.POINTER(BuildDesc), P, ctypes.POINTER(P)]
        L.bingo_build.restype = ctypes.c_int
        L.bingo_destroy.argtypes = [P]
        L.bingo_destroy.restype = None
        L.bingo_apply_updates.argtypes = [P, P, u64, u32, ctypes.POINTER(UpdateStats), P]
        L.bingo_apply_updates.restype = ctypes.c_int
        L.bingo_apply_updates_f64.argtypes = [P, P, P, u64, u32, ctypes.POINTER(UpdateStats), P]
        L.bingo_apply_updates_f64.restype = ctypes.c_int
        L.bingo_walk.argtypes = [P, ctypes.POINTER(WalkDesc), P, u32, P, P, P]
        L.bingo_walk.restype = ctypes.c_int
        L.bingo_visit_counts.argtypes = [P, P, ctypes.c_int, u32, P]
        L.bingo_visit_counts.restype = ctypes.c_int
        L.bingo_export.argtypes = [P, P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), P]
        L.bingo_export.restype = ctypes.c_int
        L.bingo_digests.argtypes = [P, P, P]
        L.bingo_digests.restype = ctypes.c_int
        L.bingo_get_info.argtypes = [P, ctypes.POINTER(Info), P]
        L.bingo_get_info.restype = ctypes.c_int
        L.bingo_walk_profile.argtypes = [P, ctypes.POINTER(WalkDesc), P, u32, P, P, P, P]
        L.bingo_walk_profile.restype = ctypes.c_int
        L.bingo_walk_partition.argtypes = [P, ctypes.POINTER(WalkDesc), u32, P, u32, u32, P, u32, P, u64, P, P, P,
                                           P, P]
        L.bingo_walk_partition.restype = ctypes.c_int
        L.bingo_stream_update.argtypes = [P, P, ctypes.POINTER(UpdateStats), P]
        L.bingo_stream_update.restype = ctypes.c_int
        L.bingo_walk_trace.argtypes = [P, ctypes.POINTER(WalkDesc), P, u32, P, P, u64, P, P]
        L.bingo_walk_trace.restype = ctypes.c_int
        L.bingo_walk_replay.argtypes = [P, P, P, u32, u32, P, P]
        L.bingo_walk_replay.restype = ctypes.c_int
        L.bingo_export_vertices.argtypes = [P, P, u32, P, u64, P, ctypes.POINTER(u64), P]
        L.bingo_export_vertices.restype = ctypes.c_int
        L.bingo_import_vertices.argtypes = [P, P, P, u32, P]
        L.bingo_import_vertices.restype = ctypes.c_int
        L.bingo_status_str.argtypes = [ctypes.c_int]
        L.bingo_status_str.restype = ctypes.c_char_p
        _LIB = L
    return _LIB


def _check(st: int, where: str):
    if st != OK:
        raise BingoError(st, where)


_TORCH = None


def _torch():
    global _TORCH
    if _TORCH is None:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2504_10233_b200 needs a CUDA device (B200); there is no CPU fallback")
        _TORCH = torch
    return _TORCH


def _stream_ptr(stream) -> Optional[int]:
    torch = _torch()
    if stream is None:   # the current stream's raw handle without building a Stream object
        return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())
    return stream.cuda_stream


def _order_on(stream, device, *tensors):
    """A call on a caller-given stream: that stream first waits for the current stream (where
    the temporaries / outputs below were allocated and filled), and every device tensor is
    marked as used by it, so the caching allocator does not hand its memory out again
    before the launch completes."""
    if stream is None:
        return
    torch = _torch()
    cur = torch.cuda.current_stream(device)
    if stream != cur:
        stream.wait_stream(cur)
    for t in tensors:
        if t is not None and isinstance(t, torch.Tensor) and t.is_cuda:
            t.record_stream(stream)


def _dev_u32(x, torch, device):
    if isinstance(x, torch.Tensor):
        t = x.to(device=device)
        if t.dtype not in (torch.int32, torch.uint32):
            t = t.to(torch.int64).to(torch.int32)
        return t.contiguous()
    a = np.ascontiguousarray(x, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).to(device)


def _dev_u64(x, torch, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int64).contiguous()
    a = np.ascontiguousarray(x, dtype=np.uint64)
    return torch.from_numpy(a.view(np.int64)).to(device)


class _TorchAllocator:
    """Routes the library's device allocations to PyTorch's caching allocator."""

    def __init__(self, device):
        import torch
        self.device = torch.device(device)
        self.live = {}
        release = torch.cuda.caching_allocator_delete     # bound now: callbacks may run at interpreter exit

        def _alloc(nbytes, ctx):
            try:
                with torch.cuda.device(self.device):
                    p = torch.cuda.caching_allocator_alloc(int(nbytes), self.device.index)
                self.live[p] = nbytes
                return p
            except Exception:
                return None

        def _free(ptr, ctx):
            if ptr:
                self.live.pop(ptr, None)
                try:
                    release(ptr)
                except Exception:
                    pass

        self.alloc = ALLOC_FN(_alloc)
        self.free = FREE_FN(_free)


class Graph:
    """A Bingo sampling structure resident in HBM (one replica per GPU)."""

    def __init__(self, row_offsets, dst, bias, alpha: int = 40, beta: int = 10, bs_mode: bool = False,
                 arc_slack: float = 0.25, member_slack: float = 0.25, pool_reserve: float = 0.1,
                 neighbor_index: bool = False, float_bias: bool = False, device=None, stream=None,
                 torch_alloc: bool = True, radix_log2: int = 0):
        torch = _torch()
        L = _lib()
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        ro = _dev_u64(row_offsets, torch, self.device)
        ds = _dev_u32(dst, torch, self.device)
        self.float_mode = bool(float_bias)
        if float_bias:
            bf = (bias.to(self.device, torch.float64) if isinstance(bias, torch.Tensor)
                  else torch.from_numpy(np.ascontiguousarray(bias, dtype=np.float64)).to(self.device))
            bs = torch.zeros(1, dtype=torch.int32, device=self.device)
        else:
            bf = None
            bs = _dev_u32(bias, torch, self.device)
        self.V = ro.numel() - 1
        self._alloc = _TorchAllocator(self.device) if torch_alloc else None
        d = BuildDesc(num_vertices=self.V, num_arcs=ds.numel(), row_offsets=ro.data_ptr(), dst=ds.data_ptr(),
                      bias=bs.data_ptr(), alpha_pct=alpha, beta_pct=beta,
                      flags=(BUILD_BS_MODE if bs_mode else 0) | (BUILD_NEIGHBOR_INDEX if neighbor_index else 0)
                      | (BUILD_FLOAT_BIAS if float_bias else 0) | ((int(radix_log2) & 0xF) << 8),
                      arc_slack=arc_slack, member_slack=member_slack, pool_reserve=pool_reserve,
                      alloc=self._alloc.alloc if self._alloc else ALLOC_FN(), free=self._alloc.free if self._alloc else FREE_FN(),
                      alloc_ctx=None, bias_f64=bf.data_ptr() if bf is not None else None)
        h = ctypes.c_void_p()
        _order_on(stream, self.device, ro, ds, bs, bf)
        with torch.cuda.device(self.device):
            _check(L.bingo_build(ctypes.byref(d), _stream_ptr(stream), ctypes.byref(h)), "bingo_build")
        self._h = h

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib().bingo_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------- updates
    def apply_updates(self, batch, stream=None, bias_f64=None) -> dict:
        """Batched insert/delete; ``batch`` is an (n, 4) u32 {op, src, dst, bias} array:
        a CUDA tensor (device path) or a numpy array (host path, H2D inside the call).
        Float-bias graphs take the inserted biases from ``bias_f64`` ([n] float64, same
        memory space as ``batch``; bingo_apply_updates_f64, R-16)."""
        torch = _torch()
        st = UpdateStats()
        flags = 0
        wf = None
        if isinstance(batch, torch.Tensor) and batch.is_cuda:
            b = batch.contiguous()
            n = b.numel() // 4
            ptr = b.data_ptr() if n else None
            if bias_f64 is not None:
                wf = torch.as_tensor(bias_f64, dtype=torch.float64, device=b.device).contiguous()
        else:
            arr = np.ascontiguousarray(batch, dtype=np.uint32).reshape(-1, 4)
            n = arr.shape[0]
            ptr = arr.ctypes.data if n else None
            flags = UPD_HOST_BATCH
            b = arr
            if bias_f64 is not None:
                wf = np.ascontiguousarray(bias_f64, dtype=np.float64)
        if isinstance(b, torch.Tensor):
            _order_on(stream, self.device, b, wf)
        same = self.device.index is None or torch.cuda.current_device() == self.device.index
        with contextlib.nullcontext() if same else torch.cuda.device(self.device):
            if wf is None:
                rc = _lib().bingo_apply_updates(self._h, ptr, n, flags, ctypes.byref(st), _stream_ptr(stream))
            else:
                wptr = (wf.data_ptr() if isinstance(wf, torch.Tensor) else wf.ctypes.data) if n else None
                rc = _lib().bingo_apply_updates_f64(self._h, ptr, wptr, n, flags, ctypes.byref(st),
                                                    _stream_ptr(stream))
            _check(rc, "bingo_apply_updates")
        return {"inserted": st.inserted, "deleted": st.deleted, "missing_deletes": st.missing_deletes,
                "touched_vertices": st.touched_vertices,
                "kind_transitions": np.array(st.kind_transitions, dtype=np.uint64).reshape(5, 5),
                "epoch": st.epoch}

    def stream_update(self, record, stream=None, stats: bool = True):
        """bingo_stream_update: one {op, src, dst, bias} record through the persistent
        streaming queue (no launch per record); returns the statistics like apply_updates."""
        torch = _torch()
        rec = np.ascontiguousarray(record, dtype=np.uint32).reshape(4)
        st = UpdateStats()
        with contextlib.nullcontext() if torch.cuda.current_device() == self.device.index else \
                torch.cuda.device(self.device):
            _check(_lib().bingo_stream_update(self._h, rec.ctypes.data, ctypes.byref(st) if stats else None,
                                              _stream_ptr(stream)), "bingo_stream_update")
        if not stats:
            return None
        return {"inserted": st.inserted, "deleted": st.deleted, "missing_deletes": st.missing_deletes,
                "touched_vertices": st.touched_vertices,
                "kind_transitions": np.array(st.kind_transitions, dtype=np.uint64).reshape(5, 5),
                "epoch": st.epoch}

    def try_apply_updates(self, batch, stream=None, bias_f64=None) -> int:
        try:
            self.apply_updates(batch, stream, bias_f64=bias_f64)
            return OK
        except BingoError as e:
            return e.status

    # ---------------------------------------------------------- walks
    def walk(self, app: int = DEEPWALK, length: int = 80, seed: int = 0, first_walker: int = 0, starts=None,
             num_walkers: Optional[int] = None, p: float = 1.0, q: float = 1.0, stop=(1, 80), paths=True,
             lengths=True, walker_major: bool = False, stream=None):
        """Launch ``num_walkers`` walkers (default: one per vertex).  Returns device tensors
        {"paths": int32 [(length+1), W] (or [W, length+1] walker-major) or None,
         "lengths": int32 [W] or None}."""
        torch = _torch()
        W = num_walkers if num_walkers is not None else (len(starts) if starts is not None else self.V)
        st = _dev_u32(starts, torch, self.device) if starts is not None else None
        pa = None
        if paths is True:
            shape = (W, length + 1) if walker_major else (length + 1, W)
            pa = torch.empty(shape, dtype=torch.int32, device=self.device)
        elif paths is not None and paths is not False:
            pa = paths
        ln = None
        if lengths is True:
            ln = torch.empty(W, dtype=torch.int32, device=self.device)
        elif lengths is not None and lengths is not False:
            ln = lengths
        d = WalkDesc(app=app, length=length, p=p, q=q, stop_num=stop[0], stop_den=stop[1], seed=seed,
                     first_walker_id=first_walker, flags=WALK_WALKER_MAJOR if walker_major else 0)
        _order_on(stream, self.device, st, pa, ln)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_walk(self._h, ctypes.byref(d), st.data_ptr() if st is not None else None, W,
                                     pa.data_ptr() if pa is not None else None,
                                     ln.data_ptr() if ln is not None else None, _stream_ptr(stream)),
                   "bingo_walk")
        return {"paths": pa, "lengths": ln}

    def walk_host(self, app: int = DEEPWALK, length: int = 80, seed: int = 0, first_walker: int = 0,
                  starts: Optional[np.ndarray] = None, num_walkers: Optional[int] = None, p: float = 1.0,
                  q: float = 1.0, stop=(1, 80), paths: Optional[np.ndarray] = None,
                  lengths: Optional[np.ndarray] = None, walker_major: bool = False, stream=None):
        """Same walk with HOST (ideally pinned) buffers: the library stages H2D/D2H itself."""
        torch = _torch()
        W = num_walkers if num_walkers is not None else (len(starts) if starts is not None else self.V)
        d = WalkDesc(app=app, length=length, p=p, q=q, stop_num=stop[0], stop_den=stop[1], seed=seed,
                     first_walker_id=first_walker,
                     flags=WALK_HOST_OUTPUT | (WALK_WALKER_MAJOR if walker_major else 0))

        def ptr(a):
            if a is None:
                return None
            return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data
        with torch.cuda.device(self.device):
            _check(_lib().bingo_walk(self._h, ctypes.byref(d), ptr(starts), W, ptr(paths), ptr(lengths),
                                     _stream_ptr(stream)), "bingo_walk")
        return {"paths": paths, "lengths": lengths}

    def walk_profile(self, app: int = DEEPWALK, length: int = 80, seed: int = 0, first_walker: int = 0, starts=None,
                     num_walkers: Optional[int] = None, p: float = 1.0, q: float = 1.0, stop=(1, 80), paths=True,
                     stream=None) -> dict:
        """bingo_walk that also counts the records each step loaded (see bingo.h)."""
        torch = _torch()
        W = num_walkers if num_walkers is not None else (len(starts) if starts is not None else self.V)
        st = _dev_u32(starts, torch, self.device) if starts is not None else None
        pa = torch.empty((length + 1, W), dtype=torch.int32, device=self.device) if paths else None
        ln = torch.empty(W, dtype=torch.int32, device=self.device)
        d = WalkDesc(app=app, length=length, p=p, q=q, stop_num=stop[0], stop_den=stop[1], seed=seed,
                     first_walker_id=first_walker, flags=0)
        c = np.zeros(8, dtype=np.uint64)
        _order_on(stream, self.device, st, pa, ln)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_walk_profile(self._h, ctypes.byref(d), st.data_ptr() if st is not None else None, W,
                                             pa.data_ptr() if pa is not None else None, ln.data_ptr(), c.ctypes.data,
                                             _stream_ptr(stream)), "bingo_walk_profile")
        names = ("steps", "hdr", "bkt", "mem", "arc", "probe", "visit", "walkers")
        out = {k: int(v) for k, v in zip(names, c)}
        out["paths"] = pa
        out["lengths"] = ln
        return out

    def walk_partition(self, bounds, me: int, inbox, outbox, out_count, app: int = DEEPWALK, length: int = 80,
                       seed: int = 0, first_walker: int = 0, num_walkers: Optional[int] = None, stop=(1, 80),
                       paths=None, lengths=None, stream=None) -> int:
        """bingo_walk_partition: one round of the 1-D partitioned walk on this partition graph.
        bounds: int32 CUDA tensor [parts + 1]; inbox: int32 CUDA [n, 4]; outbox: int32 CUDA
        [parts, cap, 4] (cap >= n); out_count: int32 CUDA [parts], zeroed.  Returns the number of
        walkers that finished here."""
        torch = _torch()
        W = num_walkers if num_walkers is not None else self.V
        n = inbox.shape[0]
        parts = bounds.numel() - 1
        d = WalkDesc(app=app, length=length, p=1.0, q=1.0, stop_num=stop[0], stop_den=stop[1], seed=seed,
                     first_walker_id=first_walker, flags=0)
        fin = ctypes.c_uint64(0)
        _order_on(stream, self.device, bounds, inbox, outbox, out_count, paths, lengths)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_walk_partition(
                self._h, ctypes.byref(d), W, bounds.data_ptr(), parts, me, inbox.data_ptr() if n else None, n,
                outbox.data_ptr(), outbox.shape[1], out_count.data_ptr(),
                paths.data_ptr() if paths is not None else None, lengths.data_ptr() if lengths is not None else None,
                ctypes.byref(fin), _stream_ptr(stream)), "bingo_walk_partition")
        return int(fin.value)

    def walk_trace(self, rec_off, trace, app: int = DEEPWALK, length: int = 80, seed: int = 0,
                   first_walker: int = 0, num_walkers: Optional[int] = None, stop=(1, 80), stream=None) -> dict:
        """bingo_walk_trace: the same walks, with every step's loads recorded into `trace`
        (CUDA tensor of 16 B x n_records, e.g. int32 [n_records, 4]) at rec_off[i] + t (int64
        CUDA tensor [num_walkers + 1], exclusive prefix sum of the lengths).  Returns the
        load counters."""
        torch = _torch()
        W = num_walkers if num_walkers is not None else self.V
        n = trace.numel() * trace.element_size() // 16
        d = WalkDesc(app=app, length=length, p=1.0, q=1.0, stop_num=stop[0], stop_den=stop[1], seed=seed,
                     first_walker_id=first_walker, flags=0)
        c = np.zeros(8, dtype=np.uint64)
        _order_on(stream, self.device, rec_off, trace)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_walk_trace(self._h, ctypes.byref(d), None, W, rec_off.data_ptr(), trace.data_ptr(), n,
                                           c.ctypes.data, _stream_ptr(stream)), "bingo_walk_trace")
        names = ("steps", "hdr", "bkt", "mem", "arc", "probe", "visit", "walkers")
        return {k: int(v) for k, v in zip(names, c)}

    def walk_replay(self, trace, rec_off, ahead: int = 4, blocks_per_sm: int = 8, stream=None) -> dict:
        """bingo_walk_replay: the traced loads, walker by walker, `ahead` steps in flight per
        thread and no dependency between steps.  Returns the loads issued per record type."""
        torch = _torch()
        c = np.zeros(4, dtype=np.uint64)
        _order_on(stream, self.device, trace, rec_off)
        with torch.cuda.device(self.device):
            flags = {1: 0, 2: 1, 4: 2, 8: 3}[ahead] | (blocks_per_sm << 8)
            _check(_lib().bingo_walk_replay(self._h, trace.data_ptr(), rec_off.data_ptr(), rec_off.numel() - 1,
                                            flags, c.ctypes.data, _stream_ptr(stream)), "bingo_walk_replay")
        return {"hdr": int(c[0]), "bkt": int(c[1]), "mem": int(c[2]), "arc": int(c[3])}

    def export_vertices(self, ids, stream=None):
        """bingo_export_vertices: the state records of the vertices `ids` (CUDA int tensor, the
        caller's ids).  Returns (buf int32 CUDA tensor of u32 words, offsets int64 [n + 1])."""
        torch = _torch()
        ids = ids.to(device=self.device, dtype=torch.int32).contiguous()
        n = ids.numel()
        off = torch.empty(n + 1, dtype=torch.int64, device=self.device)
        words = ctypes.c_uint64(0)
        _order_on(stream, self.device, ids, off)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_export_vertices(self._h, ids.data_ptr() if n else None, n, None, 0, off.data_ptr(),
                                                ctypes.byref(words), _stream_ptr(stream)), "bingo_export_vertices")
            buf = torch.empty(max(int(words.value), 1), dtype=torch.int32, device=self.device)
            if n:
                _check(_lib().bingo_export_vertices(self._h, ids.data_ptr(), n, buf.data_ptr(), buf.numel(),
                                                    off.data_ptr(), ctypes.byref(words), _stream_ptr(stream)),
                       "bingo_export_vertices")
        return buf[:int(words.value)], off

    def import_vertices(self, buf, offsets, stream=None):
        """bingo_import_vertices: install records exported by a replica of this graph."""
        torch = _torch()
        n = offsets.numel() - 1
        if n <= 0:
            return
        buf = buf.to(device=self.device, dtype=torch.int32).contiguous()
        offsets = offsets.to(device=self.device, dtype=torch.int64).contiguous()
        _order_on(stream, self.device, buf, offsets)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_import_vertices(self._h, buf.data_ptr(), offsets.data_ptr(), n, _stream_ptr(stream)),
                   "bingo_import_vertices")

    def visit_counts(self, reset: bool = False, stream=None):
        torch = _torch()
        out = torch.empty(self.V, dtype=torch.int64, device=self.device)
        _order_on(stream, self.device, out)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_visit_counts(self._h, out.data_ptr(), int(reset), 0, _stream_ptr(stream)),
                   "bingo_visit_counts")
        return out

    def visit_counts_host(self, reset: bool = False, stream=None) -> np.ndarray:
        """The same counts copied to a host array by the library (BINGO_COUNTS_HOST)."""
        torch = _torch()
        out = np.empty(self.V, dtype=np.uint64)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_visit_counts(self._h, out.ctypes.data if self.V else None, int(reset), COUNTS_HOST,
                                             _stream_ptr(stream)), "bingo_visit_counts")
        return out

    def reset_visit_counts(self, stream=None):
        torch = _torch()
        with torch.cuda.device(self.device):
            _check(_lib().bingo_visit_counts(self._h, None, 1, 0, _stream_ptr(stream)), "bingo_visit_counts")

    # ---------------------------------------------------------- inspection
    def export(self, stream=None) -> bytes:
        torch = _torch()
        n = ctypes.c_size_t(0)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_export(self._h, None, 0, ctypes.byref(n), _stream_ptr(stream)), "bingo_export")
            buf = np.zeros(max(n.value, 1), dtype=np.uint8)
            _check(_lib().bingo_export(self._h, buf.ctypes.data, n.value, ctypes.byref(n), _stream_ptr(stream)),
                   "bingo_export")
        return buf[:n.value].tobytes()

    def digests(self, stream=None):
        torch = _torch()
        out = torch.empty(self.V, dtype=torch.int64, device=self.device)
        _order_on(stream, self.device, out)
        with torch.cuda.device(self.device):
            _check(_lib().bingo_digests(self._h, out.data_ptr(), _stream_ptr(stream)), "bingo_digests")
        return out

    def info(self, stream=None) -> dict:
        torch = _torch()
        i = Info()
        with torch.cuda.device(self.device):
            _check(_lib().bingo_get_info(self._h, ctypes.byref(i), _stream_ptr(stream)), "bingo_get_info")
        return {f: getattr(i, f) for f, _ in Info._fields_}
