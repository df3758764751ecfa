"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/bingo_oracle.c``, the plain CPU oracle of the
Bingo hot path (arXiv 2504.10233).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with ``paper_2504_10233_b200`` and never imports it.

Function-by-function citations are in the C source; the canonical readings
(R-1 ... R-12) are listed in DESIGN.md section 3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bingo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

EMPTY, ONE, DENSE, SPARSE, REGULAR = 0, 1, 2, 3, 4
KIND_NAMES = {EMPTY: "EMPTY", ONE: "ONE", DENSE: "DENSE", SPARSE: "SPARSE", REGULAR: "REGULAR"}
FLAG_BS_MODE = 1
NONE = 0xFFFFFFFF
APP_DEEPWALK, APP_NODE2VEC, APP_PPR = 0, 1, 2


def build_lib(force: bool = False) -> str:
    """Compile the oracle (plain C, gcc -O2, OpenMP across walkers only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build_lib()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            u32, u64 = ctypes.c_uint32, ctypes.c_uint64
            L.ora_philox4x32_10.argtypes = [P, P, P]
            L.ora_classify.argtypes = [u32, u32, u32, u32, u32]
            L.ora_classify.restype = u32
            L.ora_alias_build.argtypes = [u32, P, P, P]
            L.ora_build.argtypes = [u32, P, P, P, u32, u32, u32, ctypes.POINTER(P)]
            L.ora_build.restype = ctypes.c_int
            L.ora_build_lazy.argtypes = [u32, P, P, P, u32, u32, u32, ctypes.POINTER(P)]
            L.ora_build_lazy.restype = ctypes.c_int
            L.ora_dump_vertex.argtypes = [P, u32, P, ctypes.c_size_t]
            L.ora_dump_vertex.restype = ctypes.c_size_t
            L.ora_build_float.argtypes = [u32, P, P, P, u32, u32, u32, ctypes.POINTER(P)]
            L.ora_build_float.restype = ctypes.c_int
            L.ora_free.argtypes = [P]
            L.ora_epoch.argtypes = [P]
            L.ora_epoch.restype = u32
            L.ora_degree.argtypes = [P, u32]
            L.ora_degree.restype = u32
            L.ora_two_phase_u32.argtypes = [P, u32, P, u32]
            L.ora_two_phase_u32.restype = u32
            L.ora_apply_updates.argtypes = [P, P, u64, P]
            L.ora_apply_updates.restype = ctypes.c_int
            L.ora_apply_updates_f.argtypes = [P, P, P, u64, P]
            L.ora_apply_updates_f.restype = ctypes.c_int
            L.ora_sample.argtypes = [P, u32, u64, u32, u32, u32]
            L.ora_sample.restype = u32
            L.ora_walk.argtypes = [P, u32, u32, u64, u32, P, u32, P, P, P, P, P, u64, u32,
                                   ctypes.c_int, P]
            L.ora_dump.argtypes = [P, P, ctypes.c_size_t]
            L.ora_dump.restype = ctypes.c_size_t
            L.ora_digests.argtypes = [P, P]
            L.ora_touch.argtypes = [P, P, u64, ctypes.c_int]
            L.ora_build_radix.argtypes = [u32, P, P, P, u32, ctypes.POINTER(P)]
            L.ora_build_radix.restype = ctypes.c_int
            L.ora_radix_free.argtypes = [P]
            L.ora_radix_sample.argtypes = [P, u32, u64, u32, u32]
            L.ora_radix_sample.restype = u32
            L.ora_radix_walk.argtypes = [P, u32, u32, u64, u32, P, u32, P, P, P, u64, u32, ctypes.c_int]
            L.ora_radix_dump.argtypes = [P, P, ctypes.c_size_t]
            L.ora_radix_dump.restype = ctypes.c_size_t
            L.ora_radix_apply_updates.argtypes = [P, P, u64, P]
            L.ora_radix_apply_updates.restype = ctypes.c_int
            L.ora_radix_adj.argtypes = [P, u32, P]
            L.ora_radix_adj.restype = u32
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().ora_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def classify(c: int, d: int, alpha: int = 40, beta: int = 10, flags: int = 0) -> int:
    return int(lib().ora_classify(c, d, alpha, beta, flags))


def alias_build(W) -> tuple[np.ndarray, np.ndarray]:
    W = np.ascontiguousarray(W, dtype=np.uint64)
    n = len(W)
    thr = np.zeros(max(n, 1), dtype=np.uint64)
    al = np.zeros(max(n, 1), dtype=np.uint32)
    lib().ora_alias_build(n, _p(W), _p(thr), _p(al))
    return thr[:n], al[:n]


def two_phase(arr, deleted) -> list:
    a = np.ascontiguousarray(arr, dtype=np.uint32).copy()
    d = np.ascontiguousarray(sorted(deleted), dtype=np.uint32)
    n = lib().ora_two_phase_u32(_p(a), len(a), _p(d) if len(d) else None, len(d))
    return a[:n].tolist()


def n2v_thresholds(p: float, q: float):
    """Eq.1 factors f = 1/p, 1, 1/q by distance 0/1/2, accept ratio f/f_max
    mapped to a 64-bit threshold floor(ratio * 2^64) (R-1); ratio 1 -> always."""
    f = [1.0 / p, 1.0, 1.0 / q]
    fmax = max(f)
    thr = np.zeros(3, dtype=np.uint64)
    always = np.zeros(3, dtype=np.uint32)
    for i, fi in enumerate(f):
        r = fi / fmax
        if r >= 1.0:
            always[i] = 1
        else:
            thr[i] = int(Fraction(r) * (1 << 64))   # floor(ratio * 2^64), exact
            if thr[i] == 0:   # never accepted: a walker could reject forever (bingo.h: EINVAL)
                raise ValueError(f"node2vec ratio {r} < 2^-64 can never be accepted")
    return thr, always


def stop_threshold(num: int, den: int):
    """PPR termination probability num/den -> floor(num * 2^64 / den) (R-1)."""
    if num >= den:
        return 0, 1
    return (num << 64) // den, 0


class OracleGraph:
    """One oracle graph instance (host memory)."""

    def __init__(self, row_offsets, dst, bias, alpha=40, beta=10, flags=0, float_bias=False, lazy=False):
        L = lib()
        self.V = len(row_offsets) - 1
        self.float_mode = bool(float_bias)
        ro = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        ds = np.ascontiguousarray(dst, dtype=np.uint32)
        h = ctypes.c_void_p()
        if lazy:
            # vertices are built from these arrays on first access: keep them alive
            bs = np.ascontiguousarray(bias, dtype=np.uint32)
            self._keep = (ro, ds, bs)
            rc = L.ora_build_lazy(self.V, _p(ro), _p(ds), _p(bs), alpha, beta, flags, ctypes.byref(h))
        elif float_bias:
            bf = np.ascontiguousarray(bias, dtype=np.float64)
            rc = L.ora_build_float(self.V, _p(ro), _p(ds), _p(bf), alpha, beta, flags, ctypes.byref(h))
        else:
            bs = np.ascontiguousarray(bias, dtype=np.uint32)
            rc = L.ora_build(self.V, _p(ro), _p(ds), _p(bs), alpha, beta, flags, ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"ora_build failed with status {rc}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:   # module globals are gone at interpreter exit
            lib().ora_free(h)
            self._h = None

    @property
    def epoch(self) -> int:
        return int(lib().ora_epoch(self._h))

    def apply_updates(self, recs, bias_f64=None) -> dict:
        """Apply one batch; float-mode graphs take the inserted biases from bias_f64 (R-16)."""
        r = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 4)
        st = np.zeros(30, dtype=np.uint64)
        rc = self._apply(r, bias_f64, st)
        if rc != 0:
            raise ValueError(f"ora_apply_updates failed with status {rc}")
        return {"inserted": int(st[0]), "deleted": int(st[1]), "missing_deletes": int(st[2]),
                "touched_vertices": int(st[3]), "kind_transitions": st[4:29].reshape(5, 5).copy(),
                "epoch": int(st[29])}

    def _apply(self, r, bias_f64, st):
        if bias_f64 is None:
            return int(lib().ora_apply_updates(self._h, _p(r) if len(r) else None, len(r), _p(st)))
        wf = np.ascontiguousarray(bias_f64, dtype=np.float64)
        return int(lib().ora_apply_updates_f(self._h, _p(r) if len(r) else None, _p(wf) if len(wf) else None,
                                             len(r), _p(st)))

    def try_apply_updates(self, recs, bias_f64=None) -> int:
        r = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 4)
        return self._apply(r, bias_f64, None)

    def sample(self, u, seed, w, t, outer=0) -> int:
        return int(lib().ora_sample(self._h, u, seed, w, t, outer))

    def touch(self, ids, threads=0):
        """Materialise these vertices now (lazy graphs; measurement support)."""
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        lib().ora_touch(self._h, _p(a) if len(a) else None, len(a), threads)

    def walk(self, app=APP_DEEPWALK, length=80, seed=0, first_walker=0, starts=None, num_walkers=None,
             p=1.0, q=1.0, stop=(1, 80), paths=True, counts=False, threads=0):
        W = num_walkers if num_walkers is not None else (len(starts) if starts is not None else self.V)
        st = np.ascontiguousarray(starts, dtype=np.uint32) if starts is not None else None
        pa = np.zeros(((length + 1), W), dtype=np.uint32) if (paths and length != NONE) else None
        ln = np.zeros(W, dtype=np.uint32)
        cn = np.zeros(self.V, dtype=np.uint64) if counts else None
        thr, alw = n2v_thresholds(p, q)
        sthr, salw = stop_threshold(*stop)
        dense = np.zeros(1, dtype=np.uint64)
        lib().ora_walk(self._h, app, length, seed, first_walker, _p(st), W, _p(pa), _p(ln), _p(cn),
                       _p(thr), _p(alw), sthr, salw, threads, _p(dense))
        return {"paths": pa, "lengths": ln, "counts": cn, "dense_attempts": int(dense[0])}

    def dump(self) -> bytes:
        n = lib().ora_dump(self._h, None, 0)
        buf = np.zeros(n, dtype=np.uint8)
        lib().ora_dump(self._h, _p(buf), n)
        return buf.tobytes()

    def dump_vertex(self, u: int) -> bytes:
        n = lib().ora_dump_vertex(self._h, u, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.uint8)
        lib().ora_dump_vertex(self._h, u, _p(buf), n)
        return buf[:n].tobytes()

    def vertex_digest(self, u: int) -> int:
        h = 0xcbf29ce484222325
        for b in self.dump_vertex(u):
            h ^= b
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
        return h

    def digests(self) -> np.ndarray:
        d = np.zeros(self.V, dtype=np.uint64)
        lib().ora_digests(self._h, _p(d))
        return d


def parse_dump(buf: bytes, V: int, float_mode: bool = False) -> list:
    """Parse the canonical dump (R-11) into per-vertex dicts (test helper)."""
    mv = memoryview(buf)
    pos = 0
    out = []

    def u32():
        nonlocal pos
        v = int.from_bytes(mv[pos:pos + 4], "little")
        pos += 4
        return v

    def u64():
        nonlocal pos
        v = int.from_bytes(mv[pos:pos + 8], "little")
        pos += 8
        return v

    for _ in range(V):
        d = u32()
        adj = [(u32(), u32(), u32()) for _ in range(d)]
        n = u32()
        groups = []
        for _ in range(n):
            k, c, kind, thr, al = u32(), u32(), u32(), u64(), u32()
            mem = None
            one = None
            if kind in (REGULAR, SPARSE):
                mem = [u32() for _ in range(c)]
            elif kind == ONE:
                one = u32()
            groups.append({"k": k, "c": c, "kind": kind, "thr": thr, "alias": al, "mem": mem, "one": one})
        T = u64()
        v = {"d": d, "adj": adj, "groups": groups, "T": T}
        if float_mode:
            v["lam"], v["fflags"], v["dmax"], v["thrD"] = u32(), u32(), u64(), u64()
            dc = u32()
            v["dec"] = [(u32(), u64()) for _ in range(dc)]
        out.append(v)
    assert pos == len(buf), (pos, len(buf))
    return out


class RadixGraph:
    """The arbitrary-radix-base structure (base B = 2^b, reading R-17): static
    build + sampling; DeepWalk and PPR walks."""

    def __init__(self, row_offsets, dst, bias, b: int):
        L = lib()
        self.V = len(row_offsets) - 1
        self.b = b
        ro = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        ds = np.ascontiguousarray(dst, dtype=np.uint32)
        bs = np.ascontiguousarray(bias, dtype=np.uint32)
        h = ctypes.c_void_p()
        rc = L.ora_build_radix(self.V, _p(ro), _p(ds), _p(bs), b, ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"ora_build_radix failed with status {rc}")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:
            lib().ora_radix_free(h)
            self._h = None

    def sample(self, u, seed, w, t) -> int:
        return int(lib().ora_radix_sample(self._h, u, seed, w, t))

    def apply_updates(self, recs) -> dict:
        """One batch (reading R-19): the base-2 adjacency readings R-6..R-9, then the touched
        vertices' nested structure rebuilt from their adjacency."""
        r = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 4)
        st = np.zeros(30, dtype=np.uint64)
        rc = int(lib().ora_radix_apply_updates(self._h, _p(r) if len(r) else None, len(r), _p(st)))
        if rc != 0:
            raise ValueError(f"ora_radix_apply_updates failed with status {rc}")
        return {"inserted": int(st[0]), "deleted": int(st[1]), "missing_deletes": int(st[2]),
                "touched_vertices": int(st[3]), "epoch": int(st[29])}

    def try_apply_updates(self, recs) -> int:
        r = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 4)
        return int(lib().ora_radix_apply_updates(self._h, _p(r) if len(r) else None, len(r), None))

    def adjacency(self, u):
        """[d, 3] uint32 array of (dst, bias, epoch) in adjacency order."""
        d = int(lib().ora_radix_adj(self._h, u, None))
        out = np.zeros((max(d, 1), 3), dtype=np.uint32)
        lib().ora_radix_adj(self._h, u, _p(out))
        return out[:d]

    def walk(self, app=APP_DEEPWALK, length=80, seed=0, first_walker=0, starts=None, num_walkers=None,
             stop=(1, 80), paths=True, counts=False, threads=0):
        W = num_walkers if num_walkers is not None else (len(starts) if starts is not None else self.V)
        st = np.ascontiguousarray(starts, dtype=np.uint32) if starts is not None else None
        pa = np.zeros(((length + 1), W), dtype=np.uint32) if (paths and length != NONE) else None
        ln = np.zeros(W, dtype=np.uint32)
        cn = np.zeros(self.V, dtype=np.uint64) if counts else None
        sthr, salw = stop_threshold(*stop)
        lib().ora_radix_walk(self._h, app, length, seed, first_walker, _p(st), W, _p(pa), _p(ln), _p(cn), sthr, salw,
                             threads)
        return {"paths": pa, "lengths": ln, "counts": cn}

    def dump(self) -> bytes:
        n = lib().ora_radix_dump(self._h, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.uint8)
        lib().ora_radix_dump(self._h, _p(buf), n)
        return buf[:n].tobytes()


def parse_radix_dump(buf: bytes, V: int) -> list:
    """Parse the radix canonical dump (R-18) into per-vertex dicts (test helper)."""
    mv = memoryview(buf)
    pos = 0

    def u32():
        nonlocal pos
        v = int.from_bytes(mv[pos:pos + 4], "little")
        pos += 4
        return v

    def u64():
        nonlocal pos
        v = int.from_bytes(mv[pos:pos + 8], "little")
        pos += 8
        return v
    out = []
    for _ in range(V):
        d, n = u32(), u32()
        groups = []
        for _ in range(n):
            i, thr, al, ns = u32(), u64(), u32(), u32()
            subs = []
            for _ in range(ns):
                j, c, sthr, sal = u32(), u32(), u64(), u32()
                subs.append({"j": j, "c": c, "thr": sthr, "alias": sal, "mem": [u32() for _ in range(c)]})
            groups.append({"i": i, "thr": thr, "alias": al, "subs": subs})
        out.append({"d": d, "groups": groups, "T": u64()})
    assert pos == len(buf), (pos, len(buf))
    return out
