"""synth -- seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the Bingo method: it only produces graphs,
biases, update streams and walker start lists ("Input
recipe").  Both ``oracle`` (through tests/bench) and ``paper_2504_10233_b200``
consume its outputs; neither side's code lives here.

Recipe (PAPER.md S6.1 P:656-665):
* R-MAT (a, b, c, d) = (0.57, 0.19, 0.19, 0.05) on 2^scale ids; self loops and
  duplicate edges dropped (a simple base graph); random vertex relabelling;
  symmetrised (each undirected edge -> two arcs); optionally compacted to the
  non-isolated vertices so that V matches the dataset shape.
* Biases "based on the degree of vertices": w(u, v) = max(1, deg(v))
  (reading R-12), optionally clamped (config 1: 1..255); uniform and
  log-uniform variants exercise every group kind.
* Update stream: hold out R * BS undirected edges as B, the rest is the
  initial graph A; each event flips a fair coin (Mixed): delete a
  uniform live edge of A, or insert a uniform unused edge of B into A.  Each
  undirected event becomes two arc records {op, src, dst, bias}.
"""
from __future__ import annotations

import numpy as np

RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)
INSERT, DELETE = 0, 1

# name -> recipe.  V / arcs are the targets of BASELINE.json configs; "scale" and
# "edges" are the generator parameters that land near them.
CONFIGS = {
    "c1": dict(desc="tiny power-law 1K V / 16K arcs, biases 1-255", scale=10, edges=11850,
               compact=False, bias="degree", clamp=(1, 255), batch=500, app="deepwalk"),
    "c2": dict(desc="LiveJournal-shaped R-MAT (4.8M V, 69M arcs), DeepWalk, 100K-edge batches",
               scale=24, edges=35_000_000, compact=True, bias="degree", clamp=None, batch=50_000,
               app="deepwalk"),
    "c3": dict(desc="Orkut-shaped R-MAT (3.1M V, 234M arcs), node2vec p=2 q=0.5, 1M-edge batches",
               scale=22, edges=125_000_000, compact=True, bias="degree", clamp=None, batch=1_000_000,
               app="node2vec"),
    "c4": dict(desc="Twitter-shaped R-MAT (41.7M V, 1.47B arcs), PPR", scale=27, edges=740_000_000,
               compact=True, bias="degree", clamp=None, batch=50_000, app="ppr"),
    "c5": dict(desc="Friendster-shaped R-MAT (65.6M V, 3.6B arcs), streaming updates + DeepWalk batches",
               scale=27, edges=1_830_000_000, compact=True, bias="degree", clamp=None, batch=1,
               app="deepwalk"),
}


def rmat_edges(scale: int, n_edges: int, seed: int, abcd=RMAT_ABCD, chunk: int = 1 << 24, device="cpu"):
    """Raw directed R-MAT endpoint pairs (int64 ids < 2^scale), torch RNG on `device`
    (the CPU and CUDA streams differ; each is deterministic for a given seed)."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    a, b, c, _ = abcd
    src = torch.empty(n_edges, dtype=torch.int64, device=device)
    dst = torch.empty(n_edges, dtype=torch.int64, device=device)
    for lo in range(0, n_edges, chunk):
        hi = min(n_edges, lo + chunk)
        m = hi - lo
        s = torch.zeros(m, dtype=torch.int64, device=device)
        t = torch.zeros(m, dtype=torch.int64, device=device)
        for lvl in range(scale):
            r = torch.rand(m, generator=g, device=device)
            bit = 1 << (scale - 1 - lvl)
            # quadrant: [0,a) -> (0,0); [a,a+b) -> (0,1); [a+b,a+b+c) -> (1,0); else (1,1)
            down = r >= (a + b)
            right = ((r >= a) & (r < a + b)) | (r >= a + b + c)
            s += down.to(torch.int64) * bit
            t += right.to(torch.int64) * bit
        src[lo:hi] = s
        dst[lo:hi] = t
    return src, dst


def simple_undirected(scale: int, n_edges: int, seed: int, compact: bool, device="cpu", resident=False):
    """Undirected simple edge list (lo < hi pairs, unique) with a random relabelling.
    resident=True returns int32 tensors on `device` instead of numpy u32 arrays."""
    import torch
    s, t = rmat_edges(scale, n_edges, seed, device=device)
    keep = s != t
    s, t = s[keep], t[keep]
    key = torch.unique((torch.minimum(s, t) << 32) | torch.maximum(s, t))
    del s, t
    lo = key >> 32
    hi = key & 0xFFFFFFFF
    n_ids = 1 << scale
    if compact:
        used = torch.zeros(n_ids, dtype=torch.bool, device=device)
        used[lo] = True
        used[hi] = True
        newid = torch.cumsum(used.to(torch.int64), 0) - 1
        V = int(used.sum())
        lo, hi = newid[lo], newid[hi]
    else:
        V = n_ids
    g = torch.Generator(device=device).manual_seed(seed + 1000003)
    perm = torch.randperm(V, generator=g, device=device)
    lo, hi = perm[lo], perm[hi]
    a = torch.minimum(lo, hi).to(torch.int32)
    b = torch.maximum(lo, hi).to(torch.int32)
    del lo, hi, perm
    if resident:
        return V, a, b
    return V, a.cpu().numpy().view(np.uint32), b.cpu().numpy().view(np.uint32)


def csr_from_arcs(V: int, src: np.ndarray, dst: np.ndarray, extra=None, device="cpu", lim: int = 1 << 30):
    """CSR with arcs ordered by (src, dst); returns row_offsets u64, dst u32 (+ extra permuted).
    Large inputs are sorted in source-vertex ranges of < 2^30 arcs (torch.sort's limit)."""
    import torch
    counts = np.bincount(src, minlength=V).astype(np.uint64)
    ro = np.zeros(V + 1, dtype=np.uint64)
    np.cumsum(counts, out=ro[1:])
    n = len(src)
    LIM = lim
    if n <= LIM:
        key = (torch.from_numpy(src.astype(np.int64)).to(device) << 32) | torch.from_numpy(dst.astype(np.int64)).to(device)
        order = torch.sort(key, stable=True).indices.cpu().numpy()
        del key
    else:
        s_t = torch.from_numpy(src.view(np.int32)).to(device)
        d_t = torch.from_numpy(dst.view(np.int32)).to(device)
        order = np.empty(n, dtype=np.int64)
        v0 = 0
        while v0 < V:
            # the largest v1 with ro[v1] - ro[v0] <= LIM (at least one vertex)
            v1 = int(np.searchsorted(ro, ro[v0] + LIM, side="right")) - 1
            v1 = max(v1, v0 + 1)
            m = (s_t >= v0) & (s_t < v1)
            idx = m.nonzero().squeeze(1)
            del m
            key = (s_t[idx].to(torch.int64) << 32) | d_t[idx].to(torch.int64)
            o = torch.sort(key, stable=True).indices
            order[int(ro[v0]):int(ro[v1])] = idx[o].cpu().numpy()
            del idx, key, o
            v0 = v1
        del s_t, d_t
    d = dst[order].astype(np.uint32)
    if extra is not None:
        return ro, d, extra[order]
    return ro, d


def degree_bias_of(deg: np.ndarray, dst: np.ndarray, clamp=None) -> np.ndarray:
    """w(u, v) = max(1, deg(v)) (reading R-12), optionally clamped."""
    w = np.maximum(deg[dst].astype(np.int64), 1)
    if clamp is not None:
        w = np.clip(w, clamp[0], clamp[1])
    return w.astype(np.uint32)


def make_workload(name: str, rounds: int = 1, device="cpu", hold_rounds=None, resident=False,
                  **over):
    """resident=True (device must be CUDA): the graph stays in HBM as tensors
    (DeviceWorkload); otherwise numpy arrays (Workload)."""
    cfg = dict(CONFIGS[name])
    cfg.update(over)
    cls = DeviceWorkload if resident else Workload
    return cls(cfg["scale"], cfg["edges"], compact=cfg["compact"], bias=cfg["bias"],
               clamp=cfg["clamp"], batch=cfg["batch"], rounds=rounds, device=device, hold_rounds=hold_rounds)


class Workload:
    """A seeded graph + update stream following the recipe above.

    hold_rounds: the held-out set B is hold_rounds x batch edges (default: `rounds`), so the
    initial graph does not depend on how many batches are drawn (P:658 holds out the edges of
    its 10 rounds); batch i is the same whatever `rounds` is.  Once B is used up, edges deleted
    earlier become insertable again (the stream never runs dry)."""

    def __init__(self, scale, edges, seed=1, compact=True, bias="degree", clamp=None, batch=1000,
                 rounds=1, update_seed=2, undirected=True, device="cpu", hold_rounds=None):
        V, a, b = simple_undirected(scale, edges, seed, compact, device=device)
        self.V = V
        E = len(a)
        # full-graph degrees fix every bias, including those of later inserts
        deg_full = np.bincount(a, minlength=V) + np.bincount(b, minlength=V)
        rng = np.random.default_rng(update_seed)
        n_hold = min(E // 2, (hold_rounds if hold_rounds is not None else rounds) * batch)
        perm = rng.permutation(E)
        held = perm[:n_hold]
        live = perm[n_hold:]
        self._setup(V, batch, rounds, deg_full, bias, clamp, seed)
        # initial graph A
        src = np.concatenate([a[live], b[live]])
        dst = np.concatenate([b[live], a[live]])
        w = self._bias(src, dst)
        self.row_offsets, self.dst, self.bias = csr_from_arcs(V, src, dst, extra=w, device=device)
        del src, dst, w
        self.num_arcs = int(self.row_offsets[-1])
        self.batches = []
        for ev_src, ev_dst, ops in _update_events(rng, live, held, batch, rounds, lambda e: (a[e], b[e])):
            self.batches.append(self._records(ev_src, ev_dst, ops))

    def _setup(self, V, batch, rounds, deg_full, bias, clamp, seed):
        self.V = V
        self.batch = batch
        self.rounds = rounds
        self.deg_full = deg_full
        self.bias_kind = bias
        self.clamp = clamp
        self._bias_seed = seed + 7

    def _records(self, src_r, dst_r, ops):
        """Each undirected event -> two arc records {op, src, dst, bias} (S5.2)."""
        n = len(ops)
        recs = np.zeros((2 * n, 4), dtype=np.uint32)
        recs[0::2, 0] = ops
        recs[1::2, 0] = ops
        recs[0::2, 1] = src_r
        recs[0::2, 2] = dst_r
        recs[1::2, 1] = dst_r
        recs[1::2, 2] = src_r
        ins = ops == INSERT
        recs[0::2, 3] = np.where(ins, self._bias(src_r, dst_r), 0)
        recs[1::2, 3] = np.where(ins, self._bias(dst_r, src_r), 0)
        return recs

    def _bias(self, src, dst):
        if self.bias_kind == "degree":
            return degree_bias_of(self.deg_full, dst, self.clamp)
        lo, hi = self.clamp if self.clamp else (1, 255)
        # edge-keyed hash so that the same arc always gets the same bias
        h = (src.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15) ^
             (dst.astype(np.uint64) + np.uint64(self._bias_seed)) * np.uint64(0xC2B2AE3D27D4EB4F))
        h ^= h >> np.uint64(29)
        h *= np.uint64(0xBF58476D1CE4E5B9)
        h ^= h >> np.uint64(32)
        x = (h >> np.uint64(11)).astype(np.float64) / float(1 << 53)
        if self.bias_kind == "uniform":
            return (lo + np.floor(x * (hi - lo + 1))).astype(np.uint32)
        if self.bias_kind == "loguniform":
            return np.floor(np.exp(np.log(lo) + x * (np.log(hi + 1) - np.log(lo)))).clip(lo, hi).astype(np.uint32)
        raise ValueError(self.bias_kind)


def _update_events(rng, live, held, batch, rounds, endpoints):
    """The P:658 stream over edge ids: per event a fair coin (Mixed) -- delete a
    uniform live edge (swap-remove from the live list) or insert the next unused edge of the
    shuffled held-out pool; a deleted edge joins the end of the pool, so inserts continue
    once the held-out edges are used up.  Yields (src, dst, ops) per round; `endpoints(e)`
    maps an int array of edge ids to their (lo, hi) endpoint arrays."""
    live_list = np.array(live, dtype=np.int64)       # a private copy: swap-removal mutates it
    n_live = len(live_list)
    pool = list(np.array(held, dtype=np.int64)[rng.permutation(len(held))])
    pool_pos = 0
    for _ in range(rounds):
        ops = rng.integers(0, 2, size=batch)
        uni = rng.random(batch)
        ev = np.zeros(batch, dtype=np.int64)
        for i in range(batch):
            if (ops[i] == 1 and n_live > 0) or pool_pos >= len(pool):
                ops[i] = 1
                j = int(uni[i] * n_live)
                e = int(live_list[j])
                live_list[j] = live_list[n_live - 1]
                n_live -= 1
                pool.append(e)
            else:
                ops[i] = 0
                e = int(pool[pool_pos])
                pool_pos += 1
                if n_live == len(live_list):
                    live_list = np.concatenate([live_list, np.zeros(max(1024, batch), live_list.dtype)])
                live_list[n_live] = e
                n_live += 1
            ev[i] = e
        src_r, dst_r = endpoints(ev)
        yield np.asarray(src_r, dtype=np.int64), np.asarray(dst_r, dtype=np.int64), ops


class DeviceWorkload(Workload):
    """The same recipe with the graph generated and kept in HBM (torch CUDA ops): R-MAT,
    simple + relabelled + symmetrised, the held-out split, the (src, dst)-sorted CSR and the
    degree biases never leave the device.  row_offsets (int64), dst and bias (int32 holding
    u32) are CUDA tensors; the update batches are numpy (the host stream of P:658; edge ids
    are drawn on the host, their endpoints gathered on the device).  `host_csr()` copies the
    CSR out for the CPU oracle.  Minutes -> seconds at Twitter/Friendster scale."""

    def __init__(self, scale, edges, seed=1, compact=True, bias="degree", clamp=None, batch=1000,
                 rounds=1, update_seed=2, undirected=True, device="cuda", hold_rounds=None):
        import torch
        dev = torch.device(device)
        assert dev.type == "cuda", "DeviceWorkload keeps the graph in HBM"
        if bias != "degree":
            raise ValueError("DeviceWorkload: degree biases only (P:664)")
        V, a, b = simple_undirected(scale, edges, seed, compact, device=dev, resident=True)
        E = a.numel()
        deg_full = torch.bincount(a, minlength=V) + torch.bincount(b, minlength=V)
        self._setup(V, batch, rounds, deg_full.cpu().numpy(), bias, clamp, seed)
        n_hold = min(E // 2, (hold_rounds if hold_rounds is not None else rounds) * batch)
        g = torch.Generator(device=dev).manual_seed(update_seed)
        perm = torch.randperm(E, generator=g, device=dev)
        held, live = perm[:n_hold], perm[n_hold:]
        # initial graph A: both arcs of every live edge, CSR sorted by (src, dst)
        la, lb = a[live], b[live]
        src = torch.cat([la, lb])
        dst = torch.cat([lb, la])
        del la, lb
        cnt = torch.bincount(src, minlength=V)
        ro = torch.zeros(V + 1, dtype=torch.int64, device=dev)
        ro[1:] = torch.cumsum(cnt, 0)
        del cnt
        key = (src.to(torch.int64) << 32) | dst.to(torch.int64)
        del dst
        out = torch.empty_like(key)
        ro_h = ro.cpu().numpy()
        v0 = 0
        LIM = 1 << 30                   # sort in source-vertex ranges of <= 2^30 arcs
        while v0 < V:
            v1 = max(int(np.searchsorted(ro_h, ro_h[v0] + LIM, side="right")) - 1, v0 + 1)
            if v0 == 0 and v1 >= V:
                out = torch.sort(key).values
            else:
                m = (src >= v0) & (src < v1)
                out[int(ro_h[v0]):int(ro_h[v1])] = torch.sort(key[m]).values
                del m
            v0 = v1
        del key, src
        dsorted = (out & 0xFFFFFFFF).to(torch.int32)
        del out
        w = torch.clamp(deg_full[dsorted.to(torch.int64)], min=1)
        if clamp is not None:
            w = torch.clamp(w, clamp[0], clamp[1])
        self.row_offsets = ro
        self.dst = dsorted
        self.bias = w.to(torch.int64).to(torch.int32)
        del w
        self.num_arcs = int(ro_h[-1])
        rng = np.random.default_rng(update_seed)
        live_h = live.to(torch.int32).cpu().numpy()
        held_h = held.cpu().numpy()
        del perm, held, live

        def endpoints(ev):
            idx = torch.from_numpy(ev).to(dev)
            return a[idx].cpu().numpy().view(np.uint32), b[idx].cpu().numpy().view(np.uint32)
        self.batches = [self._records(s_, d_, o_)
                        for s_, d_, o_ in _update_events(rng, live_h, held_h, batch, rounds, endpoints)]
        del a, b
        torch.cuda.empty_cache()

    def host_csr(self):
        """(row_offsets u64, dst u32, bias u32) numpy copies for the CPU oracle."""
        return (self.row_offsets.cpu().numpy().view(np.uint64), self.dst.cpu().numpy().view(np.uint32),
                self.bias.cpu().numpy().view(np.uint32))


def random_small_graph(rng: np.random.Generator, V: int, max_deg: int, max_bias: int, directed=True):
    """Tiny random multigraph CSR (duplicates allowed) for property tests."""
    deg = rng.integers(0, max_deg + 1, size=V)
    ro = np.zeros(V + 1, dtype=np.uint64)
    ro[1:] = np.cumsum(deg)
    A = int(ro[-1])
    dst = rng.integers(0, V, size=A).astype(np.uint32)
    bias = rng.integers(1, max_bias + 1, size=A).astype(np.uint32)
    return ro, dst, bias


def random_batch(rng: np.random.Generator, V: int, n: int, max_bias: int, existing=None, p_delete=0.5):
    """Random mixed arc batch; deletes target existing arcs (from `existing`
    = list of (src, dst)) with probability 0.8, else random (possibly missing)."""
    recs = np.zeros((n, 4), dtype=np.uint32)
    for i in range(n):
        if rng.random() < p_delete:
            if existing and rng.random() < 0.8:
                s, d = existing[int(rng.integers(0, len(existing)))]
            else:
                s, d = int(rng.integers(0, V)), int(rng.integers(0, V))
            recs[i] = (DELETE, s, d, 0)
        else:
            recs[i] = (INSERT, int(rng.integers(0, V)), int(rng.integers(0, V)), int(rng.integers(1, max_bias + 1)))
    return recs
