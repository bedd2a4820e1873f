"""Industry-scale synthetic KG (BASELINE configs[4]: ~50M entities, ~1B
triples, d=128) generated on the device, one row block at a time.

The reference generator (data.py:356-411) is a per-user / per-item Python loop
that took 92 s at Amazon shape and cannot reach 10^9
triples; this one keeps its design -- users belong to one of G groups and
draw ``3 + Poisson(rate-3)`` items, with probability ``group_affinity`` from
their group (Zipf within the group) and otherwise from the global Zipf
popularity; every item links to its group's attribute hub (relation 0) plus
``Poisson(attr_links_per_item)`` uniform attribute entities (relations
1..R-1); a Bernoulli split keeps each user's first pair in train -- but is
written as counter-keyed chunks so that

* any chunk can be regenerated independently (``torch.Generator`` seeded by
  (seed, kind, chunk)), so every rank of a row partition streams the same
  global graph and keeps only the edges incident to its rows;
* duplicates can only arise inside one chunk (a user's own draws, an item's
  own attribute links) and are removed there, so the node degrees of the
  normalised adjacency are plain bincounts over the streamed edges.

``row_block`` returns the CSR rows [lo, hi) of D^-1/2 (A+I) D^-1/2 over
(train interactions + triples), values computed exactly as
``data.adjacency_arrays`` / the reference's build_adjacency (data.py:230-266):
float64 ``1 * inv_sqrt[row] * inv_sqrt[col]`` rounded once to fp32, columns
ascending.  The concatenation of all blocks equals ``adjacency_arrays`` of
``dataset()`` bit for bit (tested on CPU at small shapes).
"""

from dataclasses import dataclass

import numpy as np
import torch

from .data import KgDataset


@dataclass(frozen=True)
class IndustryShape:
    users: int = 5_000_000
    items: int = 2_000_000
    entities: int = 50_000_000
    relations: int = 64
    groups: int = 1000
    interactions_per_user: float = 40.0
    group_affinity: float = 0.85
    zipf: float = 0.8
    attr_links_per_item: float = 500.0    # ~1.0e9 triples at 2M items
    test_frac: float = 0.2
    user_chunk: int = 1 << 20
    item_chunk: int = 1 << 16

    @property
    def num_nodes(self) -> int:
        return self.users + self.entities


INDUSTRY = IndustryShape()

_USERS, _ITEMS = 1, 2


def _gen(seed: int, kind: int, chunk: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + kind * 7_919 + chunk * 104_729) & ((1 << 63) - 1))
    return g


def _zipf_cdf(n: int, a: float, device) -> torch.Tensor:
    w = 1.0 / torch.arange(1, n + 1, dtype=torch.float64, device=device).pow(a)
    c = torch.cumsum(w, 0)
    return c / c[-1]


class IndustryGraph:
    """Chunked generator of one ``IndustryShape`` on ``device``."""

    def __init__(self, shape: IndustryShape = INDUSTRY, seed: int = 0, device="cuda"):
        s = shape
        if s.items > s.entities or s.entities < s.items + s.groups or s.groups > s.items:
            raise ValueError("need items <= entities, room for the group hubs, groups <= items")
        self.shape, self.seed, self.device = s, seed, torch.device(device)
        self.n = s.users + s.entities
        self.per_group = -(-s.items // s.groups)
        self.gcdf = _zipf_cdf(self.per_group, s.zipf, self.device)
        self.icdf = _zipf_cdf(s.items, s.zipf, self.device)
        self.n_user_chunks = -(-s.users // s.user_chunk)
        self.n_item_chunks = -(-s.items // s.item_chunk)

    # -- chunks ------------------------------------------------------------
    def user_chunk(self, c: int):
        """(train pairs, test pairs) of users [c*UC, ...): int64 (n, 2) user, item."""
        s, dev = self.shape, self.device
        g = _gen(self.seed, _USERS, c, dev)
        u0 = c * s.user_chunk
        nu = min(s.user_chunk, s.users - u0)
        group = torch.randint(0, s.groups, (nu,), generator=g, device=dev)
        lam = torch.full((nu,), max(s.interactions_per_user - 3.0, 0.0), dtype=torch.float64, device=dev)
        want = torch.clamp(3 + torch.poisson(lam, generator=g).long(), max=s.items)
        uid = torch.repeat_interleave(torch.arange(nu, device=dev), want)
        m = uid.numel()
        in_group = torch.rand(m, generator=g, device=dev, dtype=torch.float64) < s.group_affinity
        r = torch.searchsorted(self.gcdf, torch.rand(m, generator=g, device=dev, dtype=torch.float64))
        gg = group[uid]
        count_g = (s.items - gg + s.groups - 1) // s.groups
        item_in = gg + (r % count_g) * s.groups
        item_gl = torch.searchsorted(self.icdf, torch.rand(m, generator=g, device=dev, dtype=torch.float64))
        item = torch.where(in_group, item_in, torch.clamp(item_gl, max=s.items - 1))
        key = torch.unique(uid * s.items + item)                  # sorted: by user, then item
        users, items = key // s.items + u0, key % s.items
        is_test = torch.rand(key.numel(), generator=g, device=dev, dtype=torch.float64) < s.test_frac
        first = torch.ones_like(is_test)
        first[1:] = users[1:] != users[:-1]
        is_test &= ~first
        pairs = torch.stack([users, items], 1)
        return pairs[~is_test], pairs[is_test]

    def item_chunk(self, c: int):
        """Triples (head item, relation, tail entity) of items [c*IC, ...), int64 (m, 3), lexsorted."""
        s, dev = self.shape, self.device
        g = _gen(self.seed, _ITEMS, c, dev)
        i0 = c * s.item_chunk
        ni = min(s.item_chunk, s.items - i0)
        lam = torch.full((ni,), s.attr_links_per_item, dtype=torch.float64, device=dev)
        n_extra = torch.poisson(lam, generator=g).long()
        heads = torch.repeat_interleave(torch.arange(i0, i0 + ni, device=dev), n_extra)
        free_lo = s.items + s.groups
        tails = torch.randint(free_lo, s.entities, (heads.numel(),), generator=g, device=dev)
        rels = torch.randint(1, max(s.relations, 2), (heads.numel(),), generator=g, device=dev)
        # relations are collapsed in the adjacency; one triple per (head, tail)
        key, inv = torch.unique(heads * s.entities + tails, return_inverse=True)
        rel_first = torch.full((key.numel(),), s.relations, dtype=torch.long, device=dev)
        rel_first.scatter_reduce_(0, inv, rels, reduce="amin")
        hub_h = torch.arange(i0, i0 + ni, device=dev)
        hub = torch.stack([hub_h, torch.zeros_like(hub_h), s.items + hub_h % s.groups], 1)
        extra = torch.stack([key // s.entities, rel_first, key % s.entities], 1)
        tri = torch.cat([hub, extra], 0)
        order = torch.argsort(tri[:, 0] * (s.relations * s.entities) + tri[:, 1] * s.entities + tri[:, 2])
        return tri[order]

    def edges(self):
        """Undirected node-id edges (a, b), a != b, each exactly once, by chunk."""
        U = self.shape.users
        for c in range(self.n_user_chunks):
            train, _ = self.user_chunk(c)
            yield train[:, 0], U + train[:, 1]
        for c in range(self.n_item_chunks):
            tri = self.item_chunk(c)
            yield U + tri[:, 0], U + tri[:, 2]

    # -- adjacency -----------------------------------------------------------
    def degrees(self) -> torch.Tensor:
        """Row counts of A + I (int64, all nodes)."""
        deg = torch.ones(self.n, dtype=torch.int64, device=self.device)
        for a, b in self.edges():
            deg += torch.bincount(a, minlength=self.n)
            deg += torch.bincount(b, minlength=self.n)
        return deg

    def partition(self, deg: torch.Tensor, world: int) -> np.ndarray:
        """Equal-nnz contiguous row cuts (data.partition_rows on the implied indptr)."""
        indptr = torch.zeros(self.n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(deg, 0, out=indptr[1:])
        from .data import partition_rows
        return partition_rows(indptr.cpu().numpy(), world)

    def row_block(self, lo: int, hi: int, deg: torch.Tensor):
        """CSR rows [lo, hi): (indptr int32 [hi-lo+1], indices int32, vals fp32), on the device."""
        dev = self.device
        keys = [torch.arange(lo, hi, device=dev) * self.n + torch.arange(lo, hi, device=dev)]
        for a, b in self.edges():
            for r, c in ((a, b), (b, a)):
                sel = (r >= lo) & (r < hi)
                if bool(sel.any()):
                    keys.append(r[sel] * self.n + c[sel])
        k = torch.sort(torch.cat(keys)).values
        del keys
        rows, cols = k // self.n, k % self.n
        del k
        inv = 1.0 / torch.sqrt(deg.to(torch.float64))
        vals = (inv[rows] * inv[cols]).to(torch.float32)   # (1 * inv_r) * inv_c, as numpy
        counts = torch.bincount(rows - lo, minlength=hi - lo)
        indptr = torch.zeros(hi - lo + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=indptr[1:])
        if int(indptr[-1]) >= 1 << 31:
            raise ValueError("row block has >= 2^31 nonzeros; use more ranks")
        return indptr.to(torch.int32), cols.to(torch.int32), vals

    def referenced_by_others(self, lo: int, hi: int, cuts) -> torch.Tensor:
        """For the row block [lo, hi): how many distinct local rows each rank
        (by ``cuts``) references through its own CSR block -- the send side
        of the halo exchange (HaloPlan.send_counts), from one streaming pass."""
        dev = self.device
        cuts_t = torch.as_tensor(np.asarray(cuts, dtype=np.int64), device=dev)
        n_loc = hi - lo
        keys = []
        for a, b in self.edges():
            for r, c in ((a, b), (b, a)):
                sel = (c >= lo) & (c < hi) & ((r < lo) | (r >= hi))
                if bool(sel.any()):
                    q = torch.searchsorted(cuts_t, r[sel], right=True) - 1
                    keys.append(torch.unique(q * n_loc + (c[sel] - lo)))
        if not keys:
            return torch.zeros(len(cuts) - 1, dtype=torch.int64, device=dev)
        k = torch.unique(torch.cat(keys))
        return torch.bincount(k // n_loc, minlength=len(cuts) - 1)

    # -- small shapes: the whole dataset (tests) ------------------------------
    def dataset(self) -> KgDataset:
        s = self.shape
        trains, tests, tris = [], [], []
        for c in range(self.n_user_chunks):
            tr, te = self.user_chunk(c)
            trains.append(tr)
            tests.append(te)
        for c in range(self.n_item_chunks):
            tris.append(self.item_chunk(c))
        cat = lambda xs, w: torch.cat(xs, 0).cpu().numpy().astype(np.int32).reshape(-1, w)
        return KgDataset(s.users, s.items, s.entities, cat(trains, 2), np.zeros((0, 2), np.int32),
                         cat(tests, 2), cat(tris, 3), s.relations)
