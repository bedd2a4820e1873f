"""Input formats consumed by the hot path: the unified user/entity graph.

Host-side preprocessing (numpy), restated from the reference's semantics
(kgact.data, /root/reference/pkg/src/kgact/data.py) -- this is the caller
side of the hot path, not the hot path itself:

* ``KgDataset``: users in [0, U), entities in [U, U+E) with items as the
  first entity slots (data.py:1-12, :35-57).
* ``build_adjacency``: symmetric D^-1/2 (A+I) D^-1/2 over the union of train
  interactions and KG triples, relations collapsed (data.py:230-266); values
  computed in float64 in the reference's order, so the CSR is bit-identical.
* ``sample_negatives``: one uniform negative per train pair with rejection of
  the user's train items, drawing from the caller's numpy Generator in the
  reference's order (data.py:274-294), so batches are identical.
* ``synth_kg``: a vectorized synthetic KG generator with the reference's
  design (block-structured user groups, Zipf item popularity, one attribute
  hub per group plus Poisson extra attribute links; data.py:301-411) for the
  large shapes (Last-FM / Amazon-book / industry), where the reference's
  Python-loop generator does not scale.  Its RNG stream
  differs from the reference's, so it is used for throughput, not parity;
  parity runs use datasets produced by the reference (tests/golden/, and
  ``reference_dataset`` for the Amazon-book / Last-FM shapes).
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from .tensorops import CSR


class SamplingError(RuntimeError):
    """data.py:28."""


@dataclass
class KgDataset:
    num_users: int
    num_items: int
    num_entities: int
    train: np.ndarray       # (n, 2) int32 (user, item)
    val: np.ndarray
    test: np.ndarray
    triples: np.ndarray     # (m, 3) int32 (head, relation, tail), entity ids
    num_relations: int = 1
    _train_keys: np.ndarray | None = field(default=None, repr=False)
    # string <-> index vocabularies (data.py:44-46); None for generated graphs
    user_vocab: dict | None = field(default=None, repr=False)
    entity_vocab: dict | None = field(default=None, repr=False)
    relation_vocab: dict | None = field(default=None, repr=False)

    def validate(self) -> None:
        """data.py:67-90 (vectorized): index ranges, no pair in two splits,
        triple endpoints / relations in range, items a prefix of entities."""
        for name, arr in (("train", self.train), ("val", self.val), ("test", self.test)):
            if len(arr):
                if arr[:, 0].min() < 0 or arr[:, 0].max() >= self.num_users:
                    raise ValueError(f"{name}: user index out of range")
                if arr[:, 1].min() < 0 or arr[:, 1].max() >= self.num_items:
                    raise ValueError(f"{name}: item index out of range")
        parts = [a for a in (self.train, self.val, self.test) if len(a)]
        if parts:
            allp = np.concatenate(parts).astype(np.int64)
            keys = allp[:, 0] * max(self.num_items, 1) + allp[:, 1]
            if len(np.unique(keys)) != len(keys):
                raise ValueError("a pair appears in more than one split")
        if len(self.triples):
            ends = self.triples[:, [0, 2]]
            if ends.min() < 0 or ends.max() >= self.num_entities:
                raise ValueError("triple endpoint out of entity range")
            n_rel = len(self.relation_vocab) if self.relation_vocab is not None else self.num_relations
            rels = self.triples[:, 1]
            if rels.min() < 0 or rels.max() >= n_rel:
                raise ValueError("triple relation out of range")
        if self.num_items > self.num_entities:
            raise ValueError("items must be a prefix of the entity space")

    @property
    def num_nodes(self) -> int:
        return self.num_users + self.num_entities

    def item_node(self, item):
        return self.num_users + item

    def train_keys(self) -> np.ndarray:
        """Sorted unique user*num_items+item keys of the train split."""
        if self._train_keys is None:
            t = self.train.astype(np.int64)
            self._train_keys = np.unique(t[:, 0] * self.num_items + t[:, 1])
        return self._train_keys

    def train_positives(self) -> list[set]:
        pos = [set() for _ in range(self.num_users)]
        for u, i in self.train:
            pos[int(u)].add(int(i))
        return pos

    @classmethod
    def from_npz(cls, path) -> "KgDataset":
        z = np.load(path)
        return cls(int(z["num_users"]), int(z["num_items"]), int(z["num_entities"]),
                   z["train"].astype(np.int32), z["val"].astype(np.int32).reshape(-1, 2),
                   z["test"].astype(np.int32).reshape(-1, 2), z["triples"].astype(np.int32).reshape(-1, 3),
                   int(z["num_relations"]) if "num_relations" in z else 1)

    def save_npz(self, path) -> None:
        np.savez_compressed(path, num_users=self.num_users, num_items=self.num_items,
                            num_entities=self.num_entities, train=self.train, val=self.val,
                            test=self.test, triples=self.triples, num_relations=self.num_relations)


def _uint(n: int):
    return np.uint8 if n < 1 << 8 else np.uint16 if n < 1 << 16 else np.uint32


def pack_dataset(ds: KgDataset) -> dict:
    """Lossless compact arrays of a dataset in the reference generator's
    canonical order (splits grouped by ascending user, split_interactions
    data.py:200-227; triples lexsorted, data.py:392): per-user run counts +
    narrow item ids, per-head counts + relations + within-(head, relation)
    tail deltas as byte planes.  ~5x smaller than the raw int32 arrays
    after compression."""
    out = {"num_users": ds.num_users, "num_items": ds.num_items, "num_entities": ds.num_entities,
           "num_relations": ds.num_relations}
    for name in ("train", "val", "test"):
        a = np.asarray(getattr(ds, name)).reshape(-1, 2)
        if len(a) and np.any(np.diff(a[:, 0]) < 0):
            raise ValueError(f"{name}: pairs are not grouped by ascending user")
        cnt = np.bincount(a[:, 0], minlength=ds.num_users) if len(a) else np.zeros(ds.num_users, np.int64)
        out[f"{name}_ucount"] = cnt.astype(_uint(int(cnt.max(initial=0)) + 1))
        out[f"{name}_item"] = a[:, 1].astype(_uint(ds.num_items))
    t = np.asarray(ds.triples).reshape(-1, 3).astype(np.int64)
    if len(t):
        order = np.lexsort((t[:, 2], t[:, 1], t[:, 0]))
        if np.any(order != np.arange(len(t))):
            raise ValueError("triples are not lexsorted by (head, relation, tail)")
    hc = np.bincount(t[:, 0], minlength=ds.num_entities) if len(t) else np.zeros(ds.num_entities, np.int64)
    out["tri_hcount"] = hc.astype(_uint(int(hc.max(initial=0)) + 1))
    out["tri_rel"] = t[:, 1].astype(_uint(max(ds.num_relations, int(t[:, 1].max(initial=0)) + 1)))
    start = np.ones(len(t), bool)
    start[1:] = (t[1:, 0] != t[:-1, 0]) | (t[1:, 1] != t[:-1, 1])
    delta = t[:, 2].copy()
    delta[1:] -= np.where(start[1:], 0, t[:-1, 2])
    nb = max(1, (int(delta.max(initial=0)).bit_length() + 7) // 8)
    # byte planes: zlib finds the near-constant high bytes (~25% smaller)
    out["tri_tdelta_planes"] = np.stack([(delta >> (8 * i)).astype(np.uint8) for i in range(nb)])
    return out


def unpack_dataset(z) -> KgDataset:
    """Inverse of ``pack_dataset`` (bit-identical arrays)."""
    U, I, E = int(z["num_users"]), int(z["num_items"]), int(z["num_entities"])
    splits = {}
    for name in ("train", "val", "test"):
        cnt = z[f"{name}_ucount"].astype(np.int64)
        users = np.repeat(np.arange(U, dtype=np.int32), cnt)
        splits[name] = np.stack([users, z[f"{name}_item"].astype(np.int32)], axis=1).reshape(-1, 2)
    heads = np.repeat(np.arange(E, dtype=np.int64), z["tri_hcount"].astype(np.int64))
    rels = z["tri_rel"].astype(np.int64)
    planes = z["tri_tdelta_planes"].astype(np.int64)
    delta = np.zeros(planes.shape[1], np.int64)
    for i in range(planes.shape[0]):
        delta |= planes[i] << (8 * i)
    start = np.ones(len(heads), bool)
    start[1:] = (heads[1:] != heads[:-1]) | (rels[1:] != rels[:-1])
    cs = np.cumsum(delta)
    run = np.cumsum(start) - 1
    base = (cs - delta)[start]
    tails = cs - base[run] if len(heads) else cs
    tri = np.stack([heads, rels, tails], axis=1).astype(np.int32).reshape(-1, 3)
    return KgDataset(U, I, E, splits["train"], splits["val"], splits["test"], tri, int(z["num_relations"]))


def save_compact(ds: KgDataset, path) -> None:
    np.savez_compressed(path, **pack_dataset(ds))


def load_compact(path) -> KgDataset:
    with np.load(path) as z:
        return unpack_dataset(z)


REFERENCE_DATASETS = ("amazon", "lastfm", "default")


def reference_dataset(name: str) -> KgDataset:
    """The Amazon-book / Last-FM-shaped datasets exactly as the REFERENCE
    generator produces them (synth_generate, data.py:356-411, seed 0, spec
    overrides of SURVEY.md 8(d)); written by datasets/make_reference_datasets.py."""
    import os
    if name not in REFERENCE_DATASETS:
        raise ValueError(f"no reference dataset {name!r} (have {REFERENCE_DATASETS})")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return load_compact(os.path.join(root, "datasets", f"{name}_seed0.npz"))


def adjacency_arrays(ds: KgDataset):
    """CSR arrays (indptr int32, indices int32, data fp32) of the normalized
    adjacency, data.py:230-266 semantics."""
    n = ds.num_nodes
    heads, tails = [], []
    if len(ds.train):
        heads.append(ds.train[:, 0].astype(np.int64))
        tails.append(ds.num_users + ds.train[:, 1].astype(np.int64))
    if len(ds.triples):
        heads.append(ds.num_users + ds.triples[:, 0].astype(np.int64))
        tails.append(ds.num_users + ds.triples[:, 2].astype(np.int64))
    if heads:
        a = np.concatenate(heads)
        b = np.concatenate(tails)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        keep = lo != hi
        enc = np.unique(lo[keep] * n + hi[keep])          # undirected, deduplicated
        lo, hi = enc // n, enc % n
        diag = np.arange(n, dtype=np.int64)
        rows = np.concatenate([lo, hi, diag])
        cols = np.concatenate([hi, lo, diag])
    else:
        rows = cols = np.arange(n, dtype=np.int64)
    order = np.lexsort((cols, rows))                       # canonical: row-major, sorted columns
    rows, cols = rows[order], cols[order]
    deg = np.bincount(rows, minlength=n).astype(np.float64)
    inv_sqrt = 1.0 / np.sqrt(deg)
    vals = (np.ones(len(rows), dtype=np.float64) * inv_sqrt[rows] * inv_sqrt[cols]).astype(np.float32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    return indptr.astype(np.int32), cols.astype(np.int32), vals


def build_adjacency(ds: KgDataset, device="cuda") -> CSR:
    indptr, indices, vals = adjacency_arrays(ds)
    n = ds.num_nodes
    return CSR.from_arrays(indptr, indices, vals, (n, n), device=device, symmetric=True)


def sample_negatives(ds: KgDataset, rng: np.random.Generator, pairs: np.ndarray | None = None) -> np.ndarray:
    """data.py:274-294: one uniform negative per pair, redrawn while it is a
    train positive of that user.  Same Generator calls as the reference."""
    if pairs is None:
        pairs = ds.train
    keys = ds.train_keys()
    users = pairs[:, 0].astype(np.int64)
    per_user = np.bincount(keys // ds.num_items, minlength=ds.num_users)
    if np.any(per_user[np.unique(users)] >= ds.num_items):
        raise SamplingError("a user has interacted with every item")
    n = len(pairs)
    neg = rng.integers(0, ds.num_items, size=n, dtype=np.int64)

    def is_pos(u, i):
        k = u * ds.num_items + i
        pos = np.searchsorted(keys, k)
        pos = np.minimum(pos, len(keys) - 1) if len(keys) else pos
        return keys[pos] == k if len(keys) else np.zeros(len(k), dtype=bool)

    pending = is_pos(users, neg)
    while pending.any():
        idx = np.nonzero(pending)[0]
        redraw = rng.integers(0, ds.num_items, size=len(idx), dtype=np.int64)
        neg[idx] = redraw
        pending[idx] = is_pos(users[idx], redraw)
    out = np.empty((n, 3), dtype=np.int32)
    out[:, :2] = pairs
    out[:, 2] = neg
    return out


# ---------------------------------------------------------------------------
# Vectorized synthetic KG (throughput shapes)
# ---------------------------------------------------------------------------

@dataclass
class SynthShape:
    users: int
    items: int
    entities: int
    relations: int = 5
    groups: int = 10
    interactions_per_user: float = 6.0
    group_affinity: float = 0.85
    zipf: float = 0.8
    attr_links_per_item: float = 1.0


SHAPES = {
    # BASELINE.json configs; rates as SURVEY.md 8(d) uses with the reference generator
    "small": SynthShape(2000, 3000, 10000, relations=20),
    "lastfm": SynthShape(23566, 48123, 58266, relations=9, interactions_per_user=128.8,
                         attr_links_per_item=8.66),
    "amazon": SynthShape(70679, 24915, 88572, relations=39, interactions_per_user=12.0,
                         attr_links_per_item=101.7),
    "industry": SynthShape(5_000_000, 2_000_000, 50_000_000, relations=64, groups=1000,
                           interactions_per_user=40.0, attr_links_per_item=250.0),
}


def _zipf_cdf(n, a):
    w = 1.0 / np.power(np.arange(1, n + 1, dtype=np.float64), a)
    c = np.cumsum(w)
    return c / c[-1]


def synth_kg(shape: SynthShape, seed: int = 0, test_frac: float = 0.2) -> KgDataset:
    """Vectorized generator with the reference's design (module docstring)."""
    rng = np.random.default_rng(seed)
    U, I, E, Gn = shape.users, shape.items, shape.entities, shape.groups
    item_group = np.arange(I) % Gn
    user_group = rng.integers(0, Gn, size=U)
    # interactions: 3 + Poisson(rate - 3) draws per user, group-affine Zipf
    want = np.minimum(3 + rng.poisson(max(shape.interactions_per_user - 3.0, 0.0), size=U), I)
    uid = np.repeat(np.arange(U, dtype=np.int64), want)
    m = len(uid)
    in_group = rng.random(m) < shape.group_affinity
    per_group = np.ceil(I / Gn).astype(np.int64)
    gcdf = _zipf_cdf(per_group, shape.zipf)
    r = np.searchsorted(gcdf, rng.random(m))                 # rank within the group
    g = user_group[uid]
    count_g = (I - g + Gn - 1) // Gn                          # items of group g: g, g+Gn, ...
    item_in = g + (r % count_g) * Gn
    item_glob = np.searchsorted(_zipf_cdf(I, shape.zipf), rng.random(m))
    item = np.where(in_group, item_in, item_glob).astype(np.int64)
    key = np.unique(uid * I + item)
    pairs = np.stack([key // I, key % I], axis=1).astype(np.int32)
    # split: per pair Bernoulli test membership, keeping >= 1 train item per user
    is_test = rng.random(len(pairs)) < test_frac
    first = np.r_[True, pairs[1:, 0] != pairs[:-1, 0]]
    is_test &= ~first
    train, test = pairs[~is_test], pairs[is_test]
    # triples: item -> its group hub (relation 0) + Poisson extra attribute links
    hub = I + item_group
    n_extra = rng.poisson(shape.attr_links_per_item, size=I)
    heads = np.concatenate([np.arange(I), np.repeat(np.arange(I), n_extra)])
    free_lo = I + Gn
    tails = np.concatenate([hub, rng.integers(free_lo, E, size=int(n_extra.sum()))])
    rels = np.concatenate([np.zeros(I, dtype=np.int64),
                           rng.integers(1, max(shape.relations, 2), size=int(n_extra.sum()))])
    tri = np.unique(np.stack([heads, rels, tails], axis=1).astype(np.int64), axis=0).astype(np.int32)
    return KgDataset(U, I, E, train, np.zeros((0, 2), np.int32), test, tri, shape.relations)


# ---------------------------------------------------------------------------
# Row partitioning (multi-GPU)
# ---------------------------------------------------------------------------

def partition_rows(indptr: np.ndarray, world: int) -> np.ndarray:
    """Equal-nnz contiguous row ranges cut on indptr:
    returns world+1 row boundaries."""
    n = len(indptr) - 1
    nnz = int(indptr[-1])
    cuts = np.searchsorted(indptr, np.linspace(0, nnz, world + 1), side="left").astype(np.int64)
    cuts[0], cuts[-1] = 0, n
    return np.maximum.accumulate(np.minimum(cuts, n))


def row_block(indptr, indices, vals, lo: int, hi: int):
    """CSR rows [lo, hi) with global column ids."""
    a, b = int(indptr[lo]), int(indptr[hi])
    return (indptr[lo:hi + 1] - a).astype(np.int32), indices[a:b], vals[a:b]


def to_device_pairs(arr: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)
