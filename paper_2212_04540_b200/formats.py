"""On-disk formats on either side of the hot path:
the reference's dataset directory (TSV + vocabulary sidecars) and its
versioned binary checkpoint (``KGACTCK1``), restated so files written by one
side load on the other byte for byte.

* Dataset directory (data.py:1-12 file formats, :97-159 parsing, :413-489
  round trip): ``interactions.tsv`` (``user<TAB>item``), ``triples.tsv``
  (``head<TAB>relation<TAB>tail``), and ``{users,entities,relations,items}
  .vocab.tsv`` (``string<TAB>index``).  Without sidecars indices follow
  first-seen order with triples extending the item vocabulary; with them the
  sidecars pin the index assignment.  Splits come from ``split_interactions``
  (data.py:202-227: per-user 80/20 then 10 % of the pool to validation, numpy
  ``default_rng(seed)`` permutations in first-seen user order) and an optional
  k-core filter (data.py:185-199).
* Checkpoint (checkpoint.py:1-55): 8-byte magic ``KGACTCK1``, little-endian
  uint32 header length, UTF-8 JSON header with sorted keys (array names,
  shapes, numpy dtype strings, free-form ``meta``), then the arrays'
  little-endian payloads in header order.

Host-side numpy; not part of the timed path.
"""
import json
import os
import struct

import numpy as np
import torch

from .data import KgDataset

MAGIC = b"KGACTCK1"


class ParseError(ValueError):
    """A data file line does not match the documented schema (data.py:24)."""


class CheckpointError(ValueError):
    """checkpoint.py:19."""


# ---------------------------------------------------------------------------
# TSV parsing
# ---------------------------------------------------------------------------

def _intern(vocab: dict, key: str) -> int:
    idx = vocab.get(key)
    if idx is None:
        idx = vocab[key] = len(vocab)
    return idx


def _records(path, width, what):
    with open(path, encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.rstrip("\n")
            if not line:
                continue
            parts = line.split("\t")
            if len(parts) != width or not all(parts):
                raise ParseError(f"{path}:{lineno}: expected {what}, got {line!r}")
            yield lineno, parts


def load_interactions(path):
    """data.py:97-120: (pairs int32 (n, 2), user_vocab, item_vocab); ids in
    first-seen order, exact duplicate pairs dropped (first occurrence kept)."""
    users, items, pairs, seen = {}, {}, [], set()
    for _, (u, i) in _records(path, 2, "<user>\\t<item>"):
        key = (_intern(users, u), _intern(items, i))
        if key not in seen:
            seen.add(key)
            pairs.append(key)
    return np.array(pairs, dtype=np.int32).reshape(-1, 2), users, items


def load_triples(path, entity_vocab=None, relation_vocab=None, strict=False):
    """data.py:123-148: extends copies of the given vocabularies (pass the
    item vocabulary to align items with their entities); ``strict`` rejects
    relations missing from ``relation_vocab``."""
    ents = {} if entity_vocab is None else dict(entity_vocab)
    rels = {} if relation_vocab is None else dict(relation_vocab)
    out = []
    for lineno, (h, r, t) in _records(path, 3, "<head>\\t<relation>\\t<tail>"):
        hi = _intern(ents, h)
        if strict and r not in rels:
            raise ParseError(f"{path}:{lineno}: unknown relation {r!r}")
        out.append((hi, _intern(rels, r), _intern(ents, t)))
    return np.array(out, dtype=np.int32).reshape(-1, 3), ents, rels


def save_vocab(path, vocab: dict) -> None:
    """data.py:151-154: one ``key<TAB>index`` line per entry, by index."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{k}\t{v}\n" for k, v in sorted(vocab.items(), key=lambda kv: kv[1]))


def load_vocab(path) -> dict:
    """data.py:157-168."""
    vocab = {}
    with open(path, encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.rstrip("\n")
            if not line:
                continue
            parts = line.split("\t")
            if len(parts) != 2:
                raise ParseError(f"{path}:{lineno}: expected <string>\\t<index>")
            vocab[parts[0]] = int(parts[1])
    return vocab


# ---------------------------------------------------------------------------
# Preprocessing
# ---------------------------------------------------------------------------

def kcore_filter(pairs: np.ndarray, k: int) -> np.ndarray:
    """data.py:185-199: drop users/items of degree < k until nothing changes
    (vectorized; same fixpoint and surviving order)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    pairs = np.asarray(pairs)
    while len(pairs):
        du = np.bincount(pairs[:, 0])
        di = np.bincount(pairs[:, 1])
        keep = (du[pairs[:, 0]] >= k) & (di[pairs[:, 1]] >= k)
        if keep.all():
            break
        pairs = pairs[keep]
    return pairs.reshape(-1, 2)


def split_interactions(pairs: np.ndarray, seed: int, train_frac: float = 0.8,
                       val_frac: float = 0.1):
    """data.py:202-227: per user (first-seen order) a permutation from one
    ``default_rng(seed)``; floor(0.8 n) to the pool, the rest to test; then
    round-half-up 10 % of the pool (at most pool-1) to validation.  Users with
    fewer than three interactions stay entirely in train."""
    rng = np.random.default_rng(seed)
    pairs = np.asarray(pairs).reshape(-1, 2)
    if len(pairs) == 0:
        e = np.zeros((0, 2), dtype=np.int32)
        return e, e.copy(), e.copy()
    users = pairs[:, 0].astype(np.int64)
    # group each user's items in their original order, users in first-seen order
    _, first = np.unique(users, return_index=True)
    user_order = users[np.sort(first)]
    rank = np.empty(users.max() + 1, dtype=np.int64)
    rank[user_order] = np.arange(len(user_order))
    idx = np.argsort(rank[users], kind="stable")
    grouped = pairs[idx]
    bounds = np.concatenate([[0], np.cumsum(np.bincount(rank[users], minlength=len(user_order)))])
    train, val, test = [], [], []
    for g in range(len(user_order)):
        block = grouped[bounds[g]:bounds[g + 1]]
        n = len(block)
        if n < 3:
            train.append(block)
            continue
        perm = rng.permutation(n)
        n_pool = int(np.floor(train_frac * n))
        pool = block[perm[:n_pool]]
        test.append(block[perm[n_pool:]])
        n_val = min(int(val_frac * len(pool) + 0.5), len(pool) - 1)
        val.append(pool[:n_val])
        train.append(pool[n_val:])
    cat = lambda parts: (np.concatenate(parts).astype(np.int32).reshape(-1, 2) if parts
                         else np.zeros((0, 2), dtype=np.int32))
    return cat(train), cat(val), cat(test)


# ---------------------------------------------------------------------------
# Dataset directory round trip
# ---------------------------------------------------------------------------

def default_vocabs(ds: KgDataset):
    """The synthetic generator's names (data.py:399-404): u%04d, i%04d,
    a%04d, rel%d."""
    users = {f"u{u:04d}": u for u in range(ds.num_users)}
    ents = {f"i{i:04d}": i for i in range(ds.num_items)}
    ents.update({f"a{a:04d}": a for a in range(ds.num_items, ds.num_entities)})
    rels = {f"rel{r}": r for r in range(ds.num_relations)}
    return users, ents, rels


def save_dataset(ds: KgDataset, outdir: str) -> None:
    """data.py:413-436: interactions (all splits, sorted by (user, item)),
    triples in stored order, and the four vocabulary sidecars."""
    os.makedirs(outdir, exist_ok=True)
    uv, ev, rv = (ds.user_vocab, ds.entity_vocab, ds.relation_vocab) \
        if ds.user_vocab is not None else default_vocabs(ds)
    inv_u = np.empty(len(uv), dtype=object)
    inv_u[list(uv.values())] = list(uv.keys())
    inv_e = np.empty(len(ev), dtype=object)
    inv_e[list(ev.values())] = list(ev.keys())
    inv_r = np.empty(max(len(rv), 1), dtype=object)
    if rv:
        inv_r[list(rv.values())] = list(rv.keys())
    parts = [a for a in (ds.train, ds.val, ds.test) if len(a)]
    allp = np.concatenate(parts) if parts else np.zeros((0, 2), dtype=np.int32)
    order = np.lexsort((allp[:, 1], allp[:, 0])) if len(allp) else np.zeros(0, dtype=np.int64)
    with open(os.path.join(outdir, "interactions.tsv"), "w", encoding="utf-8") as fh:
        fh.writelines(f"{inv_u[u]}\t{inv_e[i]}\n" for u, i in allp[order].tolist())
    with open(os.path.join(outdir, "triples.tsv"), "w", encoding="utf-8") as fh:
        fh.writelines(f"{inv_e[h]}\t{inv_r[r]}\t{inv_e[t]}\n" for h, r, t in ds.triples.tolist())
    save_vocab(os.path.join(outdir, "users.vocab.tsv"), uv)
    save_vocab(os.path.join(outdir, "entities.vocab.tsv"), ev)
    save_vocab(os.path.join(outdir, "relations.vocab.tsv"), rv)
    save_vocab(os.path.join(outdir, "items.vocab.tsv"), {k: v for k, v in ev.items() if v < ds.num_items})


def load_dataset(datadir: str, seed: int, kcore: int = 0) -> KgDataset:
    """data.py:439-489: parse a dataset directory and split it with ``seed``."""
    ipath = os.path.join(datadir, "interactions.tsv")
    tpath = os.path.join(datadir, "triples.tsv")
    pairs, uvoc, ivoc = load_interactions(ipath)
    uv_path = os.path.join(datadir, "users.vocab.tsv")
    ev_path = os.path.join(datadir, "entities.vocab.tsv")
    rv_path = os.path.join(datadir, "relations.vocab.tsv")
    if os.path.exists(uv_path) and os.path.exists(ev_path):
        full_u, full_e = load_vocab(uv_path), load_vocab(ev_path)
        full_r = load_vocab(rv_path) if os.path.exists(rv_path) else None
        remap_u = np.array([full_u[k] for k in uvoc], dtype=np.int64)
        remap_i = np.array([full_e[k] for k in ivoc], dtype=np.int64)
        if len(pairs):
            pairs = np.stack([remap_u[pairs[:, 0]], remap_i[pairs[:, 1]]], axis=1)
        items_path = os.path.join(datadir, "items.vocab.tsv")
        num_items = (len(load_vocab(items_path)) if os.path.exists(items_path)
                     else int(remap_i.max(initial=-1) + 1))
        if os.path.exists(tpath):
            triples, ents, rels = load_triples(tpath, full_e, full_r, strict=full_r is not None)
        else:
            triples, ents, rels = np.zeros((0, 3), dtype=np.int32), full_e, full_r or {}
        users = full_u
    else:
        if os.path.exists(tpath):
            triples, ents, rels = load_triples(tpath, ivoc)
        else:
            triples, ents, rels = np.zeros((0, 3), dtype=np.int32), dict(ivoc), {}
        users = uvoc
        num_items = len(ivoc)
    if kcore > 0 and len(pairs):
        pairs = kcore_filter(pairs, kcore)
    train, val, test = split_interactions(np.asarray(pairs).astype(np.int32), seed)
    ds = KgDataset(len(users), num_items, len(ents), train, val, test,
                   np.asarray(triples, dtype=np.int32).reshape(-1, 3), max(len(rels), 1),
                   user_vocab=users, entity_vocab=ents, relation_vocab=rels)
    ds.validate()
    return ds


# ---------------------------------------------------------------------------
# Checkpoints
# ---------------------------------------------------------------------------

def save_checkpoint(path: str, params, meta: dict) -> None:
    """checkpoint.py:22-38.  ``params``: ModelParams (or a name -> tensor /
    array dict in the reference's order: E0, theta0, theta1, ...)."""
    items = list((params.as_dict() if hasattr(params, "as_dict") else params).items())
    arrays = [(k, v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v))
              for k, v in items]
    header = {"arrays": [{"name": k, "shape": list(a.shape), "dtype": a.dtype.str} for k, a in arrays],
              "meta": meta}
    blob = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<I", len(blob)))
        fh.write(blob)
        for _, a in arrays:
            fh.write(np.ascontiguousarray(a).astype(a.dtype.newbyteorder("<")).tobytes())


def load_checkpoint(path: str, device="cuda"):
    """checkpoint.py:41-55: (ModelParams on ``device``, meta)."""
    from .model import ModelParams
    with open(path, "rb") as fh:
        magic = fh.read(len(MAGIC))
        if magic != MAGIC:
            raise CheckpointError(f"{path}: not a checkpoint (bad magic {magic!r})")
        raw = fh.read(4)
        if len(raw) != 4:
            raise CheckpointError(f"{path}: truncated header")
        (hlen,) = struct.unpack("<I", raw)
        try:
            header = json.loads(fh.read(hlen).decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as exc:
            raise CheckpointError(f"{path}: corrupt header ({exc})") from None
        loaded = {}
        for spec in header["arrays"]:
            dt = np.dtype(spec["dtype"])
            count = int(np.prod(spec["shape"])) if spec["shape"] else 1
            buf = fh.read(count * dt.itemsize)
            if len(buf) != count * dt.itemsize:
                raise CheckpointError(f"{path}: truncated array {spec['name']}")
            a = np.frombuffer(buf, dtype=dt).reshape(spec["shape"]).astype(dt.newbyteorder("="))
            loaded[spec["name"]] = torch.from_numpy(a).to(device)
    return ModelParams.from_dict(loaded), header["meta"]
