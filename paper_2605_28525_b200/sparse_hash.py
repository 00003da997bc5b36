"""Hash-based sparse grid construction on the GPU (reference:
/root/reference/pkg/src/sparsempm/sparse_hash.py).

Same table semantics as the reference: power-of-two capacity, home slot
mix64(key) & (H-1), linear probing, CAS slot claim, ranks from an atomic
counter, overflow when probing exhausts the table, and the rebuild-at-2x
policy when the table overflows or ends up past half load
(sparse_hash.py:225-264).  ``deterministic=True`` reproduces the serial
build's first-encounter ranks exactly (a per-slot minimum encounter position
plus a GPU radix sort), so ``active_blocks`` equals the reference's array for
array.
"""

import numpy as np

from . import _lib
from .errors import ConfigError, KeyRangeError
from .grid_index import ActiveIndexMap, mix64, pack_key, pack_keys


def initial_slot(key, table_size):
    """Home slot of a key (sparse_hash.py:31-40)."""
    table_size = int(table_size)
    if table_size < 1 or table_size & (table_size - 1):
        raise ValueError(f"table size must be a power of two, got {table_size}")
    return mix64(key) & (table_size - 1)


class BlockHashTable:
    """Open-addressing block table on the device (sparse_hash.py:109-167)."""

    def __init__(self, capacity):
        capacity = int(capacity)
        if capacity < 1 or capacity & (capacity - 1):
            raise ValueError(f"table capacity must be a power of two, got {capacity}")
        self._t = _lib.DeviceHashTable(capacity, capacity)

    @property
    def capacity(self):
        return self._t.n_slots

    @property
    def count(self):
        return self._t.count()

    @property
    def overflowed(self):
        c = self._t.counters.cpu().numpy()
        return bool(c[1])

    @property
    def keys(self):
        return self._t.keys.cpu().numpy().view(np.uint64)

    @property
    def vals(self):
        v = self._t.vals.cpu().numpy().view(np.uint32).astype(np.int64)
        v[v == _lib.EMPTY_VAL] = -1
        return v

    def insert_many(self, packed):
        """Concurrent insert of packed keys (_insert_many, sparse_hash.py:101-106):
        returns (ranks int64, fresh bool); rank -1 on overflow."""
        torch = _lib.torch_cuda()
        packed = _lib.to_dev(np.asarray(packed, dtype=np.uint64).view(np.int64), np.int64)
        n = packed.shape[0]
        ranks = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        fresh = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().smpm_hash_insert_many(self._t.dref, _lib.ptr(packed), n, _lib.ptr(ranks),
                                                     _lib.ptr(fresh), _lib.stream_ptr()), "insert")
        r = ranks[:n].cpu().numpy().view(np.uint32).astype(np.int64)
        r[r == _lib.EMPTY_VAL] = -1
        return r, fresh[:n].cpu().numpy().astype(bool)

    def insert(self, block):
        """Insert a block; returns (rank, newly_inserted) (sparse_hash.py:140-149)."""
        r, f = self.insert_many(np.array([pack_key(block)], dtype=np.uint64))
        return int(r[0]), bool(f[0])

    def lookup(self, block):
        """Rank of a block, or -1 when absent (sparse_hash.py:151-154)."""
        return ActiveIndexMap(self._t, 0).block_index(block)

    def active_blocks(self):
        """(count, 3) block coordinates ordered by rank."""
        return self._t.active_blocks().cpu().numpy().astype(np.int64).reshape(-1, 3)


def _next_pow2(n):
    p = 1
    while p < n:
        p *= 2
    return p


def build_hash_sparse_grid(positions, h, block_size=4, initial_capacity=None, deterministic=False,
                           max_rebuilds=48, rank_order=None):
    """Insert every stencil block of every particle (sparse_hash.py:225-264).

    ``rank_order``: None keeps the concurrent assignment order; "encounter"
    (the default when ``deterministic``) reproduces the serial build's
    first-encounter ranks; "key" gives the scan backend's row-major order.
    """
    if int(block_size) != 4:
        raise ConfigError(f"the GPU grid uses 4x4x4 blocks (one u64 node mask per block), got {block_size}")
    xp = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    if xp.shape[0] == 0:
        raise ValueError("cannot build a grid from an empty particle set")
    if not np.all(np.isfinite(xp)):
        raise ValueError("particle positions must be finite")
    if rank_order is None and deterministic:
        rank_order = "encounter"
    if initial_capacity is None:
        capacity = _next_pow2(max(64, xp.shape[0] // 4))
    else:
        capacity = int(initial_capacity)
        if capacity < 1 or capacity & (capacity - 1):
            raise ValueError(f"table capacity must be a power of two, got {capacity}")
    torch = _lib.torch_cuda()
    x = _lib.to_dev(xp, np.float64)
    inv_h = 1.0 / float(h)
    for _ in range(max_rebuilds):
        t = _lib.DeviceHashTable(capacity, capacity)
        err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        first = None
        if rank_order == "encounter":
            first = torch.full((capacity,), -1, dtype=torch.int64, device="cuda")
        _lib.check(_lib.load().smpm_insert_particle_blocks(t.dref, _lib.ptr(x), xp.shape[0], inv_h,
                                                           _lib.ptr(first), _lib.ptr(err), _lib.stream_ptr()),
                   "insert particle blocks")
        code, _p = _lib.err_code(np.uint64(err.cpu().numpy()[0]))
        if code:
            raise KeyRangeError("particle stencil block outside packable coordinate range")
        c = t.counters.cpu().numpy().view(np.uint32)
        if not c[1] and int(c[0]) <= capacity // 2:
            if rank_order == "encounter":
                t.canonicalize(1, first)
            elif rank_order == "key":
                t.canonicalize(0)
            return ActiveIndexMap(t, int(c[0]))
        capacity *= 2
    raise RuntimeError("hash table rebuild limit reached")


__all__ = ["BlockHashTable", "build_hash_sparse_grid", "initial_slot", "pack_keys"]
