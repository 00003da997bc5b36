"""Active-node indexing over 4x4x4 grid blocks (reference:
/root/reference/pkg/src/sparsempm/grid_index.py).

The key packing and mixing constants are identical to the reference
(grid_index.py:14-38, 41-121) so keys, hash slots and ranks are
interchangeable.  ``ActiveIndexMap`` here is backed by a device hash table;
its host views (``active_blocks``, ``keys``, ``vals``) are materialised on
demand for inspection and parity checks.
"""

import numpy as np

from . import _lib
from .errors import InactiveNodeError, KeyRangeError

KEY_BITS = 21
KEY_BIAS = 1 << 20
COORD_MIN = -(1 << 20)
COORD_MAX = (1 << 20) - 1
EMPTY_KEY = (1 << 64) - 1
MODE_FLAT = 0
MODE_HASH = 1
BLOCK_SIZE = 4

_MASK64 = (1 << 64) - 1
_MIX_MUL1 = 0xBF58476D1CE4E5B9
_MIX_MUL2 = 0x94D049BB133111EB


def pack_key(block, bits=KEY_BITS, bias=KEY_BIAS):
    """Pack a block triple into one non-negative key (grid_index.py:41-59)."""
    lo = -bias
    hi = (1 << bits) - bias
    packed = 0
    for c in block:
        c = int(c)
        if not lo <= c < hi:
            raise KeyRangeError(f"block coordinate {c} outside packable range [{lo}, {hi - 1}]")
        packed = (packed << bits) | (c + bias)
    return packed


def unpack_key(key, bits=KEY_BITS, bias=KEY_BIAS):
    """Invert pack_key (grid_index.py:62-68)."""
    key = int(key)
    mask = (1 << bits) - 1
    return ((key >> (2 * bits)) & mask) - bias, ((key >> bits) & mask) - bias, (key & mask) - bias


def mix64(key):
    """SplitMix64 finaliser used to spread keys over slots (grid_index.py:71-80)."""
    z = int(key) & _MASK64
    z = ((z ^ (z >> 30)) * _MIX_MUL1) & _MASK64
    z = ((z ^ (z >> 27)) * _MIX_MUL2) & _MASK64
    return z ^ (z >> 31)


def block_of(node, block_size=4):
    """Block containing a node, floor division (grid_index.py:83-87)."""
    i, j, k = (int(c) for c in node)
    return (i // block_size, j // block_size, k // block_size)


def local_offset(node, block_size=4):
    """Row-major offset of a node within its block (grid_index.py:90-97)."""
    i, j, k = (int(c) for c in node)
    b = block_size
    return ((i - b * (i // b)) * b + (j - b * (j // b))) * b + (k - b * (k // b))


def pack_keys(blocks):
    """Vectorised pack of an (n,3) int array (no range check)."""
    b = np.asarray(blocks, dtype=np.int64).reshape(-1, 3) + KEY_BIAS
    b = b.astype(np.uint64)
    return (b[:, 0] << np.uint64(42)) | (b[:, 1] << np.uint64(21)) | b[:, 2]


def unpack_keys(keys):
    k = np.asarray(keys, dtype=np.uint64)
    m = np.uint64((1 << 21) - 1)
    out = np.empty((k.shape[0], 3), dtype=np.int64)
    out[:, 2] = (k & m).astype(np.int64) - KEY_BIAS
    out[:, 1] = ((k >> np.uint64(21)) & m).astype(np.int64) - KEY_BIAS
    out[:, 0] = ((k >> np.uint64(42)) & m).astype(np.int64) - KEY_BIAS
    return out


class ActiveIndexMap:
    """Compact node indexing over the active blocks of a device hash table
    (grid_index.py:179-248, hash mode).  Block rank r owns compact nodes
    r*64 .. r*64+63 in row-major local order."""

    def __init__(self, table, n_blocks=None):
        self.table = table
        self.block_size = BLOCK_SIZE
        self.mode = MODE_HASH
        self._n_blocks = table.count() if n_blocks is None else int(n_blocks)
        self._active = None

    @property
    def n_blocks(self):
        return self._n_blocks

    @property
    def n_nodes(self):
        return self._n_blocks * self.block_size ** 3

    @property
    def active_blocks(self):
        """(n_blocks, 3) int64 block coordinates in rank order."""
        if self._active is None:
            self._active = self.table.active_blocks().cpu().numpy().astype(np.int64).reshape(-1, 3)
        return self._active

    @property
    def keys(self):
        return self.table.keys.cpu().numpy().view(np.uint64)

    @property
    def vals(self):
        v = self.table.vals.cpu().numpy().view(np.uint32).astype(np.int64)
        v[v == _lib.EMPTY_VAL] = -1
        return v

    def block_index(self, block):
        """Rank of a block, or -1 when inactive."""
        return int(self.block_indices(np.asarray(block).reshape(1, 3))[0])

    def block_indices(self, blocks):
        torch = _lib.torch_cuda()
        packed = _lib.to_dev(pack_keys(blocks).view(np.int64), np.int64)
        out = torch.empty(packed.shape[0], dtype=torch.int32, device="cuda")
        _lib.check(_lib.load().smpm_hash_lookup_many(self.table.dref, _lib.ptr(packed), packed.shape[0],
                                                     _lib.ptr(out), _lib.stream_ptr()), "lookup")
        r = out.cpu().numpy().view(np.uint32).astype(np.int64)
        r[r == _lib.EMPTY_VAL] = -1
        return r

    def node_index(self, node):
        """Compact index of a node; raises InactiveNodeError on a miss."""
        b = block_of(node, self.block_size)
        rank = self.block_index(b)
        if rank < 0:
            raise InactiveNodeError(f"node {tuple(int(c) for c in node)} lies in inactive block {b}")
        return rank * self.block_size ** 3 + local_offset(node, self.block_size)

    def node_coords(self):
        """(n_nodes, 3) node coordinates in compact-index order (grid_index.py:229-237)."""
        b = self.block_size
        rng = np.arange(b, dtype=np.int64)
        li, lj, lk = np.meshgrid(rng, rng, rng, indexing="ij")
        local = np.stack([li.ravel(), lj.ravel(), lk.ravel()], axis=1)
        return (self.active_blocks[:, None, :] * b + local[None, :, :]).reshape(-1, 3)

    def kernel_args(self):
        """The C-ABI descriptor consumed by the transfer kernels."""
        return self.table.dref

    @classmethod
    def from_blocks(cls, active_blocks):
        """Device map whose rank r is ``active_blocks[r]`` -- any rank order,
        e.g. the reference's scan (row-major) or dense maps
        (grid_index.py:179-198, 256-277).  Concurrent insert, then the ranks
        are re-ordered by each key's position in the list."""
        torch = _lib.torch_cuda()
        blocks = np.asarray(active_blocks, dtype=np.int64).reshape(-1, 3)
        n = blocks.shape[0]
        if n and (blocks.min() < COORD_MIN or blocks.max() > COORD_MAX):
            raise KeyRangeError("block coordinate outside packable range")
        cap = 64
        while cap < 2 * max(n, 1):
            cap *= 2
        t = _lib.DeviceHashTable(cap, max(n, 1))
        if n:
            packed = _lib.to_dev(pack_keys(blocks).view(np.int64), np.int64)
            ranks = torch.empty(n, dtype=torch.int32, device="cuda")
            fresh = torch.empty(n, dtype=torch.uint8, device="cuda")
            _lib.check(_lib.load().smpm_hash_insert_many(t.dref, _lib.ptr(packed), n, _lib.ptr(ranks),
                                                         _lib.ptr(fresh), _lib.stream_ptr()), "insert")
            if int(fresh.sum().item()) != n:
                raise ValueError("active_blocks lists a block twice")
            # first_pos[slot of the key at list position i] = i: canonical
            # order 1 (by first encounter) is then the list order
            first = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
            slots = t.slot_of_rank[ranks.long()].long()
            first[slots] = torch.arange(n, dtype=torch.int64, device="cuda")
            t.canonicalize(1, first)
        return cls(t, n)


def as_index_map(index_map):
    """The device map for any of the reference's map forms: this package's
    ActiveIndexMap, an object with ``active_blocks`` in rank order (the
    reference's ActiveIndexMap of any backend), or the reference's flat
    ``kernel_args()`` tuple (grid_index.py:239-248)."""
    if isinstance(index_map, ActiveIndexMap):
        return index_map
    if isinstance(index_map, tuple) and len(index_map) == 11:
        mode, b0, b1, b2, s0, s1, s2, phi_flat, keys, vals, bs = index_map
        if int(bs) != BLOCK_SIZE:
            raise ValueError(f"the GPU grid uses {BLOCK_SIZE}x{BLOCK_SIZE}x{BLOCK_SIZE} blocks, got {int(bs)}")
        if int(mode) == MODE_FLAT:
            phi = np.asarray(phi_flat, dtype=np.int64)
            live = np.nonzero(phi >= 0)[0]
            blocks = np.stack(np.unravel_index(live, (int(s0), int(s1), int(s2))), axis=1) + np.array(
                [int(b0), int(b1), int(b2)], dtype=np.int64)
            order = np.argsort(phi[live], kind="stable")
            return ActiveIndexMap.from_blocks(blocks[order])
        k = np.asarray(keys, dtype=np.uint64)
        v = np.asarray(vals, dtype=np.int64)
        used = np.nonzero((k != np.uint64(EMPTY_KEY)) & (v >= 0))[0]
        order = np.argsort(v[used], kind="stable")
        return ActiveIndexMap.from_blocks(unpack_keys(k[used][order]))
    blocks = getattr(index_map, "active_blocks", None)
    if blocks is None:
        raise TypeError(f"not an index map: {type(index_map).__name__}")
    if int(getattr(index_map, "block_size", BLOCK_SIZE)) != BLOCK_SIZE:
        raise ValueError(f"the GPU grid uses {BLOCK_SIZE}x{BLOCK_SIZE}x{BLOCK_SIZE} blocks")
    return ActiveIndexMap.from_blocks(blocks)


def node_index(index_map, node):
    return index_map.node_index(node)
