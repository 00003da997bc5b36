"""ctypes binding of libsmpm.so (the C ABI in include/smpm.h).

The library is the only compute path: every public function of this package
that does physics or grid construction ends in one of these calls.  There is
no CPU fallback -- a missing library or a machine without CUDA raises.
PyTorch is used only for device memory and the current stream.
"""

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import ConfigError, InactiveNodeError, KeyRangeError, SimulationError

HERE = Path(__file__).resolve().parent
# SMPM_LIB selects an in-tree build variant (tools/build_variant.sh) for A/B timing
LIB_PATH = HERE / os.environ.get("SMPM_LIB", "libsmpm.so")

OK = 0
ERR_NONFINITE_X = 1
ERR_DEGENERATE_F = 2
ERR_DT_BOUND = 3
ERR_KEY_RANGE = 4
ERR_INACTIVE = 5
ERR_CAPACITY = 6
ERR_CONFIG = 20
RETRY = 41
ERR_CUDA = 30
ERR_ARG = 31
ERR_STATE = 32

EMPTY_VAL = 0xFFFFFFFF
ERR_CLEAR = (1 << 64) - 1

P = ctypes.c_void_p
D = ctypes.c_double
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U32 = ctypes.c_uint32
U64 = ctypes.c_uint64


class HashDesc(ctypes.Structure):
    _fields_ = [("keys", P), ("vals", P), ("n_slots", U64), ("counter", P), ("overflow", P),
                ("active_keys", P), ("slot_of_rank", P), ("cap_blocks", U32), ("pad", U32)]


class StencilParams(ctypes.Structure):
    _fields_ = [("h", D), ("inv_h", D), ("gravity", D * 3)]


class Boundary(ctypes.Structure):
    _fields_ = [("kind", I32), ("pad", I32), ("mu", D), ("point", D * 3), ("normal", D * 3)]


class GridParams(ctypes.Structure):
    _fields_ = [("h", D), ("dt", D), ("mass_floor", D), ("gravity", D * 3), ("n_bc", I32), ("pad", I32),
                ("bc", P), ("hf_data", P), ("hf_nx", I64), ("hf_ny", I64), ("hf_x0", D), ("hf_y0", D),
                ("hf_cell", D)]


class Material(ctypes.Structure):
    _fields_ = [("mu", D), ("lam", D), ("alpha", D), ("kind", I32), ("pad", I32)]


class SimConfigC(ctypes.Structure):
    _fields_ = [("h", D), ("gravity", D * 3), ("cfl", D), ("wave_speed", D), ("mass_floor", D),
                ("n_mat", I32), ("n_bc", I32), ("mats", P), ("bc", P), ("hf_data", P), ("hf_nx", I64),
                ("hf_ny", I64), ("hf_x0", D), ("hf_y0", D), ("hf_cell", D), ("particle_capacity", I64),
                ("block_capacity", I64), ("deterministic", I32), ("record_conservation", I32),
                ("device", I32), ("precise_grid", I32), ("stream", P)]


class StepStatsC(ctypes.Structure):
    _fields_ = [("step", I64), ("t", D), ("dt", D), ("n_active", I64), ("n_blocks", I64), ("vmax", D),
                ("mass_sum", D), ("mom_sum", D * 3), ("status", I32), ("pad", I32), ("err_particle", I64),
                ("ms_map", ctypes.c_float), ("ms_grid", ctypes.c_float), ("ms_fused", ctypes.c_float),
                ("ms_total", ctypes.c_float)]


_lib = None

_SIGS = {
    "smpm_last_error": (ctypes.c_char_p, []),
    "smpm_version": (ctypes.c_int, []),
    "smpm_hash_clear": (ctypes.c_int, [P, P]),
    "smpm_hash_insert_many": (ctypes.c_int, [P, P, I64, P, P, P]),
    "smpm_hash_lookup_many": (ctypes.c_int, [P, P, I64, P, P]),
    "smpm_insert_particle_blocks": (ctypes.c_int, [P, P, I64, D, P, P, P]),
    "smpm_hash_canonicalize": (ctypes.c_int, [P, ctypes.c_int, P, P, P]),
    "smpm_hash_active_blocks": (ctypes.c_int, [P, I64, P, P]),
    "smpm_bspline": (ctypes.c_int, [P, I64, D, P, P, P, P]),
    "smpm_p2g": (ctypes.c_int, [P, P, I64, P, P, P, P, P, P, P, P, P, P, P, P]),
    "smpm_grid_update": (ctypes.c_int, [P, I64, P, P, P, P, P]),
    "smpm_g2p": (ctypes.c_int, [P, P, D, I64, P, P, P, P, P, P, P]),
    "smpm_stress": (ctypes.c_int, [P, I32, I64, P, P, P, P, P, P]),
    "smpm_count_active_nodes": (ctypes.c_int, [P, P, I64, D, P, P, P, P]),
    "smpm_sim_create": (ctypes.c_int, [P, P]),
    "smpm_sim_destroy": (ctypes.c_int, [P]),
    "smpm_sim_set_particles": (ctypes.c_int, [P, I64, P, P, P, P, P, P, P]),
    "smpm_sim_get_particles": (ctypes.c_int, [P, P, P, P, P, P, P]),
    "smpm_sim_step": (ctypes.c_int, [P, D]),
    "smpm_sim_sync": (ctypes.c_int, [P, P]),
    "smpm_sim_run": (ctypes.c_int, [P, I64, D, P, P]),
    "smpm_sim_query_grid": (ctypes.c_int, [P, P, P, P, P]),
    "smpm_sim_num_particles": (I64, [P]),
    "smpm_sim_vmax": (D, [P]),
    "smpm_sim_launch_count": (ctypes.c_int, [P, P]),
    "smpm_sim_grid_size": (ctypes.c_int, [P, P]),
    "smpm_sim_retain_fields": (ctypes.c_int, [P, ctypes.c_int]),
    "smpm_sim_snapshot_xv": (ctypes.c_int, [P, P]),
    "smpm_sim_last_grid_size": (ctypes.c_int, [P, P]),
    "smpm_sim_last_grid": (ctypes.c_int, [P, P, P, P, P]),
    "smpm_sim_set_slab": (ctypes.c_int, [P, I32, I32, I64, I64]),
    "smpm_sim_set_dense_domain": (ctypes.c_int, [P, P, P]),
    "smpm_sim_set_external_bounds": (ctypes.c_int, [P, ctypes.c_int]),
    "smpm_sim_prologue_needed": (ctypes.c_int, [P]),
    "smpm_sim_prologue_begin": (ctypes.c_int, [P, P]),
    "smpm_sim_prologue_finish": (ctypes.c_int, [P, P]),
    "smpm_sim_p2g_bounds": (ctypes.c_int, [P, ctypes.c_int, P]),
    "smpm_sim_exchange_record_bytes": (I64, [P]),
    "smpm_sim_debug_stats": (ctypes.c_int, [P, P]),
    "smpm_release_cached_memory": (ctypes.c_int, []),
    "smpm_sim_exchange_pack": (ctypes.c_int, [P, ctypes.c_int, P, I64, P]),
    "smpm_sim_exchange_unpack": (ctypes.c_int, [P, P, I64, ctypes.c_int]),
    "smpm_sim_migrants": (ctypes.c_int, [P, ctypes.c_int, P, I64, P]),
    "smpm_sim_accept": (ctypes.c_int, [P, P, I64]),
    "smpm_sim_get_local": (ctypes.c_int, [P, P, P, P, P]),
    "smpm_sim_num_stored": (I64, [P]),
    "smpm_sim_frame_bytes": (I64, [P, I64, I64]),
    "smpm_sim_frame_pack": (ctypes.c_int, [P, ctypes.c_int, P, I64, I64]),
    "smpm_sim_frame_unpack": (ctypes.c_int, [P, P, I64, I64, ctypes.c_int]),
    "smpm_sim_stats_vector": (ctypes.c_int, [P, P]),
    "smpm_sim_stats_vector_len": (ctypes.c_int, []),
    "smpm_sim_apply_global": (ctypes.c_int, [P, P, ctypes.c_int]),
    "smpm_sim_migrants_delivered": (ctypes.c_int, [P, ctypes.c_int]),
}


def load():
    """Load libsmpm.so (built in-tree by __graft_entry__.build()).  Raises
    if the extension is missing -- there is no fallback path."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"CUDA extension {LIB_PATH} is missing; run `python -c 'import "
                               "__graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def last_error():
    return load().smpm_last_error().decode(errors="replace")


def check(rc, what="libsmpm call"):
    """Map a status code onto the reference's exception classes."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}"
    if rc in (ERR_NONFINITE_X, ERR_DEGENERATE_F, ERR_DT_BOUND):
        raise SimulationError(msg)
    if rc == ERR_KEY_RANGE:
        raise KeyRangeError("particle stencil block outside packable coordinate range")
    if rc == ERR_INACTIVE:
        raise InactiveNodeError("a particle stencil node is outside the active grid; with the dense backend this means "
                                "a particle left the declared domain")
    if rc == ERR_CONFIG:
        raise ConfigError(msg)
    raise RuntimeError(f"{msg} (status {rc})")


def err_code(word):
    word = int(word)
    if word == ERR_CLEAR:
        return OK, -1
    return word >> 40, word & ((1 << 40) - 1)


# ------------------------------------------------------------ device memory

def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_28525_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch


def stream_ptr():
    torch = torch_cuda()
    return torch.cuda.current_stream().cuda_stream


def to_dev(a, dtype):
    torch = torch_cuda()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(arr).cuda()


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _next_pow2(n):
    p = 1
    while p < n:
        p *= 2
    return p


class DeviceHashTable:
    """Device storage of one open-addressing block table (u64 keys, u32
    ranks) plus rank->key / rank->slot compaction arrays."""

    def __init__(self, n_slots, cap_blocks=None):
        torch = torch_cuda()
        n_slots = int(n_slots)
        if n_slots < 1 or n_slots & (n_slots - 1):
            raise ValueError(f"table capacity must be a power of two, got {n_slots}")
        self.n_slots = n_slots
        self.cap_blocks = int(cap_blocks if cap_blocks is not None else n_slots)
        self.keys = torch.empty(n_slots, dtype=torch.int64, device="cuda")
        self.vals = torch.empty(n_slots, dtype=torch.int32, device="cuda")
        self.counters = torch.zeros(2, dtype=torch.int32, device="cuda")
        self.active_keys = torch.empty(max(self.cap_blocks, 1), dtype=torch.int64, device="cuda")
        self.slot_of_rank = torch.empty(max(self.cap_blocks, 1), dtype=torch.int32, device="cuda")
        self.desc = HashDesc(self.keys.data_ptr(), self.vals.data_ptr(), n_slots, self.counters.data_ptr(),
                             self.counters.data_ptr() + 4, self.active_keys.data_ptr(),
                             self.slot_of_rank.data_ptr(), self.cap_blocks, 0)
        self.clear()

    @property
    def dref(self):
        return ctypes.byref(self.desc)

    def clear(self):
        check(load().smpm_hash_clear(self.dref, stream_ptr()), "hash clear")

    def count(self):
        return int(self.counters[0].item())

    def overflowed(self):
        c = self.counters.cpu().numpy()
        return bool(c[1]) or int(np.uint32(c[0])) > self.cap_blocks

    def active_keys_host(self):
        n = min(self.count(), self.cap_blocks)
        return self.active_keys[:n].cpu().numpy().view(np.uint64)

    def active_blocks(self):
        torch = torch_cuda()
        n = min(self.count(), self.cap_blocks)
        out = torch.empty((max(n, 1), 3), dtype=torch.int32, device="cuda")
        check(load().smpm_hash_active_blocks(self.dref, n, ptr(out), stream_ptr()), "active blocks")
        return out[:n]

    def canonicalize(self, mode, first_pos=None):
        torch = torch_cuda()
        cap = max(self.cap_blocks, 1)
        scratch = torch.empty(40 * cap + 1024 * (cap // 4096 + 1) + 4096, dtype=torch.uint8, device="cuda")
        check(load().smpm_hash_canonicalize(self.dref, int(mode), ptr(first_pos), ptr(scratch), stream_ptr()),
              "canonicalize")


def stress_inplace(particles, materials):
    """GPU _stress_kernel (materials.py:169-238) on a host ParticleSet."""
    torch = torch_cuda()
    n = particles.x.shape[0]
    mats = material_array(materials)
    F = to_dev(particles.F, np.float64)
    sig = torch.empty((n, 3, 3), dtype=torch.float64, device="cuda")
    jac = torch.empty(n, dtype=torch.float64, device="cuda")
    mid = to_dev(particles.mat_id, np.int64)
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    check(load().smpm_stress(mats, len(materials), n, ptr(F), ptr(sig), ptr(jac), ptr(mid), ptr(err),
                             stream_ptr()), "stress")
    code, p = err_code(np.uint64(err.cpu().numpy()[0]))
    if code:
        from .materials import _degenerate_message

        raise SimulationError(_degenerate_message(particles, p))
    particles.F[...] = F.cpu().numpy().reshape(particles.F.shape)
    particles.sigma[...] = sig.cpu().numpy().reshape(particles.sigma.shape)
    particles.jac[...] = jac.cpu().numpy()


def material_array(materials):
    arr = (Material * max(len(materials), 1))()
    for i, m in enumerate(materials):
        arr[i].mu = m.lame_mu
        arr[i].lam = m.lame_lambda
        arr[i].alpha = m.dp_alpha
        arr[i].kind = m.kind_id
    return arr
