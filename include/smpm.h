/*
 * smpm.h -- C ABI of libsmpm.so, the sm_100a sparse-MPM hot path.
 *
 * Drop-in boundary for the reference's hash-backend time step
 * (/root/reference/pkg/src/sparsempm/, cited file:line below).  Plain C types
 * only: device pointers are `void*`/typed pointers obtained from any CUDA
 * allocator (the Python host uses torch), streams are `void*` (cudaStream_t).
 * Every function returns an int status (SMPM_OK or a code below) and never
 * throws.  Host-pointer arguments are marked "host".
 */
#ifndef SMPM_H
#define SMPM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; map 1:1 onto the reference's exception classes
 * (errors.py:4-21). */
enum {
  SMPM_OK = 0,
  SMPM_ERR_NONFINITE_X = 1,   /* SimulationError (solver.py:1005-1006) */
  SMPM_ERR_DEGENERATE_F = 2,  /* SimulationError (solver.py:1013-1020) */
  SMPM_ERR_DT_BOUND = 3,      /* SimulationError (solver.py:1027-1030) */
  SMPM_ERR_KEY_RANGE = 4,     /* KeyRangeError (sparse_hash.py:255-258) */
  SMPM_ERR_INACTIVE = 5,      /* InactiveNodeError (solver.py:1053-1058) */
  SMPM_ERR_CAPACITY = 6,      /* internal capacity overflow (handled by growth) */
  SMPM_ERR_CONFIG = 20,       /* ConfigError (solver.py:776-810) */
  SMPM_ERR_CUDA = 30,         /* CUDA runtime failure (message: smpm_last_error) */
  SMPM_ERR_ARG = 31,          /* invalid argument */
  SMPM_ERR_STATE = 32,        /* the requested data is not available in the current state */
  SMPM_NEED_BOUNDS = 40,      /* internal: prologue measured, waiting for the caller's bounds */
  SMPM_RETRY = 41,            /* prologue capacity grew: call smpm_sim_prologue_begin again */
  SMPM_NEED_PROLOGUE = 42     /* external-bounds mode: run the coordinated prologue first */
};

const char* smpm_last_error(void);
/* Device memory of destroyed simulations is kept in a process-wide cache and
 * reused by later simulations with the same buffer sizes (bounded to a quarter
 * of the device memory, dropped automatically when one of this library's
 * allocations fails).  This returns the cached memory to the driver; call it
 * before large allocations by other libraries in the same process. */
int smpm_release_cached_memory(void);
int smpm_version(void);

/* ------------------------------------------------------------------ hash
 * Replaces BlockHashTable / _insert_key / _lookup_key / _insert_many
 * (sparse_hash.py:43-167) and _insert_particle_blocks
 * (sparse_hash.py:170-215).  keys: u64[n_slots] (EMPTY = all ones),
 * vals: u32[n_slots] (EMPTY = 0xffffffff), n_slots a power of two.
 * active_keys/slot_of_rank: [cap_blocks] rank -> key / slot. */
typedef struct {
  uint64_t* keys;
  uint32_t* vals;
  uint64_t n_slots;
  uint32_t* counter;
  uint32_t* overflow;
  uint64_t* active_keys;
  uint32_t* slot_of_rank;
  uint32_t cap_blocks;
  uint32_t pad;
} smpm_hash_desc;

int smpm_hash_clear(const smpm_hash_desc* h, void* stream);
/* _insert_many (sparse_hash.py:101-106): ranks u32 out, fresh u8 out */
int smpm_hash_insert_many(const smpm_hash_desc* h, const uint64_t* packed, int64_t n, uint32_t* ranks,
                          uint8_t* fresh, void* stream);
/* _lookup_key (sparse_hash.py:81-93); 0xffffffff for absent */
int smpm_hash_lookup_many(const smpm_hash_desc* h, const uint64_t* packed, int64_t n, uint32_t* ranks,
                          void* stream);
/* _insert_particle_blocks (sparse_hash.py:170-191).  x: f64 (n,3).
 * first_pos (optional, u64[n_slots], init all ones) receives the minimum
 * p*27+corner encounter position per slot, which orders ranks exactly like
 * the reference's serial (deterministic) build.  err: u64 error word. */
int smpm_insert_particle_blocks(const smpm_hash_desc* h, const double* x, int64_t n, double inv_h,
                                uint64_t* first_pos, unsigned long long* err, void* stream);
/* Reorders ranks: mode 0 = by key (== scan backend order,
 * sparse_scan.py:145-164), mode 1 = by first_pos (== serial hash build
 * order).  Rewrites vals, active_keys and slot_of_rank.  n_blocks is read
 * from h->counter.  scratch: >= 40 * cap_blocks bytes (device). */
int smpm_hash_canonicalize(const smpm_hash_desc* h, int mode, const uint64_t* first_pos, void* scratch,
                           void* stream);
/* active_blocks() (sparse_hash.py:156-167): int32 (n,3) in rank order */
int smpm_hash_active_blocks(const smpm_hash_desc* h, int64_t n_blocks, int32_t* blocks, void* stream);

/* ------------------------------------------------------- module transfers
 * Reference module API (solver.py:863-924, materials.py:250-267) over a hash
 * map; fields are fp32 on the compact node range rank*64 + local. */
typedef struct {
  double h, inv_h;
  double gravity[3];
} smpm_stencil_params;

/* bspline_weights (solver.py:80-92): base i64 (n,3), w/dw f64 (n,3,3) */
int smpm_bspline(const double* x, int64_t n, double h, int64_t* base, double* w, double* dw, void* stream);
/* p2g + grid_forces (solver.py:309-453).  Any of mass/mom/force may be NULL. */
int smpm_p2g(const smpm_hash_desc* h, const smpm_stencil_params* sp, int64_t n, const double* x, const double* v,
             const double* C, const double* m, const double* sigma, const double* jac, const double* V0,
             float* mass, float* mom, float* force, unsigned long long* err, void* stream);

typedef struct {
  int32_t kind; /* 0 plane, 1 heightfield */
  int32_t pad;
  double mu;
  double point[3];
  double normal[3];
} smpm_boundary;

typedef struct {
  double h, dt, mass_floor;
  double gravity[3]; /* added as m*g; zero when force already holds gravity */
  int32_t n_bc;
  int32_t pad;
  const smpm_boundary* bc;  /* host */
  const double* hf_data;    /* host [nx][ny] or NULL */
  int64_t hf_nx, hf_ny;
  double hf_x0, hf_y0, hf_cell;
} smpm_grid_params;

/* _grid_update (solver.py:578-625): vel holds momentum on entry, velocity on
 * exit.  active_blocks: int32 (n_blocks,3) device. */
int smpm_grid_update(const smpm_grid_params* gp, int64_t n_nodes, float* mass, float* vel, const float* force,
                     const int32_t* active_blocks, void* stream);
/* _g2p (solver.py:628-732): x,v,C,F f64 in/out */
int smpm_g2p(const smpm_hash_desc* h, const smpm_stencil_params* sp, double dt, int64_t n, double* x, double* v,
             double* C, double* F, const float* vel, unsigned long long* err, void* stream);

typedef struct {
  double mu, lam, alpha;
  int32_t kind; /* 0 elastic, 1 drucker_prager (materials.py:17-20) */
  int32_t pad;
} smpm_material;

/* _stress_kernel (materials.py:169-238): F in/out, sigma/jac out */
int smpm_stress(const smpm_material* mats /*host*/, int32_t n_mat, int64_t n, double* F, double* sigma, double* jac,
                const int64_t* mat_id, unsigned long long* err, void* stream);
/* count_active_nodes (solver.py:749-757): scratch hash given by h */
int smpm_count_active_nodes(const smpm_hash_desc* h, const double* x, int64_t n, double inv_h, uint64_t* nodemask,
                            unsigned long long* err, uint64_t* count_out /*host*/, void* stream);

/* ------------------------------------------------------------ simulation
 * Simulation.step with backend="hash" (solver.py:1001-1093) as one fused
 * device pipeline.  The context owns the particle state (double-buffered,
 * block-binned) and the sparse grid.  set/get take reference-layout f64
 * arrays (host or device pointers). */
typedef struct smpm_sim smpm_sim;

typedef struct {
  double h;
  double gravity[3];
  double cfl;
  double wave_speed;  /* max over materials (solver.py:951) */
  double mass_floor;  /* MASS_FLOOR_SCALE * max m (solver.py:952) */
  int32_t n_mat;
  int32_t n_bc;
  const smpm_material* mats; /* host */
  const smpm_boundary* bc;   /* host */
  const double* hf_data;     /* host [nx][ny] or NULL */
  int64_t hf_nx, hf_ny;
  double hf_x0, hf_y0, hf_cell;
  int64_t particle_capacity;
  int64_t block_capacity;    /* 0: automatic */
  int32_t deterministic;     /* ranks by key (scan order) */
  int32_t record_conservation;
  int32_t device;
  int32_t precise_grid;      /* non-deterministic mode: 1 = per-cell register P2G
                                into a split fixed-point arena with per-item
                                scales (fp32-grade grid sums on every node); 0 =
                                per-particle int32 fixed point, one global scale
                                (faster, coarser on light nodes); DESIGN.md s.4 */
  void* stream;              /* cudaStream_t or NULL (own stream) */
} smpm_sim_config;

typedef struct {
  int64_t step;
  double t, dt;
  int64_t n_active;     /* bit-exact |union of particle stencils| */
  int64_t n_blocks;     /* allocated = n_blocks * 64 */
  double vmax;          /* max |v| after the step (next dt bound) */
  double mass_sum, mom_sum[3];
  int32_t status;       /* SMPM_OK or error code */
  int32_t pad;
  int64_t err_particle; /* particle index for errors */
  float ms_map, ms_grid, ms_fused, ms_total; /* device phase times */
} smpm_step_stats;

int smpm_sim_create(const smpm_sim_config* cfg, smpm_sim** out);
int smpm_sim_destroy(smpm_sim* s);
/* ParticleSet fields (solver.py:95-132): x,v (n,3) f64; C,F (n,3,3) f64;
 * m,V0 (n) f64; mat_id (n) i64. */
int smpm_sim_set_particles(smpm_sim* s, int64_t n, const double* x, const double* v, const double* C,
                           const double* F, const double* m, const double* V0, const int64_t* mat_id);
/* Any output may be NULL; sigma/jac are evaluated from the current F. */
int smpm_sim_get_particles(smpm_sim* s, double* x, double* v, double* C, double* F, double* sigma, double* jac);
/* One step; dt <= 0 selects the CFL bound.  Asynchronous. */
int smpm_sim_step(smpm_sim* s, double dt);
/* Waits for the last step and returns its stats (status != 0 on error). */
int smpm_sim_sync(smpm_sim* s, smpm_step_stats* out);
/* n steps (dt <= 0: the CFL bound each step) with one host synchronisation
 * per batch of up to 1024 steps: the reference's loop of Simulation.step
 * calls (solver.py:1001-1093; bench.py:216-226).  The between-step checks
 * (dt bound, errors, grid capacity) run on the device; a failing step halts
 * its batch and is handled as after smpm_sim_step + smpm_sim_sync.  out[i]
 * (may be NULL) receives step i's stats, *n_done the steps completed; returns
 * the first error. */
int smpm_sim_run(smpm_sim* s, int64_t n, double dt, smpm_step_stats* out, int64_t* n_done);
/* Active blocks (int32 (n,3), rank order) and nodal fields after the
 * step's P2G: mass, momentum, force (f32, gravity included). Host pointers,
 * sized by smpm_sim_sync's n_blocks. */
int smpm_sim_query_grid(smpm_sim* s, int32_t* blocks, float* mass, float* mom, float* force);
/* Block count of the grid smpm_sim_query_grid returns (runs a pending
 * prologue). */
int smpm_sim_grid_size(smpm_sim* s, int64_t* n_blocks);
/* Grid of the last completed step: Simulation.last_map / last_fields
 * (solver.py:1087-1090).  Blocks in rank order, node mass, grid velocity after
 * the update and boundary projection, and (after smpm_sim_retain_fields(s, 1),
 * which makes every later step keep them) the nodal force incl. gravity.
 * SMPM_ERR_STATE when no step completed since the last (re)binning. */
int smpm_sim_retain_fields(smpm_sim* s, int on);
/* Frame output without stalling the stream (scenarios.py:483-513 frames):
 * x then v (fp64, pid order, 6 n doubles) into a device buffer, enqueued on
 * the simulation's stream after the last step; no host sync.  The caller
 * copies it out on a side stream (paper_2605_28525_b200/frames.py). */
int smpm_sim_snapshot_xv(smpm_sim* s, double* out /*device*/);
int smpm_sim_last_grid_size(smpm_sim* s, int64_t* n_blocks);
int smpm_sim_last_grid(smpm_sim* s, int32_t* blocks, float* mass, float* vel, float* force);
int64_t smpm_sim_num_particles(const smpm_sim* s);
double smpm_sim_vmax(smpm_sim* s);
int smpm_sim_launch_count(const smpm_sim* s, int64_t* kernels_per_step);

/* Dense allocation mode, the comparison baseline of bench.compare
 * (replaces build_dense_grid, grid_index.py:256-277, for
 * SimConfig.backend == "dense"): every block of the inclusive block box
 * [bmin, bmax] is allocated each step (ranks in row-major order), so
 * n_allocated = n_dense and the grid update runs over the whole domain. */
int smpm_sim_set_dense_domain(smpm_sim* s, const int32_t* bmin, const int32_t* bmax);

/* Deterministic mode across ranks: every rank must scale its fixed-point
 * partial sums identically, so the prologue's bounds are agreed by the caller
 * (max over ranks) between the measure and scatter passes:
 *   smpm_sim_set_external_bounds(s, 1);
 *   if (smpm_sim_prologue_needed(s)) {   -- on every rank, together
 *     smpm_sim_prologue_begin(s, local);    allreduce(max) -> global;
 *     rc = smpm_sim_prologue_finish(s, global);  -- SMPM_RETRY: begin again
 *   }
 * and after each step the bounds the next launch scales with are replaced by
 * the max over ranks (smpm_sim_p2g_bounds get / set). */
int smpm_sim_set_external_bounds(smpm_sim* s, int on);
int smpm_sim_prologue_needed(smpm_sim* s);
int smpm_sim_prologue_begin(smpm_sim* s, float* local_bounds);
int smpm_sim_prologue_finish(smpm_sim* s, const float* global_bounds);
int smpm_sim_p2g_bounds(smpm_sim* s, int set, float* bounds);
/* Diagnostics: per table (n_blocks, n_binned, n_items, scale_ovf, overflow,
 * n_owned) x 2, then S, n_store, need_prologue, migrants_sent, and the bin
 * census of the stored particles (holes, in-flight migrants, overflowed,
 * unresolved, binned), then the work-item layout of the last scan and of the
 * next step (0 narrow, 1 wide), then the fused kernel of the last launch
 * (0 k_g2p2g_f32, 1 k_g2p2g_ws, 2 k_g2p2g int32 fixed point, 3 k_g2p2g
 * int64 deterministic): 24 int64. */
int smpm_sim_debug_stats(smpm_sim* s, int64_t* out);
/* Bytes per block record of smpm_sim_exchange_pack (2064 fp32, 4112 deterministic). */
int64_t smpm_sim_exchange_record_bytes(const smpm_sim* s);

/* ---------------------------------------------------- slab decomposition
 * Multi-GPU (the reference is single-process, PAPER.md:335-337
 * lists multi-GPU as future work).  A rank owns the particles whose base
 * block has block-x in [bx0, bx1).  After smpm_sim_step the caller (NCCL via
 * torch.distributed) moves:
 *   1. smpm_sim_exchange_pack(mode 0/1): partial node sums of blocks left /
 *      right of the slab -> owner, which smpm_sim_exchange_unpack(set=0)s them;
 *   2. smpm_sim_exchange_pack(mode 2): the owner's full sums of its layer
 *      bx == bx0 -> left neighbour, unpacked with set=1 (identical bits on
 *      both sides of the interface);
 *   3. smpm_sim_migrants(side, out): 128-byte records of particles that left the
 *      slab -> neighbour's smpm_sim_accept (appended and binned).
 * Block records are 2064 bytes (key, node mask, 64 x 8 floats). */
int smpm_sim_set_slab(smpm_sim* s, int32_t bx0, int32_t bx1, int64_t pid_base, int64_t migrant_capacity);
/* Device-resident exchange (one host sync per distributed step): fixed-
 * capacity frames whose counts travel in a 32-byte header on the device, so a
 * frame is sent whole without a size round trip.
 *   frame = [header][cap_parts x 128-B particle records][cap_blocks x record]
 * frame_pack: mode 0/1 = halo partial sums of blocks left / right of the slab
 *   plus the particles that departed to that side; mode 2 = the owner's
 *   first block layer (full sums) back to the left neighbour.  Async.
 * frame_unpack: add (set = 0) or overwrite (set = 1) the block sums, append
 *   and bin the arriving particles (device counter of storage slots).  Async.
 *   Frames that overflowed their capacity are reported, not applied.
 * stats_vector: this rank's step statistics into a device double[len]
 *   (vmax^2, n_active, n_owned, mass, momentum[3], P2G bounds[3], replay,
 *   error, storage, frame counts[3][2], frame overflow, inverse fixed-point
 *   scales[3], 0) for one all-gather;
 *   apply_global: the next launch's fixed-point bounds = max over the
 *   gathered rows (plus the precision check at the sync).  Async. */
int64_t smpm_sim_frame_bytes(const smpm_sim* s, int64_t cap_blocks, int64_t cap_parts);
int smpm_sim_frame_pack(smpm_sim* s, int mode, void* frame /*device*/, int64_t cap_blocks, int64_t cap_parts);
int smpm_sim_frame_unpack(smpm_sim* s, const void* frame /*device*/, int64_t cap_blocks, int64_t cap_parts, int set);
int smpm_sim_stats_vector(smpm_sim* s, double* out /*device*/);
int smpm_sim_stats_vector_len(void);
int smpm_sim_apply_global(smpm_sim* s, const double* rows /*device [world][len]*/, int world);
/* After the step's sync: the departed particles of the sides in side_mask
 * (bit 0 left, bit 1 right) reached their neighbour (frame not overflowed),
 * so their storage slots become holes; the others stay live for the replay. */
int smpm_sim_migrants_delivered(smpm_sim* s, int side_mask);
int smpm_sim_exchange_pack(smpm_sim* s, int mode, void* out /*device*/, int64_t cap_blocks, int64_t* n_out);
int smpm_sim_exchange_unpack(smpm_sim* s, const void* in /*device*/, int64_t n, int set);
/* count of departing particles (side 0 left, 1 right); copies their records
 * into out (device or host, >= cap records) when out != NULL */
int smpm_sim_migrants(smpm_sim* s, int side, void* out, int64_t cap, int64_t* n);
int smpm_sim_accept(smpm_sim* s, const void* recs /*device*/, int64_t n);
/* Live particles of this rank: global pid, x, v (host or device pointers
 * sized >= smpm_sim_num_stored). */
int smpm_sim_get_local(smpm_sim* s, int64_t* n_live, int64_t* pid, double* x, double* v);
int64_t smpm_sim_num_stored(const smpm_sim* s);

#ifdef __cplusplus
}
#endif
#endif
