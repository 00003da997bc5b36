/*
 * smpm_oracle.c -- CPU restatement of the reference sparse-MPM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker ("oracle") and
 * the CPU baseline arm of bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg and --impl reference) may load it.  The product
 * path (paper_2605_28525_b200/) never links or calls it.
 *
 * It restates, in plain C with fp64 arithmetic, the numba kernels of the
 * reference package `sparsempm` (paths relative to /root/reference/pkg/src/
 * sparsempm/).  Operation order follows the reference expression by
 * expression and the file is compiled with -ffp-contract=off (numba/LLVM do
 * not contract either), so results are bitwise equal to the reference on the
 * same inputs for the serial (deterministic) kernels.  Pinned against golden
 * vectors produced by the reference itself: tests/golden/ (see
 * tests/golden/make_golden.py).
 *
 * Parallel variants use OpenMP with atomic fp64 adds, like the reference's
 * prange kernels with _fetch_add_f64 (_atomics.py:53-69).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KEY_BIAS ((int64_t)1 << 20)                 /* grid_index.py:15 */
#define COORD_MIN (-((int64_t)1 << 20))             /* grid_index.py:16 */
#define COORD_MAX (((int64_t)1 << 20) - 1)          /* grid_index.py:17 */
#define EMPTY_KEY UINT64_MAX                        /* grid_index.py:20 */
#define MODE_FLAT 0
#define MODE_HASH 1
#define BC_PLANE 0
#define KIND_DP 1

/* ------------------------------------------------------------------ keys */

/* grid_index.py:100-105 (_pack_key) */
uint64_t or_pack_key(int64_t bi, int64_t bj, int64_t bk) {
  uint64_t u = (uint64_t)(bi + KEY_BIAS), v = (uint64_t)(bj + KEY_BIAS), w = (uint64_t)(bk + KEY_BIAS);
  return (u << 42) | (v << 21) | w;
}

/* grid_index.py:108-113 (_unpack_key) */
void or_unpack_key(uint64_t key, int64_t *out) {
  const uint64_t m = ((uint64_t)1 << 21) - 1;
  out[2] = (int64_t)(key & m) - KEY_BIAS;
  out[1] = (int64_t)((key >> 21) & m) - KEY_BIAS;
  out[0] = (int64_t)((key >> 42) & m) - KEY_BIAS;
}

/* grid_index.py:116-121 (_mix64, SplitMix64 finalizer) */
uint64_t or_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return q;
}

/* floor(x*inv_h - 0.5) in fp64, no contraction: solver.py:43-44,
 * sparse_hash.py:174-176. */
static inline int64_t base_node(double x, double inv_h) { return (int64_t)floor(x * inv_h - 0.5); }

/* ------------------------------------------------------------ hash table */

/* sparse_hash.py:43-73 (_insert_key).  Serial form: CAS/fetch-add degenerate
 * to plain stores; the parallel build below uses GCC atomics. */
int64_t or_hash_insert(uint64_t *keys, int64_t *vals, int64_t n_slots, int64_t *counter,
                       int64_t *overflow, uint64_t key, int32_t *fresh) {
  uint64_t mask = (uint64_t)n_slots - 1;
  uint64_t s = or_mix64(key) & mask;
  *fresh = 0;
  for (int64_t it = 0; it < n_slots; ++it) {
    uint64_t stored = __atomic_load_n(&keys[s], __ATOMIC_RELAXED);
    if (stored == key) {
      int64_t r = __atomic_load_n(&vals[s], __ATOMIC_RELAXED);
      while (r < 0) r = __atomic_fetch_add(&vals[s], 0, __ATOMIC_RELAXED);
      return r;
    }
    if (stored == EMPTY_KEY) {
      uint64_t expected = EMPTY_KEY;
      if (__atomic_compare_exchange_n(&keys[s], &expected, key, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
        int64_t rank = __atomic_fetch_add(counter, 1, __ATOMIC_RELAXED);
        __atomic_fetch_add(&vals[s], rank + 1, __ATOMIC_RELAXED);
        *fresh = 1;
        return rank;
      }
      if (expected == key) {
        int64_t r = __atomic_load_n(&vals[s], __ATOMIC_RELAXED);
        while (r < 0) r = __atomic_fetch_add(&vals[s], 0, __ATOMIC_RELAXED);
        return r;
      }
    }
    s = (s + 1) & mask;
  }
  *overflow = 1;
  return -1;
}

/* sparse_hash.py:81-93 (_lookup_key), grid_index.py:134-147 */
int64_t or_hash_lookup(const uint64_t *keys, const int64_t *vals, int64_t n_slots, uint64_t key) {
  uint64_t mask = (uint64_t)n_slots - 1;
  uint64_t s = or_mix64(key) & mask;
  for (int64_t it = 0; it < n_slots; ++it) {
    uint64_t stored = keys[s];
    if (stored == key) return vals[s];
    if (stored == EMPTY_KEY) return -1;
    s = (s + 1) & mask;
  }
  return -1;
}

/* sparse_hash.py:101-106 (_insert_many) */
void or_hash_insert_many(uint64_t *keys, int64_t *vals, int64_t n_slots, int64_t *counter,
                         int64_t *overflow, const uint64_t *packed, int64_t n, int64_t *ranks,
                         int32_t *fresh, int parallel) {
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t i = 0; i < n; ++i) ranks[i] = or_hash_insert(keys, vals, n_slots, counter, overflow, packed[i], &fresh[i]);
}

/* sparse_hash.py:170-215 (_insert_particle_blocks / _serial).  Returns the
 * key-range error flag (err[0]). */
int64_t or_insert_particle_blocks(const double *x, int64_t n, double inv_h, int64_t bsz, uint64_t *keys,
                                  int64_t *vals, int64_t n_slots, int64_t *counter, int64_t *overflow,
                                  int parallel) {
  int64_t err = 0;
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    int64_t b0 = base_node(x[3 * p], inv_h), b1 = base_node(x[3 * p + 1], inv_h), b2 = base_node(x[3 * p + 2], inv_h);
    int64_t ilo = floordiv(b0, bsz), ihi = floordiv(b0 + 2, bsz);
    int64_t jlo = floordiv(b1, bsz), jhi = floordiv(b1 + 2, bsz);
    int64_t klo = floordiv(b2, bsz), khi = floordiv(b2 + 2, bsz);
    if (ilo < COORD_MIN || ihi > COORD_MAX || jlo < COORD_MIN || jhi > COORD_MAX || klo < COORD_MIN ||
        khi > COORD_MAX) {
      __atomic_store_n(&err, 1, __ATOMIC_RELAXED);
      continue;
    }
    int32_t fresh;
    for (int64_t bi = ilo; bi <= ihi; ++bi)
      for (int64_t bj = jlo; bj <= jhi; ++bj)
        for (int64_t bk = klo; bk <= khi; ++bk)
          or_hash_insert(keys, vals, n_slots, counter, overflow, or_pack_key(bi, bj, bk), &fresh);
  }
  return err;
}

/* sparse_hash.py:156-167 (BlockHashTable.active_blocks) */
void or_hash_active_blocks(const uint64_t *keys, const int64_t *vals, int64_t n_slots, int64_t *blocks) {
  for (int64_t s = 0; s < n_slots; ++s) {
    if (keys[s] == EMPTY_KEY) continue;
    or_unpack_key(keys[s], &blocks[3 * vals[s]]);
  }
}

/* ------------------------------------------------------------ scan build */

/* sparse_scan.py:15-29 (_stencil_base_bounds, serial) -> lo[3], hi[3] */
void or_stencil_base_bounds(const double *x, int64_t n, double inv_h, int64_t *lo, int64_t *hi) {
  int64_t l[3] = {(int64_t)1 << 62, (int64_t)1 << 62, (int64_t)1 << 62};
  int64_t h[3] = {-((int64_t)1 << 62), -((int64_t)1 << 62), -((int64_t)1 << 62)};
  for (int64_t p = 0; p < n; ++p)
    for (int a = 0; a < 3; ++a) {
      int64_t b = base_node(x[3 * p + a], inv_h);
      if (b < l[a]) l[a] = b;
      if (b > h[a]) h[a] = b;
    }
  for (int a = 0; a < 3; ++a) {
    lo[a] = l[a];
    hi[a] = h[a] + 2;
  }
}

/* sparse_scan.py:58-80 (_mark_blocks) */
int64_t or_mark_blocks(const double *x, int64_t n, double inv_h, int64_t bsz, const int64_t *blo,
                       const int64_t *bs, uint8_t *mask, int parallel) {
  int64_t err = 0;
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    int64_t b0 = base_node(x[3 * p], inv_h), b1 = base_node(x[3 * p + 1], inv_h), b2 = base_node(x[3 * p + 2], inv_h);
    int64_t ilo = floordiv(b0, bsz), ihi = floordiv(b0 + 2, bsz);
    int64_t jlo = floordiv(b1, bsz), jhi = floordiv(b1 + 2, bsz);
    int64_t klo = floordiv(b2, bsz), khi = floordiv(b2 + 2, bsz);
    if (ilo < blo[0] || jlo < blo[1] || klo < blo[2] || ihi >= blo[0] + bs[0] || jhi >= blo[1] + bs[1] ||
        khi >= blo[2] + bs[2]) {
      __atomic_store_n(&err, 1, __ATOMIC_RELAXED);
      continue;
    }
    for (int64_t bi = ilo; bi <= ihi; ++bi)
      for (int64_t bj = jlo; bj <= jhi; ++bj)
        for (int64_t bk = klo; bk <= khi; ++bk)
          mask[((bi - blo[0]) * bs[1] + (bj - blo[1])) * bs[2] + (bk - blo[2])] = 1;
  }
  return err;
}

/* sparse_scan.py:99-142 (three-phase parallel exclusive scan).  The result
 * is independent of the segment count, so a serial scan is exact. */
int64_t or_exclusive_scan(const int64_t *values, int64_t n, int64_t *out) {
  int64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    out[i] = acc;
    acc += values[i];
  }
  return acc;
}

/* solver.py:735-747 (_mark_nodes) */
void or_mark_nodes(const double *x, int64_t n, double inv_h, const int64_t *lo, int64_t s1, int64_t s2,
                   uint8_t *mask, int parallel) {
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    int64_t b0 = base_node(x[3 * p], inv_h), b1 = base_node(x[3 * p + 1], inv_h), b2 = base_node(x[3 * p + 2], inv_h);
    for (int oi = 0; oi < 3; ++oi)
      for (int oj = 0; oj < 3; ++oj)
        for (int ok = 0; ok < 3; ++ok)
          mask[((b0 + oi - lo[0]) * s1 + (b1 + oj - lo[1])) * s2 + (b2 + ok - lo[2])] = 1;
  }
}

/* ----------------------------------------------------- compact indexing */

typedef struct {
  int64_t mode;
  int64_t bmin[3];
  int64_t bshape[3];
  const int64_t *phi_flat;
  const uint64_t *keys;
  const int64_t *vals;
  int64_t n_slots;
  int64_t bsz;
} or_map;

/* grid_index.py:124-156 (_flat_block_lookup, _block_rank) */
static inline int64_t block_rank(const or_map *m, int64_t bi, int64_t bj, int64_t bk) {
  if (m->mode == MODE_FLAT) {
    int64_t ri = bi - m->bmin[0], rj = bj - m->bmin[1], rk = bk - m->bmin[2];
    if (ri < 0 || rj < 0 || rk < 0 || ri >= m->bshape[0] || rj >= m->bshape[1] || rk >= m->bshape[2]) return -1;
    return m->phi_flat[(ri * m->bshape[1] + rj) * m->bshape[2] + rk];
  }
  return or_hash_lookup(m->keys, m->vals, m->n_slots, or_pack_key(bi, bj, bk));
}

/* grid_index.py:159-172 (_node_to_compact) */
int64_t or_node_to_compact(const or_map *m, int64_t i, int64_t j, int64_t k) {
  int64_t b = m->bsz;
  int64_t bi = floordiv(i, b), bj = floordiv(j, b), bk = floordiv(k, b);
  int64_t r = block_rank(m, bi, bj, bk);
  if (r < 0) return -1;
  return r * b * b * b + ((i - b * bi) * b + (j - b * bj)) * b + (k - b * bk);
}

/* ------------------------------------------------------------- stencil */

/* solver.py:35-52 (_stencil) */
static inline void stencil(const double *xrow, double inv_h, int64_t *base, double w[3][3], double g[3][3]) {
  for (int a = 0; a < 3; ++a) {
    double u = xrow[a] * inv_h;
    int64_t b = (int64_t)floor(u - 0.5);
    double d = u - (double)b;
    double t0 = 1.5 - d, t1 = d - 1.0, t2 = d - 0.5;
    w[a][0] = 0.5 * (t0 * t0);
    w[a][1] = 0.75 - (t1 * t1);
    w[a][2] = 0.5 * (t2 * t2);
    g[a][0] = d - 1.5;
    g[a][1] = -2.0 * (d - 1.0);
    g[a][2] = d - 0.5;
    base[a] = b;
  }
}

/* solver.py:80-92 (bspline_weights; g returned per unit x/h, caller divides) */
void or_stencil(const double *xrow, double inv_h, int64_t *base, double *w, double *g) {
  stencil(xrow, inv_h, base, (double(*)[3])w, (double(*)[3])g);
}

static inline void add_f64(double *p, double v, int atomic) {
  if (atomic) {
#pragma omp atomic
    *p += v;
  } else {
    *p += v;
  }
}

/* solver.py:456-543 (_scatter_particle): fused mass/momentum/force.
 * mass/mom/force may individually be NULL (p2g-only or forces-only). */
static int scatter_particle(int64_t p, const double *xp, const double *vp, const double *cp, const double *mp,
                            const double *sigma, const double *jac, const double *v0p, double inv_h, double h,
                            double g0, double g1, double g2, const or_map *m, double *mass, double *mom,
                            double *force, int atomic) {
  int64_t base[3];
  double w[3][3], g[3][3];
  stencil(&xp[3 * p], inv_h, base, w, g);
  int64_t bsz = m->bsz;
  int64_t bi = floordiv(base[0], bsz), bj = floordiv(base[1], bsz), bk = floordiv(base[2], bsz);
  int64_t ranks[8];
  for (int s = 0; s < 8; ++s) ranks[s] = block_rank(m, bi + (s >> 2), bj + ((s >> 1) & 1), bk + (s & 1));
  int64_t li0 = base[0] - bi * bsz, lj0 = base[1] - bj * bsz, lk0 = base[2] - bk * bsz;
  int64_t bcube = bsz * bsz * bsz;
  double mpart = mp[p];
  double vol = v0p ? v0p[p] * jac[p] : 0.0;
  double x0 = xp[3 * p], x1 = xp[3 * p + 1], x2 = xp[3 * p + 2];
  const double *c = cp ? &cp[9 * p] : NULL;
  const double *sg = sigma ? &sigma[9 * p] : NULL;
  int err = 0;
  for (int oi = 0; oi < 3; ++oi) {
    double dx0 = (double)(base[0] + oi) * h - x0;
    int64_t ii = li0 + oi;
    int hi_i = ii >= bsz;
    int64_t li = hi_i ? ii - bsz : ii;
    int si = hi_i ? 4 : 0;
    for (int oj = 0; oj < 3; ++oj) {
      double dx1 = (double)(base[1] + oj) * h - x1;
      int64_t jj = lj0 + oj;
      int hi_j = jj >= bsz;
      int64_t lj = hi_j ? jj - bsz : jj;
      int sij = si + (hi_j ? 2 : 0);
      int64_t lij = (li * bsz + lj) * bsz;
      for (int ok = 0; ok < 3; ++ok) {
        int64_t kk = lk0 + ok;
        int hi_k = kk >= bsz;
        int64_t lk = hi_k ? kk - bsz : kk;
        int64_t rank = hi_k ? ranks[sij + 1] : ranks[sij];
        if (rank < 0) {
          err = 1;
          continue;
        }
        int64_t idx = rank * bcube + lij + lk;
        double dx2 = (double)(base[2] + ok) * h - x2;
        double wijk = w[0][oi] * w[1][oj] * w[2][ok];
        double wm = wijk * mpart;
        if (mass) {
          double pv0 = vp[3 * p], pv1 = vp[3 * p + 1], pv2 = vp[3 * p + 2];
          double mv0 = mpart * (pv0 + c[0] * dx0 + c[1] * dx1 + c[2] * dx2);
          double mv1 = mpart * (pv1 + c[3] * dx0 + c[4] * dx1 + c[5] * dx2);
          double mv2 = mpart * (pv2 + c[6] * dx0 + c[7] * dx1 + c[8] * dx2);
          add_f64(&mass[idx], wm, atomic);
          add_f64(&mom[3 * idx], wijk * mv0, atomic);
          add_f64(&mom[3 * idx + 1], wijk * mv1, atomic);
          add_f64(&mom[3 * idx + 2], wijk * mv2, atomic);
        }
        if (force) {
          double gx = g[0][oi] * w[1][oj] * w[2][ok] * inv_h;
          double gy = w[0][oi] * g[1][oj] * w[2][ok] * inv_h;
          double gz = w[0][oi] * w[1][oj] * g[2][ok] * inv_h;
          double fx = (-vol * (sg[0] * gx + sg[1] * gy + sg[2] * gz) + wm * g0);
          double fy = (-vol * (sg[3] * gx + sg[4] * gy + sg[5] * gz) + wm * g1);
          double fz = (-vol * (sg[6] * gx + sg[7] * gy + sg[8] * gz) + wm * g2);
          add_f64(&force[3 * idx], fx, atomic);
          add_f64(&force[3 * idx + 1], fy, atomic);
          add_f64(&force[3 * idx + 2], fz, atomic);
        }
      }
    }
  }
  return err;
}

/* solver.py:546-575 (_scatter_par / _scatter_ser), also p2g (:309-374,
 * mass/mom only) and grid_forces (:377-453, force only) through NULLs.
 * The unfused serial kernels accumulate in particle order exactly like the
 * fused serial scatter (solver.py:565-566), so one routine serves all. */
int64_t or_scatter(const double *xp, const double *vp, const double *cp, const double *mp, const double *sigma,
                   const double *jac, const double *v0p, int64_t n, double inv_h, double h, double g0, double g1,
                   double g2, const or_map *m, double *mass, double *mom, double *force, int parallel) {
  int64_t err = 0;
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    if (scatter_particle(p, xp, vp, cp, mp, sigma, jac, v0p, inv_h, h, g0, g1, g2, m, mass, mom, force, parallel))
      __atomic_store_n(&err, 1, __ATOMIC_RELAXED);
  }
  return err;
}

/* ---------------------------------------------------------- grid update */

/* solver.py:241-274 (_hf_sample) */
static inline void hf_sample(const double *data, int64_t nx, int64_t ny, double x0, double y0, double cell,
                             double x, double y, double *z, double *dzdx, double *dzdy) {
  double fx = (x - x0) / cell, fy = (y - y0) / cell;
  int64_t i0 = (int64_t)floor(fx), j0 = (int64_t)floor(fy);
  if (i0 < 0) i0 = 0;
  if (i0 > nx - 2) i0 = nx - 2;
  if (j0 < 0) j0 = 0;
  if (j0 > ny - 2) j0 = ny - 2;
  double tx = fx - (double)i0, ty = fy - (double)j0;
  if (tx < 0.0) tx = 0.0;
  if (tx > 1.0) tx = 1.0;
  if (ty < 0.0) ty = 0.0;
  if (ty > 1.0) ty = 1.0;
  double z00 = data[i0 * ny + j0], z10 = data[(i0 + 1) * ny + j0];
  double z01 = data[i0 * ny + j0 + 1], z11 = data[(i0 + 1) * ny + j0 + 1];
  *z = (z00 * (1.0 - tx) * (1.0 - ty) + z10 * tx * (1.0 - ty) + z01 * (1.0 - tx) * ty + z11 * tx * ty);
  *dzdx = ((z10 - z00) * (1.0 - ty) + (z11 - z01) * ty) / cell;
  *dzdy = ((z01 - z00) * (1.0 - tx) + (z11 - z10) * tx) / cell;
}

void or_hf_sample(const double *data, int64_t nx, int64_t ny, double x0, double y0, double cell, double x,
                  double y, double *out3) {
  hf_sample(data, nx, ny, x0, y0, cell, x, y, &out3[0], &out3[1], &out3[2]);
}

/* solver.py:277-291 (_coulomb_project) */
static inline void coulomb(double *v0, double *v1, double *v2, double n0, double n1, double n2, double mu) {
  double vn = *v0 * n0 + *v1 * n1 + *v2 * n2;
  if (vn >= 0.0) return;
  double t0 = *v0 - vn * n0, t1 = *v1 - vn * n1, t2 = *v2 - vn * n2;
  double tnorm = sqrt(t0 * t0 + t1 * t1 + t2 * t2);
  if (tnorm <= 0.0) {
    *v0 = *v1 = *v2 = 0.0;
    return;
  }
  double scale = 1.0 + mu * vn / tnorm;
  if (scale < 0.0) scale = 0.0;
  *v0 = scale * t0;
  *v1 = scale * t1;
  *v2 = scale * t2;
}

void or_coulomb_project(double *v3, const double *n3, double mu) { coulomb(&v3[0], &v3[1], &v3[2], n3[0], n3[1], n3[2], mu); }

/* solver.py:578-625 (_grid_update) */
void or_grid_update(double *mass, double *vel, const double *force, int64_t n_nodes, const int64_t *active_blocks,
                    int64_t bsz, double h, double dt, double mass_floor, const int64_t *bc_kind,
                    const double *bc_point, const double *bc_normal, const double *bc_mu, int64_t n_bc,
                    const double *hf_data, int64_t hf_nx, int64_t hf_ny, double hf_x0, double hf_y0,
                    double hf_cell, int parallel) {
  int64_t b3 = bsz * bsz * bsz;
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t c = 0; c < n_nodes; ++c) {
    double m = mass[c];
    if (m <= mass_floor) {
      vel[3 * c] = vel[3 * c + 1] = vel[3 * c + 2] = 0.0;
      continue;
    }
    double inv_m = 1.0 / m;
    double v0 = (vel[3 * c] + dt * force[3 * c]) * inv_m;
    double v1 = (vel[3 * c + 1] + dt * force[3 * c + 1]) * inv_m;
    double v2 = (vel[3 * c + 2] + dt * force[3 * c + 2]) * inv_m;
    int64_t r = c / b3, l = c - r * b3;
    int64_t li = l / (bsz * bsz), rem = l - li * bsz * bsz;
    int64_t lj = rem / bsz, lk = rem - lj * bsz;
    double x0 = (double)(active_blocks[3 * r] * bsz + li) * h;
    double x1 = (double)(active_blocks[3 * r + 1] * bsz + lj) * h;
    double x2 = (double)(active_blocks[3 * r + 2] * bsz + lk) * h;
    for (int64_t b = 0; b < n_bc; ++b) {
      if (bc_kind[b] == BC_PLANE) {
        double n0 = bc_normal[3 * b], n1 = bc_normal[3 * b + 1], n2 = bc_normal[3 * b + 2];
        double sdist = ((x0 - bc_point[3 * b]) * n0 + (x1 - bc_point[3 * b + 1]) * n1 + (x2 - bc_point[3 * b + 2]) * n2);
        if (sdist <= 0.0) coulomb(&v0, &v1, &v2, n0, n1, n2, bc_mu[b]);
      } else {
        double zs, zx, zy;
        hf_sample(hf_data, hf_nx, hf_ny, hf_x0, hf_y0, hf_cell, x0, x1, &zs, &zx, &zy);
        if (x2 - zs <= 0.0) {
          double inv_len = 1.0 / sqrt(zx * zx + zy * zy + 1.0);
          coulomb(&v0, &v1, &v2, -zx * inv_len, -zy * inv_len, inv_len, bc_mu[b]);
        }
      }
    }
    vel[3 * c] = v0;
    vel[3 * c + 1] = v1;
    vel[3 * c + 2] = v2;
  }
}

/* ------------------------------------------------------------------ G2P */

/* solver.py:628-732 (_g2p) */
int64_t or_g2p(double *xp, double *vp, double *cp, double *fdef, const double *vel, int64_t n, double inv_h,
               double h, double dt, const or_map *m, int parallel) {
  double d_inv = 4.0 * inv_h * inv_h;
  int64_t bsz = m->bsz, bcube = bsz * bsz * bsz;
  int64_t errflag = 0;
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    int64_t base[3];
    double w[3][3], g[3][3];
    stencil(&xp[3 * p], inv_h, base, w, g);
    int64_t bi = floordiv(base[0], bsz), bj = floordiv(base[1], bsz), bk = floordiv(base[2], bsz);
    int64_t ranks[8];
    for (int s = 0; s < 8; ++s) ranks[s] = block_rank(m, bi + (s >> 2), bj + ((s >> 1) & 1), bk + (s & 1));
    int64_t li0 = base[0] - bi * bsz, lj0 = base[1] - bj * bsz, lk0 = base[2] - bk * bsz;
    double x0 = xp[3 * p], x1 = xp[3 * p + 1], x2 = xp[3 * p + 2];
    double v0 = 0, v1 = 0, v2 = 0;
    double b00 = 0, b01 = 0, b02 = 0, b10 = 0, b11 = 0, b12 = 0, b20 = 0, b21 = 0, b22 = 0;
    double a00 = 0, a01 = 0, a02 = 0, a10 = 0, a11 = 0, a12 = 0, a20 = 0, a21 = 0, a22 = 0;
    for (int oi = 0; oi < 3; ++oi) {
      double dx0 = (double)(base[0] + oi) * h - x0;
      int64_t ii = li0 + oi;
      int hi_i = ii >= bsz;
      int64_t li = hi_i ? ii - bsz : ii;
      int si = hi_i ? 4 : 0;
      for (int oj = 0; oj < 3; ++oj) {
        double dx1 = (double)(base[1] + oj) * h - x1;
        int64_t jj = lj0 + oj;
        int hi_j = jj >= bsz;
        int64_t lj = hi_j ? jj - bsz : jj;
        int sij = si + (hi_j ? 2 : 0);
        int64_t lij = (li * bsz + lj) * bsz;
        for (int ok = 0; ok < 3; ++ok) {
          int64_t kk = lk0 + ok;
          int hi_k = kk >= bsz;
          int64_t lk = hi_k ? kk - bsz : kk;
          int64_t rank = hi_k ? ranks[sij + 1] : ranks[sij];
          if (rank < 0) {
            __atomic_store_n(&errflag, 1, __ATOMIC_RELAXED);
            continue;
          }
          int64_t idx = rank * bcube + lij + lk;
          double dx2 = (double)(base[2] + ok) * h - x2;
          double wijk = w[0][oi] * w[1][oj] * w[2][ok];
          double gx = g[0][oi] * w[1][oj] * w[2][ok] * inv_h;
          double gy = w[0][oi] * g[1][oj] * w[2][ok] * inv_h;
          double gz = w[0][oi] * w[1][oj] * g[2][ok] * inv_h;
          double gv0 = vel[3 * idx], gv1 = vel[3 * idx + 1], gv2 = vel[3 * idx + 2];
          v0 += wijk * gv0;
          v1 += wijk * gv1;
          v2 += wijk * gv2;
          b00 += wijk * gv0 * dx0;
          b01 += wijk * gv0 * dx1;
          b02 += wijk * gv0 * dx2;
          b10 += wijk * gv1 * dx0;
          b11 += wijk * gv1 * dx1;
          b12 += wijk * gv1 * dx2;
          b20 += wijk * gv2 * dx0;
          b21 += wijk * gv2 * dx1;
          b22 += wijk * gv2 * dx2;
          a00 += gv0 * gx;
          a01 += gv0 * gy;
          a02 += gv0 * gz;
          a10 += gv1 * gx;
          a11 += gv1 * gy;
          a12 += gv1 * gz;
          a20 += gv2 * gx;
          a21 += gv2 * gy;
          a22 += gv2 * gz;
        }
      }
    }
    vp[3 * p] = v0;
    vp[3 * p + 1] = v1;
    vp[3 * p + 2] = v2;
    double *c = &cp[9 * p];
    c[0] = b00 * d_inv;
    c[1] = b01 * d_inv;
    c[2] = b02 * d_inv;
    c[3] = b10 * d_inv;
    c[4] = b11 * d_inv;
    c[5] = b12 * d_inv;
    c[6] = b20 * d_inv;
    c[7] = b21 * d_inv;
    c[8] = b22 * d_inv;
    double *F = &fdef[9 * p];
    double f00 = F[0], f01 = F[1], f02 = F[2], f10 = F[3], f11 = F[4], f12 = F[5], f20 = F[6], f21 = F[7], f22 = F[8];
    F[0] = f00 + dt * (a00 * f00 + a01 * f10 + a02 * f20);
    F[1] = f01 + dt * (a00 * f01 + a01 * f11 + a02 * f21);
    F[2] = f02 + dt * (a00 * f02 + a01 * f12 + a02 * f22);
    F[3] = f10 + dt * (a10 * f00 + a11 * f10 + a12 * f20);
    F[4] = f11 + dt * (a10 * f01 + a11 * f11 + a12 * f21);
    F[5] = f12 + dt * (a10 * f02 + a11 * f12 + a12 * f22);
    F[6] = f20 + dt * (a20 * f00 + a21 * f10 + a22 * f20);
    F[7] = f21 + dt * (a20 * f01 + a21 * f11 + a22 * f21);
    F[8] = f22 + dt * (a20 * f02 + a21 * f12 + a22 * f22);
    xp[3 * p] += dt * v0;
    xp[3 * p + 1] += dt * v1;
    xp[3 * p + 2] += dt * v2;
  }
  return errflag;
}

/* ---------------------------------------------------------------- stress */

/* materials.py:81-85 (_det3) */
static inline double det3(const double *f) {
  return (f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) + f[2] * (f[3] * f[7] - f[4] * f[6]));
}

/* materials.py:88-122 (_jacobi_rotate) */
static inline void jacobi_rotate(double a[3][3], double q[3][3], int r0, int r1) {
  double apr = a[r0][r1];
  if (apr == 0.0) return;
  double app = a[r0][r0], arr = a[r1][r1];
  double theta = 0.5 * (arr - app) / apr;
  double t = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
  if (theta < 0.0) t = -t;
  double c = 1.0 / sqrt(1.0 + t * t);
  double s = t * c;
  double tau = s / (1.0 + c);
  a[r0][r0] = app - t * apr;
  a[r1][r1] = arr + t * apr;
  a[r0][r1] = 0.0;
  a[r1][r0] = 0.0;
  int o = 3 - r0 - r1;
  double aop = a[o][r0], aor = a[o][r1];
  a[o][r0] = aop - s * (aor + tau * aop);
  a[r0][o] = a[o][r0];
  a[o][r1] = aor + s * (aop - tau * aor);
  a[r1][o] = a[o][r1];
  for (int i = 0; i < 3; ++i) {
    double qip = q[i][r0], qir = q[i][r1];
    q[i][r0] = c * qip - s * qir;
    q[i][r1] = s * qip + c * qir;
  }
}

/* materials.py:125-144 (_sym_eigh3) */
static inline void sym_eigh3(double a[3][3], double q[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) q[i][j] = (i == j) ? 1.0 : 0.0;
  for (int it = 0; it < 16; ++it) {
    double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]) + off;
    if (off <= 1e-16 * scale) break;
    jacobi_rotate(a, q, 0, 1);
    jacobi_rotate(a, q, 0, 2);
    jacobi_rotate(a, q, 1, 2);
  }
}

/* materials.py:147-166 (_dp_return_map) */
static inline void dp_return_map(double e0, double e1, double e2, double alpha, double ratio, double *o) {
  double tr = e0 + e1 + e2;
  if (tr > 0.0) {
    o[0] = o[1] = o[2] = 0.0;
    return;
  }
  double m = tr / 3.0;
  double h0 = e0 - m, h1 = e1 - m, h2 = e2 - m;
  double en = sqrt(h0 * h0 + h1 * h1 + h2 * h2);
  double dg = en + alpha * ratio * tr;
  if (dg <= 0.0 || en <= 0.0) {
    o[0] = e0;
    o[1] = e1;
    o[2] = e2;
    return;
  }
  double c = dg / en;
  o[0] = e0 - c * h0;
  o[1] = e1 - c * h1;
  o[2] = e2 - c * h2;
}

void or_dp_return_map(const double *e, double alpha, double ratio, double *out) { dp_return_map(e[0], e[1], e[2], alpha, ratio, out); }

void or_sym_eigh3(double *a9, double *q9) { sym_eigh3((double(*)[3])a9, (double(*)[3])q9); }

/* materials.py:169-238 (_stress_kernel).  err[0] flag, err[1] particle. */
void or_stress(double *fdef, double *sigma, double *jac, const int64_t *mat_id, int64_t n, const double *mu_arr,
               const double *lam_arr, const double *alpha_arr, const int64_t *kind_arr, int64_t *err, int parallel) {
#pragma omp parallel for schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    double *F = &fdef[9 * p];
    double detf = det3(F);
    if (!(detf > 0.0) || !isfinite(detf)) {
      __atomic_store_n(&err[0], 1, __ATOMIC_RELAXED);
      __atomic_store_n(&err[1], p, __ATOMIC_RELAXED);
      continue;
    }
    double a[3][3], v[3][3], u[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        double cij = (F[i] * F[j] + F[3 + i] * F[3 + j] + F[6 + i] * F[6 + j]);
        a[i][j] = cij;
        a[j][i] = cij;
      }
    sym_eigh3(a, v);
    if (a[0][0] <= 0.0 || a[1][1] <= 0.0 || a[2][2] <= 0.0) {
      __atomic_store_n(&err[0], 1, __ATOMIC_RELAXED);
      __atomic_store_n(&err[1], p, __ATOMIC_RELAXED);
      continue;
    }
    double s0 = sqrt(a[0][0]), s1 = sqrt(a[1][1]), s2 = sqrt(a[2][2]);
    for (int i = 0; i < 3; ++i) {
      u[i][0] = (F[3 * i] * v[0][0] + F[3 * i + 1] * v[1][0] + F[3 * i + 2] * v[2][0]) / s0;
      u[i][1] = (F[3 * i] * v[0][1] + F[3 * i + 1] * v[1][1] + F[3 * i + 2] * v[2][1]) / s1;
      u[i][2] = (F[3 * i] * v[0][2] + F[3 * i + 1] * v[1][2] + F[3 * i + 2] * v[2][2]) / s2;
    }
    double e0 = log(s0), e1 = log(s1), e2 = log(s2);
    int64_t mid = mat_id[p];
    double mu = mu_arr[mid], lam = lam_arr[mid];
    if (kind_arr[mid] == KIND_DP) {
      double ratio = (3.0 * lam + 2.0 * mu) / (2.0 * mu);
      double pr[3];
      dp_return_map(e0, e1, e2, alpha_arr[mid], ratio, pr);
      if (pr[0] != e0 || pr[1] != e1 || pr[2] != e2) {
        e0 = pr[0];
        e1 = pr[1];
        e2 = pr[2];
        double q0 = exp(e0), q1 = exp(e1), q2 = exp(e2);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            F[3 * i + j] = (u[i][0] * q0 * v[j][0] + u[i][1] * q1 * v[j][1] + u[i][2] * q2 * v[j][2]);
      }
    }
    double trace = e0 + e1 + e2;
    double t0 = 2.0 * mu * e0 + lam * trace;
    double t1 = 2.0 * mu * e1 + lam * trace;
    double t2 = 2.0 * mu * e2 + lam * trace;
    double jp = exp(trace);
    jac[p] = jp;
    double inv_j = 1.0 / jp;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        sigma[9 * p + 3 * i + j] = inv_j * (t0 * u[i][0] * u[j][0] + t1 * u[i][1] * u[j][1] + t2 * u[i][2] * u[j][2]);
  }
}

/* solver.py:984-987 (dt_bound numerator input): max |v_p| */
double or_vmax(const double *vp, int64_t n, int parallel) {
  double vm = 0.0;
#pragma omp parallel for reduction(max : vm) schedule(static) if (parallel)
  for (int64_t p = 0; p < n; ++p) {
    double s = vp[3 * p] * vp[3 * p] + vp[3 * p + 1] * vp[3 * p + 1] + vp[3 * p + 2] * vp[3 * p + 2];
    if (s > vm) vm = s;
  }
  return sqrt(vm);
}

void or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
