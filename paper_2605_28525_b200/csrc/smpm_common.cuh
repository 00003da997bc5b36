// Shared device code for the sm_100a sparse-MPM hot path.
//
// Reference: /root/reference/pkg/src/sparsempm/ (cited as file:line).  This is
// a from-scratch GPU design, not a translation: fp64 only where parity needs it
// (block/base indexing, node positions, boundary predicates), fp32 elsewhere.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace smpm {

// grid_index.py:14-20
constexpr int64_t KEY_BIAS = int64_t(1) << 20;
constexpr int COORD_MIN = -(1 << 20);
constexpr int COORD_MAX = (1 << 20) - 1;
constexpr uint64_t EMPTY_KEY = ~uint64_t(0);
constexpr uint32_t EMPTY_VAL = 0xFFFFFFFFu;
constexpr int BSZ = 4;  // block_size (solver.py:771); fixed: one u64 node mask per block

// Error codes, ordered like the checks in Simulation.step (solver.py:1005-1085).
// The device error word is atomicMin((code << 40) | particle).
enum ErrCode : uint32_t {
  ERR_NONE = 0,
  ERR_NONFINITE_X = 1,   // SimulationError (solver.py:1005-1006)
  ERR_DEGENERATE_F = 2,  // SimulationError (solver.py:1013-1020)
  ERR_DT_BOUND = 3,      // SimulationError (solver.py:1027-1030)
  ERR_KEY_RANGE = 4,     // KeyRangeError (sparse_hash.py:255-258)
  ERR_INACTIVE = 5,      // InactiveNodeError (solver.py:1053-1058)
  ERR_CAPACITY = 6,      // internal: block capacity exceeded -> host grows + replays
};
constexpr uint64_t ERR_CLEAR = ~uint64_t(0);
__host__ __device__ inline uint64_t err_word(uint32_t code, uint64_t particle) {
  return (uint64_t(code) << 40) | (particle & ((uint64_t(1) << 40) - 1));
}

// ------------------------------------------------------------------ keys
// grid_index.py:100-105
__host__ __device__ inline uint64_t pack_key(int bi, int bj, int bk) {
  return (uint64_t(int64_t(bi) + KEY_BIAS) << 42) | (uint64_t(int64_t(bj) + KEY_BIAS) << 21) |
         uint64_t(int64_t(bk) + KEY_BIAS);
}
// grid_index.py:108-113
__host__ __device__ inline void unpack_key(uint64_t key, int& bi, int& bj, int& bk) {
  const uint64_t m = (uint64_t(1) << 21) - 1;
  bk = int(int64_t(key & m) - KEY_BIAS);
  bj = int(int64_t((key >> 21) & m) - KEY_BIAS);
  bi = int(int64_t((key >> 42) & m) - KEY_BIAS);
}
// grid_index.py:116-121 (SplitMix64 finaliser)
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------ hash table
// Open addressing with linear probing from mix64(key) & (H-1); the slot is
// claimed by CAS(EMPTY -> key) and the claimant takes rank = fetch_add(counter)
// and publishes it; a thread that finds the key already claimed waits for the
// rank (sparse_hash.py:43-73).  Ranks are u32.  The table additionally records
// rank -> key and rank -> slot so compaction and clearing are O(n_blocks).
struct HashView {
  uint64_t* keys;
  uint32_t* vals;
  uint32_t mask;           // n_slots - 1 (power of two)
  uint32_t cap_blocks;     // ranks >= cap_blocks are flagged as capacity overflow
  uint32_t* counter;       // number of ranks handed out
  uint32_t* overflow;      // probe exhaustion or capacity overflow
  uint64_t* active_keys;   // [cap_blocks] rank -> key
  uint32_t* slot_of_rank;  // [cap_blocks] rank -> slot
};

__device__ inline uint32_t ld_volatile_u32(const uint32_t* p) { return *(const volatile uint32_t*)p; }
__device__ inline uint64_t ld_volatile_u64(const uint64_t* p) { return *(const volatile uint64_t*)p; }

// Returns the rank, or EMPTY_VAL when the table overflowed.  *fresh reports a
// newly inserted key.
__device__ inline uint32_t hash_insert(const HashView& h, uint64_t key, bool* fresh = nullptr) {
  uint32_t s = uint32_t(mix64(key)) & h.mask;
  for (uint32_t it = 0; it <= h.mask; ++it) {
    uint64_t stored = ld_volatile_u64(&h.keys[s]);
    // the slot's rank in the same round trip: a key inserted earlier (the
    // common case: a block is touched by up to 27 items) returns at once
    const uint32_t rv = ld_volatile_u32(&h.vals[s]);
    if (stored == key && rv != EMPTY_VAL) {
      if (fresh) *fresh = false;
      return rv;
    }
    if (stored == EMPTY_KEY) {
      unsigned long long prev = atomicCAS((unsigned long long*)&h.keys[s], (unsigned long long)EMPTY_KEY,
                                          (unsigned long long)key);
      if (prev == EMPTY_KEY) {
        uint32_t rank = atomicAdd(h.counter, 1u);
        if (rank < h.cap_blocks) {
          h.active_keys[rank] = key;
          h.slot_of_rank[rank] = s;
        } else {
          atomicExch(h.overflow, 1u);
        }
        atomicExch(&h.vals[s], rank);
        if (fresh) *fresh = true;
        return rank;
      }
      stored = prev;
    }
    if (stored == key) {
      uint32_t r;
      while ((r = ld_volatile_u32(&h.vals[s])) == EMPTY_VAL) {
      }
      if (fresh) *fresh = false;
      return r;
    }
    s = (s + 1) & h.mask;
  }
  atomicExch(h.overflow, 1u);
  if (fresh) *fresh = false;
  return EMPTY_VAL;
}

// sparse_hash.py:81-93 / grid_index.py:134-147
__device__ inline uint32_t hash_lookup(const uint64_t* keys, const uint32_t* vals, uint32_t mask, uint64_t key) {
  uint32_t s = uint32_t(mix64(key)) & mask;
  for (uint32_t it = 0; it <= mask; ++it) {
    uint64_t stored = keys[s];
    if (stored == key) return vals[s];
    if (stored == EMPTY_KEY) return EMPTY_VAL;
    s = (s + 1) & mask;
  }
  return EMPTY_VAL;
}

// --------------------------------------------------------------- stencil
// Base node floor(x*inv_h - 0.5) in fp64 without contraction, from the same
// stored fp64 x and host inv_h = 1.0/h as the reference (solver.py:43-44,
// sparse_hash.py:174-176), so the active block/node sets are bit-exact.  The
// cell-relative offset d = u - base is then exact enough to carry in fp32.
__device__ inline bool axis_base(double x, double inv_h, int& base, float& d) {
  double u = __dmul_rn(x, inv_h);
  double fb = floor(__dadd_rn(u, -0.5));
  if (!(fabs(fb) < 4.0e6)) return false;  // also rejects NaN/inf
  base = int(fb);
  d = float(__dadd_rn(u, -fb));
  return true;
}

// block-span range check of sparse_hash.py:177-186 for one axis
__device__ inline bool axis_in_key_range(int base) {
  return (base >> 2) >= COORD_MIN && ((base + 2) >> 2) <= COORD_MAX;
}

// Quadratic B-spline weights and d/du weights per axis (solver.py:46-51).
__device__ inline void bspline(float d, float w[3], float g[3]) {
  float t0 = 1.5f - d, t1 = d - 1.0f, t2 = d - 0.5f;
  w[0] = 0.5f * t0 * t0;
  w[1] = 0.75f - t1 * t1;
  w[2] = 0.5f * t2 * t2;
  g[0] = d - 1.5f;
  g[1] = -2.0f * t1;
  g[2] = t2;
}

// ------------------------------------------------------- constitutive model
// Material table entry (materials.py:55-78 derived constants).
struct Material {
  float mu, lam, alpha, ratio;  // ratio = (3 lam + 2 mu) / (2 mu)
  int kind;                     // 0 elastic, 1 Drucker-Prager
  int pad[3];
};

__device__ inline void jacobi_rotate(float& app, float& arr, float& apr, float& aop, float& aor, float* q, int r0,
                                     int r1) {
  // materials.py:88-122 in fp32: annihilate a[r0][r1].  The angle only needs
  // to be approximately right (c and s are exactly normalised from t, so the
  // accumulated frame stays orthonormal); fast reciprocals are used.
  if (apr == 0.0f) return;
  const float theta = __fdividef(0.5f * (arr - app), apr);
  const float th2 = theta * theta;
  // t = sign(theta) / (|theta| + sqrt(1 + theta^2)); for huge |theta|, 1/(2 theta)
  const float q1 = 1.0f + th2;
  float t = th2 < 1e30f ? __fdividef(1.0f, fabsf(theta) + q1 * rsqrtf(q1)) : __fdividef(0.5f, fabsf(theta));
  if (theta < 0.0f) t = -t;
  const float c = rsqrtf(1.0f + t * t);
  const float s = t * c;
  const float tau = __fdividef(s, 1.0f + c);
  app = app - t * apr;
  arr = arr + t * apr;
  apr = 0.0f;
  float op = aop, orr = aor;
  aop = op - s * (orr + tau * op);
  aor = orr + s * (op - tau * orr);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float qip = q[3 * i + r0], qir = q[3 * i + r1];
    q[3 * i + r0] = c * qip - s * qir;
    q[3 * i + r1] = s * qip + c * qir;
  }
}

// log1p / expm1 for the small arguments of the constitutive update (strains,
// return-map increments): odd atanh series / Taylor polynomial, ~1 ulp for
// |x| <= 1/4, libm beyond.
__device__ __forceinline__ float log1p_small(float x) {
  if (fabsf(x) > 0.25f) return log1pf(x);
  const float z = x / (2.0f + x);  // log1p(x) = 2 atanh(z), |z| <= 1/7
  const float z2 = z * z;
  float p = fmaf(z2, 1.0f / 11.0f, 1.0f / 9.0f);
  p = fmaf(p, z2, 1.0f / 7.0f);
  p = fmaf(p, z2, 1.0f / 5.0f);
  p = fmaf(p, z2, 1.0f / 3.0f);
  return 2.0f * z * fmaf(p, z2, 1.0f);
}
__device__ __forceinline__ float expm1_small(float x) {
  if (fabsf(x) > 0.25f) return expm1f(x);
  float p = fmaf(x, 1.0f / 40320.0f, 1.0f / 5040.0f);
  p = fmaf(p, x, 1.0f / 720.0f);
  p = fmaf(p, x, 1.0f / 120.0f);
  p = fmaf(p, x, 1.0f / 24.0f);
  p = fmaf(p, x, 1.0f / 6.0f);
  p = fmaf(p, x, 0.5f);
  p = fmaf(p, x, 1.0f);
  return p * x;
}

// Hencky elasticity + cohesionless Drucker-Prager return map in principal
// space (materials.py:169-238), fp32, on H = F - I (row-major).  Carrying the
// displacement gradient instead of F keeps small strains exact: C - I =
// H + H^T + H^T H has no cancellation, eigen-strains come from log1p, and the
// return-mapped update H += (I + H) V diag(expm1(e' - e)) V^T never forms
// I + small.  Returns false on a degenerate F (det F <= 0 or non-finite).
// Outputs the Kirchhoff stress tau = J sigma (xx,yy,zz,xy,xz,yz) and J; when
// `project`, the return-mapped H is written back.
__device__ inline bool hencky_dp_eig(float H[9], const Material& mat, bool project, float tau[6], float& J) {
  // det(I + H) = 1 + tr H + (principal 2x2 minors of H) + det H
  const float trH = H[0] + H[4] + H[8];
  const float m2 = (H[0] * H[4] - H[1] * H[3]) + (H[0] * H[8] - H[2] * H[6]) + (H[4] * H[8] - H[5] * H[7]);
  const float dH = H[0] * (H[4] * H[8] - H[5] * H[7]) - H[1] * (H[3] * H[8] - H[5] * H[6]) +
                   H[2] * (H[3] * H[7] - H[4] * H[6]);
  const float det = 1.0f + (trH + (m2 + dH));
  if (!(det > 0.0f) || !isfinite(det)) return false;
  // C - I = H + H^T + H^T H  (materials.py:181-189 shifted by I)
  float a00 = 2.f * H[0] + (H[0] * H[0] + H[3] * H[3] + H[6] * H[6]);
  float a11 = 2.f * H[4] + (H[1] * H[1] + H[4] * H[4] + H[7] * H[7]);
  float a22 = 2.f * H[8] + (H[2] * H[2] + H[5] * H[5] + H[8] * H[8]);
  float a01 = (H[1] + H[3]) + (H[0] * H[1] + H[3] * H[4] + H[6] * H[7]);
  float a02 = (H[2] + H[6]) + (H[0] * H[2] + H[3] * H[5] + H[6] * H[8]);
  float a12 = (H[5] + H[7]) + (H[1] * H[2] + H[4] * H[5] + H[7] * H[8]);
  float V[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
  // cyclic Jacobi (materials.py:125-144); rotations are shift-invariant, the
  // stopping rule is relative to |C - I|
#pragma unroll 1
  for (int sweep = 0; sweep < 8; ++sweep) {
    float off = fabsf(a01) + fabsf(a02) + fabsf(a12);
    float scale = fabsf(a00) + fabsf(a11) + fabsf(a22) + off;
    if (off <= 1e-6f * scale) break;
    // threshold Jacobi: elements already below the per-element share of the
    // tolerance are not rotated
    const float thr = 3e-7f * scale;
    if (fabsf(a01) > thr) jacobi_rotate(a00, a11, a01, a02, a12, V, 0, 1);  // o = 2: a[2][0], a[2][1]
    if (fabsf(a02) > thr) jacobi_rotate(a00, a22, a02, a01, a12, V, 0, 2);  // o = 1: a[1][0], a[1][2]
    if (fabsf(a12) > thr) jacobi_rotate(a11, a22, a12, a01, a02, V, 1, 2);  // o = 0: a[0][1], a[0][2]
  }
  // eigenvalues of C are 1 + mu_k
  if (!(a00 > -1.0f) || !(a11 > -1.0f) || !(a22 > -1.0f)) return false;
  const float mu3[3] = {a00, a11, a22};
  float U[9], e[3], e0[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float inv_s = rsqrtf(1.0f + mu3[k]);
    // u_k = (I + H) v_k / s_k
#pragma unroll
    for (int i = 0; i < 3; ++i)
      U[3 * i + k] = (V[3 * i + k] + (H[3 * i] * V[k] + H[3 * i + 1] * V[3 + k] + H[3 * i + 2] * V[6 + k])) * inv_s;
    e[k] = 0.5f * log1p_small(mu3[k]);
    e0[k] = e[k];
  }
  if (mat.kind == 1) {
    // materials.py:147-166
    float tr = e[0] + e[1] + e[2];
    bool changed = false;
    if (tr > 0.0f) {
      changed = (e[0] != 0.f) || (e[1] != 0.f) || (e[2] != 0.f);
      e[0] = e[1] = e[2] = 0.0f;
    } else {
      float m = tr * (1.0f / 3.0f);
      float h0 = e[0] - m, h1 = e[1] - m, h2 = e[2] - m;
      float en = sqrtf(h0 * h0 + h1 * h1 + h2 * h2);
      float dg = en + mat.alpha * mat.ratio * tr;
      if (dg > 0.0f && en > 0.0f) {
        float c = dg / en;
        e[0] -= c * h0;
        e[1] -= c * h1;
        e[2] -= c * h2;
        changed = true;
      }
    }
    if (changed && project) {
      // F' = U diag(exp e') V^T = F V diag(exp(e' - e)) V^T
      //  => H' = H + (I + H) D,  D = V diag(expm1(e' - e)) V^T
      const float r0 = expm1_small(e[0] - e0[0]), r1 = expm1_small(e[1] - e0[1]), r2 = expm1_small(e[2] - e0[2]);
      float D[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          D[3 * i + j] = V[3 * i] * r0 * V[3 * j] + V[3 * i + 1] * r1 * V[3 * j + 1] + V[3 * i + 2] * r2 * V[3 * j + 2];
      float Hn[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          Hn[3 * i + j] = H[3 * i + j] + (D[3 * i + j] + (H[3 * i] * D[j] + H[3 * i + 1] * D[3 + j] + H[3 * i + 2] * D[6 + j]));
#pragma unroll
      for (int q = 0; q < 9; ++q) H[q] = Hn[q];
    }
  }
  float tr = e[0] + e[1] + e[2];
  float t0 = 2.0f * mat.mu * e[0] + mat.lam * tr;
  float t1 = 2.0f * mat.mu * e[1] + mat.lam * tr;
  float t2 = 2.0f * mat.mu * e[2] + mat.lam * tr;
  J = expf(tr);
  // tau = sum_k t_k u_k u_k^T  (materials.py:233-238 times J)
  tau[0] = t0 * U[0] * U[0] + t1 * U[1] * U[1] + t2 * U[2] * U[2];
  tau[1] = t0 * U[3] * U[3] + t1 * U[4] * U[4] + t2 * U[5] * U[5];
  tau[2] = t0 * U[6] * U[6] + t1 * U[7] * U[7] + t2 * U[8] * U[8];
  tau[3] = t0 * U[0] * U[3] + t1 * U[1] * U[4] + t2 * U[2] * U[5];
  tau[4] = t0 * U[0] * U[6] + t1 * U[1] * U[7] + t2 * U[2] * U[8];
  tau[5] = t0 * U[3] * U[6] + t1 * U[4] * U[7] + t2 * U[5] * U[8];
  return true;
}

// symmetric 3x3 stored (xx, yy, zz, xy, xz, yz); product of two commuting
// symmetric matrices (powers / polynomials of one matrix)
__device__ __forceinline__ void sym_mul(const float a[6], const float b[6], float c[6]) {
  c[0] = a[0] * b[0] + a[3] * b[3] + a[4] * b[4];
  c[1] = a[3] * b[3] + a[1] * b[1] + a[5] * b[5];
  c[2] = a[4] * b[4] + a[5] * b[5] + a[2] * b[2];
  c[3] = a[0] * b[3] + a[3] * b[1] + a[4] * b[5];
  c[4] = a[0] * b[4] + a[3] * b[5] + a[4] * b[2];
  c[5] = a[3] * b[4] + a[1] * b[5] + a[5] * b[2];
}

#ifndef SMPM_PADE
#define SMPM_PADE 1  // moderate-strain log by Pade approximants (0: the atanh series)
#endif
// inverse of a symmetric 3x3 (xx, yy, zz, xy, xz, yz)
__device__ __forceinline__ void sym_inv(const float d[6], float o[6]) {
  const float c00 = d[1] * d[2] - d[5] * d[5], c11 = d[0] * d[2] - d[4] * d[4], c22 = d[0] * d[1] - d[3] * d[3];
  const float c01 = d[4] * d[5] - d[3] * d[2], c02 = d[3] * d[5] - d[4] * d[1], c12 = d[3] * d[4] - d[0] * d[5];
  const float id = 1.0f / (d[0] * c00 + d[3] * c01 + d[4] * c02);
  o[0] = c00 * id;
  o[1] = c11 * id;
  o[2] = c22 * id;
  o[3] = c01 * id;
  o[4] = c02 * id;
  o[5] = c12 * id;
}
// eps = atanh(Z) = Z R(W), W = Z^2, with R(w) = atanh(sqrt w)/sqrt w replaced
// by its [n/n] Pade approximant P_n(W) Q_n(W)^-1.  On the spectrum (w <= 0.36,
// |z| <= 0.6: the caller's bound) the truncation of eps is <= 4e-9 for
// n = 2, 3, 4 up to w = 0.09, 0.23, 0.36 (tools/pade_atanh.py); Q_n's
// eigenvalues stay >= 0.47.  All factors are polynomials of Z, so they commute
// and every product is symmetric.  The order is chosen from the Frobenius
// norm (>= spectral radius), per warp when VOTE.
template <int N>
__device__ __forceinline__ void atanh_pade_n(const float Z[6], const float W[6], float eps[6]) {
  constexpr float P[3][5] = {{1.f, -7.f / 9.f, 64.f / 945.f, 0.f, 0.f},
                             {1.f, -50.f / 39.f, 283.f / 715.f, -256.f / 15015.f, 0.f},
                             {1.f, -91.f / 51.f, 83.f / 85.f, -1289.f / 7735.f, 16384.f / 3828825.f}};
  constexpr float Q[3][5] = {{1.f, -10.f / 9.f, 5.f / 21.f, 0.f, 0.f},
                             {1.f, -21.f / 13.f, 105.f / 143.f, -35.f / 429.f, 0.f},
                             {1.f, -36.f / 17.f, 126.f / 85.f, -84.f / 221.f, 63.f / 2431.f}};
  float Pn[6], Qn[6], Wk[6], Tm[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float dg = q < 3 ? 1.f : 0.f;
    Pn[q] = fmaf(P[N - 2][1], W[q], dg);
    Qn[q] = fmaf(Q[N - 2][1], W[q], dg);
    Wk[q] = W[q];
  }
#pragma unroll
  for (int j = 2; j <= N; ++j) {
    sym_mul(Wk, W, Tm);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      Wk[q] = Tm[q];
      Pn[q] = fmaf(P[N - 2][j], Tm[q], Pn[q]);
      Qn[q] = fmaf(Q[N - 2][j], Tm[q], Qn[q]);
    }
  }
  float Qi[6];
  sym_inv(Qn, Qi);
  sym_mul(Z, Pn, Tm);
  sym_mul(Tm, Qi, eps);
}
template <bool VOTE>
__device__ __forceinline__ void atanh_pade(const float Z[6], float r2, float eps[6]) {
  float W[6];
  sym_mul(Z, Z, W);
  uint32_t ord = r2 <= 0.09f ? 2u : (r2 <= 0.23f ? 3u : 4u);
  if (VOTE) ord = __reduce_max_sync(__activemask(), ord);
  if (ord == 2)
    atanh_pade_n<2>(Z, W, eps);
  else if (ord == 3)
    atanh_pade_n<3>(Z, W, eps);
  else
    atanh_pade_n<4>(Z, W, eps);
}

// Same model for moderate elastic strain (spectral radius of
// Z = (B - I)(B + I)^-1 up to 0.6, i.e. principal stretches^2 in [0.25, 4]),
// still without an eigen-decomposition.  eps = 1/2 log B = atanh(Z) =
// sum_k Z^(2k+1)/(2k+1); the return map is the tensor form of the series
// path below; the update uses E = exp(eps' - eps) - I = sum_k D^k/k!.  Both
// series are summed forward with a per-particle term count chosen from the
// Frobenius norm (>= spectral radius) so the truncation stays below 1e-8;
// the loop index is warp-uniform while any lane is still summing.  Returns 0
// when Z is too large (caller takes the Jacobi path), -1 on a degenerate F.
template <bool VOTE>
__device__ inline int hencky_dp_mid(float H[9], const float X[6], const Material& mat, bool project, float tau[6],
                                    float& J) {
  // M = B + I = 2I + X, Z = X M^-1 (X and M^-1 commute)
  const float m00 = 2.f + X[0], m11 = 2.f + X[1], m22 = 2.f + X[2], m01 = X[3], m02 = X[4], m12 = X[5];
  const float c00 = m11 * m22 - m12 * m12, c11 = m00 * m22 - m02 * m02, c22 = m00 * m11 - m01 * m01;
  const float c01 = m02 * m12 - m01 * m22, c02 = m01 * m12 - m02 * m11, c12 = m01 * m02 - m00 * m12;
  const float det = m00 * c00 + m01 * c01 + m02 * c02;
  if (!(det > 0.0f) || !isfinite(det)) return -1;
  const float id = 1.0f / det;
  const float Mi[6] = {c00 * id, c11 * id, c22 * id, c01 * id, c02 * id, c12 * id};
  float Z[6];
  sym_mul(X, Mi, Z);
  const float r2 = Z[0] * Z[0] + Z[1] * Z[1] + Z[2] * Z[2] + 2.f * (Z[3] * Z[3] + Z[4] * Z[4] + Z[5] * Z[5]);
  if (!(r2 <= 0.36f)) return 0;
  float W[6], T[6], eps[6];
#if SMPM_PADE
  atanh_pade<VOTE>(Z, r2, eps);
#else
  // eps = Z + Z^3/3 + Z^5/5 + ...; truncation after Z^(2K+1) <= r^(2K+3)/((2K+3)(1-r^2))
  sym_mul(Z, Z, W);
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    eps[q] = Z[q];
    T[q] = Z[q];
  }
  const float tol = 5e-9f * (1.0f - r2);
  float bound = r2 * sqrtf(r2);  // r^(2k+1), k = 1
#pragma unroll 1
  for (int k = 1; k <= 16; ++k) {
    if (bound * __fdividef(1.0f, (float)(2 * k + 1)) <= tol) break;  // next term negligible
    float Tn[6];
    sym_mul(T, W, Tn);
    const float ck = __fdividef(1.0f, (float)(2 * k + 1));
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      T[q] = Tn[q];
      eps[q] = fmaf(ck, Tn[q], eps[q]);
    }
    bound *= r2;
  }
#endif
  float e2[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) e2[q] = eps[q];
  const float tr = eps[0] + eps[1] + eps[2];
  bool changed = false;
  if (mat.kind == 1) {
    if (tr > 0.0f) {  // apex: no tensile strength
      changed = (eps[0] != 0.f) || (eps[1] != 0.f) || (eps[2] != 0.f) || (eps[3] != 0.f) || (eps[4] != 0.f) ||
                (eps[5] != 0.f);
#pragma unroll
      for (int q = 0; q < 6; ++q) e2[q] = 0.f;
    } else {
      const float m = tr * (1.0f / 3.0f);
      const float h0 = eps[0] - m, h1 = eps[1] - m, h2 = eps[2] - m;
      const float en = sqrtf(h0 * h0 + h1 * h1 + h2 * h2 + 2.f * (eps[3] * eps[3] + eps[4] * eps[4] + eps[5] * eps[5]));
      const float dg = en + mat.alpha * mat.ratio * tr;
      if (dg > 0.0f && en > 0.0f) {
        const float c = dg / en;
        e2[0] = eps[0] - c * h0;
        e2[1] = eps[1] - c * h1;
        e2[2] = eps[2] - c * h2;
        e2[3] = eps[3] - c * eps[3];
        e2[4] = eps[4] - c * eps[4];
        e2[5] = eps[5] - c * eps[5];
        changed = true;
      }
    }
  }
  if (changed && project) {
    // E = exp(D) - I = D + D^2/2! + ..., D = eps' - eps (a polynomial of eps)
    float D[6], E[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      D[q] = e2[q] - eps[q];
      E[q] = D[q];
      T[q] = D[q];
    }
    const float d2 = D[0] * D[0] + D[1] * D[1] + D[2] * D[2] + 2.f * (D[3] * D[3] + D[4] * D[4] + D[5] * D[5]);
    const float d = sqrtf(d2);
    float bound_e = d;  // ||D^k / k!||
#pragma unroll 1
    for (int k = 2; k <= 20; ++k) {
      bound_e *= d * __fdividef(1.0f, (float)k);
      if (bound_e <= 5e-9f) break;
      float Tn[6];
      sym_mul(T, D, Tn);
      const float ik = __fdividef(1.0f, (float)k);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        T[q] = Tn[q] * ik;
        E[q] += T[q];
      }
    }
    const float Ef[9] = {E[0], E[3], E[4], E[3], E[1], E[5], E[4], E[5], E[2]};
    float Hn[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        Hn[3 * i + j] = H[3 * i + j] + (Ef[3 * i + j] + (Ef[3 * i] * H[j] + Ef[3 * i + 1] * H[3 + j] + Ef[3 * i + 2] * H[6 + j]));
#pragma unroll
    for (int q = 0; q < 9; ++q) H[q] = Hn[q];
  }
  const float tr2 = e2[0] + e2[1] + e2[2];
  const float lt = mat.lam * tr2, m2u = 2.0f * mat.mu;
  tau[0] = m2u * e2[0] + lt;
  tau[1] = m2u * e2[1] + lt;
  tau[2] = m2u * e2[2] + lt;
  tau[3] = m2u * e2[3];
  tau[4] = m2u * e2[4];
  tau[5] = m2u * e2[5];
  J = expf(tr2);
  return 1;
}

// Same model without an eigen-decomposition, for small elastic strain
// (||B - I||_inf <= 0.05, the normal case: Drucker-Prager keeps elastic
// strains small).  Hencky strain eps = 1/2 log(B), B = F F^T = I + X, as a
// 5-term series (truncation < 0.05^6/6); the return map is isotropic
// so it acts on the tensor (deviator norm = Frobenius norm = principal norm,
// materials.py:147-166); tau = 2 mu eps' + lam tr(eps') I equals
// sum_k t_k u_k u_k^T of materials.py:233-238; and since eps' is a polynomial
// of eps, F' = U exp(e') V^T = exp(eps' - eps) F.
// MID: strains beyond the series range take hencky_dp_mid before the Jacobi
// path (chosen per kernel variant, see hencky_dp below).
// MODE 0: series, Jacobi beyond; 1: series, moderate-strain path beyond (Jacobi
// past that); 2: as 1, but a warp with any lane beyond the series range sends
// all its lanes down the moderate-strain path (one path per warp instead of
// both: the late, disordered regime mixes the two in most warps).  MODE 2
// makes a particle's path depend on its warp neighbours, so the deterministic
// mode (layout-independent bits) uses 1.
template <int MODE>
__device__ inline bool hencky_dp_body(float H[9], const Material& mat, bool project, float tau[6], float& J) {
  const float trH = H[0] + H[4] + H[8];
  const float m2 = (H[0] * H[4] - H[1] * H[3]) + (H[0] * H[8] - H[2] * H[6]) + (H[4] * H[8] - H[5] * H[7]);
  const float dH = H[0] * (H[4] * H[8] - H[5] * H[7]) - H[1] * (H[3] * H[8] - H[5] * H[6]) +
                   H[2] * (H[3] * H[7] - H[4] * H[6]);
  const float det = 1.0f + (trH + (m2 + dH));
  if (!(det > 0.0f) || !isfinite(det)) return false;
  // X = B - I = H + H^T + H H^T
  float X[6];
  X[0] = 2.f * H[0] + (H[0] * H[0] + H[1] * H[1] + H[2] * H[2]);
  X[1] = 2.f * H[4] + (H[3] * H[3] + H[4] * H[4] + H[5] * H[5]);
  X[2] = 2.f * H[8] + (H[6] * H[6] + H[7] * H[7] + H[8] * H[8]);
  X[3] = (H[1] + H[3]) + (H[0] * H[3] + H[1] * H[4] + H[2] * H[5]);
  X[4] = (H[2] + H[6]) + (H[0] * H[6] + H[1] * H[7] + H[2] * H[8]);
  X[5] = (H[5] + H[7]) + (H[3] * H[6] + H[4] * H[7] + H[5] * H[8]);
  const float nx = fmaxf(fabsf(X[0]) + fabsf(X[3]) + fabsf(X[4]),
                         fmaxf(fabsf(X[3]) + fabsf(X[1]) + fabsf(X[5]), fabsf(X[4]) + fabsf(X[5]) + fabsf(X[2])));
  const bool big = !(nx <= 0.05f);
  bool use_mid = MODE != 0 && big;
  if (MODE == 2) use_mid = __any_sync(__activemask(), big);
  if (use_mid) {
    const int mid = hencky_dp_mid<MODE == 2>(H, X, mat, project, tau, J);
    if (mid != 0) return mid > 0;
  }
  if (big) return hencky_dp_eig(H, mat, project, tau, J);
  // log(I + X) = X (1 - X (1/2 - X (1/3 - X (1/4 - X/5))))  (Horner); for
  // ||X|| <= 0.05 the truncation is < 0.05^6/6 = 2.6e-9, below fp32 rounding
  // of the strains (~1e-8 absolute).  For ||X|| <= 0.01 (the common case of a
  // resting or slowly deforming granular body) three terms truncate at
  // 0.01^4/4 = 2.5e-9: two matrix products fewer.
  // Two terms for ||X|| <= 1e-3 (truncation X^3/3 <= 3.3e-10).  The term
  // count is voted per warp in MODE 2 (one path per warp).
  float P[6], T[6];
  uint32_t ltier = nx <= 1e-3f ? 0u : (nx <= 0.01f ? 1u : 2u);
  if (MODE == 2) ltier = __reduce_max_sync(__activemask(), ltier);
  if (ltier == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) P[q] = -0.5f * X[q];
    P[0] += 1.f;
    P[1] += 1.f;
    P[2] += 1.f;
  } else if (ltier == 1) {
#pragma unroll
    for (int q = 0; q < 6; ++q) P[q] = -X[q] * (1.f / 3.f);
    P[0] += 0.5f;
    P[1] += 0.5f;
    P[2] += 0.5f;
    sym_mul(X, P, T);
#pragma unroll
    for (int q = 0; q < 6; ++q) P[q] = -T[q];
    P[0] += 1.f;
    P[1] += 1.f;
    P[2] += 1.f;
  } else {
    const float coef[4] = {1.f / 4.f, 1.f / 3.f, 1.f / 2.f, 1.f};
#pragma unroll
    for (int q = 0; q < 6; ++q) P[q] = -X[q] * (1.f / 5.f);
    P[0] += coef[0];
    P[1] += coef[0];
    P[2] += coef[0];
#pragma unroll
    for (int it = 1; it < 4; ++it) {
      sym_mul(X, P, T);
#pragma unroll
      for (int q = 0; q < 6; ++q) P[q] = -T[q];
      P[0] += coef[it];
      P[1] += coef[it];
      P[2] += coef[it];
    }
  }
  float eps[6];
  sym_mul(X, P, eps);
#pragma unroll
  for (int q = 0; q < 6; ++q) eps[q] *= 0.5f;
  float e2[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) e2[q] = eps[q];
  float tr = eps[0] + eps[1] + eps[2];
  bool changed = false;
  if (mat.kind == 1) {
    if (tr > 0.0f) {  // apex: no tensile strength
      changed = (eps[0] != 0.f) || (eps[1] != 0.f) || (eps[2] != 0.f) || (eps[3] != 0.f) || (eps[4] != 0.f) ||
                (eps[5] != 0.f);
#pragma unroll
      for (int q = 0; q < 6; ++q) e2[q] = 0.f;
    } else {
      const float m = tr * (1.0f / 3.0f);
      const float h0 = eps[0] - m, h1 = eps[1] - m, h2 = eps[2] - m;
      const float en = sqrtf(h0 * h0 + h1 * h1 + h2 * h2 + 2.f * (eps[3] * eps[3] + eps[4] * eps[4] + eps[5] * eps[5]));
      const float dg = en + mat.alpha * mat.ratio * tr;
      if (dg > 0.0f && en > 0.0f) {
        const float c = dg / en;
        e2[0] = eps[0] - c * h0;
        e2[1] = eps[1] - c * h1;
        e2[2] = eps[2] - c * h2;
        e2[3] = eps[3] - c * eps[3];
        e2[4] = eps[4] - c * eps[4];
        e2[5] = eps[5] - c * eps[5];
        changed = true;
      }
    }
  }
  if (changed && project) {
    // H' = H + E (I + H), E = exp(D) - I = D (1 + D/2 (1 + D/3 (1 + D/4))), D = eps' - eps;
    // two terms for ||D|| <= 1e-3 (truncation D^3/6 <= 1.7e-10), three for
    // ||D|| <= 1e-2 (D^4/24 <= 4.2e-10), voted per warp in MODE 2
    float D[6], E[6], Q[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) D[q] = e2[q] - eps[q];
    const float dn = fmaxf(fabsf(D[0]) + fabsf(D[3]) + fabsf(D[4]),
                           fmaxf(fabsf(D[3]) + fabsf(D[1]) + fabsf(D[5]), fabsf(D[4]) + fabsf(D[5]) + fabsf(D[2])));
    uint32_t et = dn <= 1e-3f ? 0u : (dn <= 1e-2f ? 1u : 2u);
    if (MODE == 2) et = __reduce_max_sync(__activemask(), et);
#pragma unroll
    for (int q = 0; q < 6; ++q) Q[q] = D[q] * (et == 2 ? 0.25f : (et == 1 ? (1.f / 3.f) : 0.5f));
    Q[0] += 1.f;
    Q[1] += 1.f;
    Q[2] += 1.f;
    if (et == 2) {
      sym_mul(D, Q, T);
#pragma unroll
      for (int q = 0; q < 6; ++q) Q[q] = T[q] * (1.f / 3.f);
      Q[0] += 1.f;
      Q[1] += 1.f;
      Q[2] += 1.f;
    }
    if (et >= 1) {
      sym_mul(D, Q, T);
#pragma unroll
      for (int q = 0; q < 6; ++q) Q[q] = T[q] * 0.5f;
      Q[0] += 1.f;
      Q[1] += 1.f;
      Q[2] += 1.f;
    }
    sym_mul(D, Q, E);
    // full 3x3 of E (symmetric)
    const float Ef[9] = {E[0], E[3], E[4], E[3], E[1], E[5], E[4], E[5], E[2]};
    float Hn[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        Hn[3 * i + j] = H[3 * i + j] + (Ef[3 * i + j] + (Ef[3 * i] * H[j] + Ef[3 * i + 1] * H[3 + j] + Ef[3 * i + 2] * H[6 + j]));
#pragma unroll
    for (int q = 0; q < 9; ++q) H[q] = Hn[q];
  }
  const float tr2 = e2[0] + e2[1] + e2[2];
  const float lt = mat.lam * tr2, m2u = 2.0f * mat.mu;
  tau[0] = m2u * e2[0] + lt;
  tau[1] = m2u * e2[1] + lt;
  tau[2] = m2u * e2[2] + lt;
  tau[3] = m2u * e2[3];
  tau[4] = m2u * e2[4];
  tau[5] = m2u * e2[5];
  J = expf(tr2);
  return true;
}

// ------------------------------------------------------------ grid update
// Boundary table (solver.py:841-860): kind 0 plane, 1 heightfield.
struct Boundary {
  double point[3];
  double normal[3];
  double mu;
  int kind;
  int pad;
};
struct Heightfield {
  const double* data;  // [nx][ny]
  int nx, ny;
  double x0, y0, cell;
};
struct GridParams {
  double h, dt, mass_floor;
  double gravity[3];
  int n_bc;
  int pad;
  const Boundary* bc;
  Heightfield hf;
};

// solver.py:241-274 (bilinear, clamped), fp64 exact mirror
__device__ inline void hf_sample(const Heightfield& hf, double x, double y, double& z, double& dzdx, double& dzdy) {
  double fx = __ddiv_rn(__dadd_rn(x, -hf.x0), hf.cell), fy = __ddiv_rn(__dadd_rn(y, -hf.y0), hf.cell);
  double fi = floor(fx), fj = floor(fy);
  long long i0 = (long long)fi, j0 = (long long)fj;
  if (i0 < 0) i0 = 0;
  if (i0 > hf.nx - 2) i0 = hf.nx - 2;
  if (j0 < 0) j0 = 0;
  if (j0 > hf.ny - 2) j0 = hf.ny - 2;
  double tx = __dadd_rn(fx, -double(i0)), ty = __dadd_rn(fy, -double(j0));
  tx = tx < 0.0 ? 0.0 : (tx > 1.0 ? 1.0 : tx);
  ty = ty < 0.0 ? 0.0 : (ty > 1.0 ? 1.0 : ty);
  double z00 = hf.data[i0 * hf.ny + j0], z10 = hf.data[(i0 + 1) * hf.ny + j0];
  double z01 = hf.data[i0 * hf.ny + j0 + 1], z11 = hf.data[(i0 + 1) * hf.ny + j0 + 1];
  double omx = __dadd_rn(1.0, -tx), omy = __dadd_rn(1.0, -ty);
  z = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(z00, omx), omy), __dmul_rn(__dmul_rn(z10, tx), omy)),
                          __dmul_rn(__dmul_rn(z01, omx), ty)),
                __dmul_rn(__dmul_rn(z11, tx), ty));
  dzdx = __ddiv_rn(__dadd_rn(__dmul_rn(__dadd_rn(z10, -z00), omy), __dmul_rn(__dadd_rn(z11, -z01), ty)), hf.cell);
  dzdy = __ddiv_rn(__dadd_rn(__dmul_rn(__dadd_rn(z01, -z00), omx), __dmul_rn(__dadd_rn(z11, -z10), tx)), hf.cell);
}

// solver.py:277-291
__device__ inline void coulomb_project(double& v0, double& v1, double& v2, double n0, double n1, double n2,
                                       double mu) {
  double vn = v0 * n0 + v1 * n1 + v2 * n2;
  if (vn >= 0.0) return;
  double t0 = v0 - vn * n0, t1 = v1 - vn * n1, t2 = v2 - vn * n2;
  double tn = sqrt(t0 * t0 + t1 * t1 + t2 * t2);
  if (tn <= 0.0) {
    v0 = v1 = v2 = 0.0;
    return;
  }
  double scale = 1.0 + mu * vn / tn;
  if (scale < 0.0) scale = 0.0;
  v0 = scale * t0;
  v1 = scale * t1;
  v2 = scale * t2;
}

// Terrain under one node column (nx, ny): the heightfield sample depends
// only on the node's x, y, so it is evaluated once per column of a block.
struct Column {
  double zs, n0, n1, n2;  // terrain height and unit normal (-zx, -zy, 1)/len
};
__device__ inline void column_terrain(const GridParams& gp, int nx, int ny, Column& col) {
  col.zs = 0.0;
  col.n0 = col.n1 = 0.0;
  col.n2 = 1.0;
  for (int b = 0; b < gp.n_bc; ++b) {
    if (gp.bc[b].kind != 1) continue;
    double zx, zy;
    hf_sample(gp.hf, __dmul_rn(double(nx), gp.h), __dmul_rn(double(ny), gp.h), col.zs, zx, zy);
    const double il = 1.0 / sqrt(zx * zx + zy * zy + 1.0);
    col.n0 = -zx * il;
    col.n1 = -zy * il;
    col.n2 = il;
  }
}

// One node of _grid_update (solver.py:578-625).  `force` excludes gravity
// here; gravity enters as m*g (the scatter's sum_p w m g equals m_node g).
// Node position and boundary predicates are fp64 and contraction-free, so the
// plane / terrain decisions match the reference for the same node.  `col` is
// the node column's terrain (column_terrain).
__device__ inline void grid_node_col(const GridParams& gp, const Column& col, int nx, int ny, int nz, double m,
                                     double p0, double p1, double p2, double f0, double f1, double f2, float& o0,
                                     float& o1, float& o2) {
  if (m <= gp.mass_floor) {
    o0 = o1 = o2 = 0.0f;
    return;
  }
  double inv_m = 1.0 / m;
  double v0 = (p0 + gp.dt * (f0 + m * gp.gravity[0])) * inv_m;
  double v1 = (p1 + gp.dt * (f1 + m * gp.gravity[1])) * inv_m;
  double v2 = (p2 + gp.dt * (f2 + m * gp.gravity[2])) * inv_m;
  if (gp.n_bc > 0) {
    double x0 = __dmul_rn(double(nx), gp.h), x1 = __dmul_rn(double(ny), gp.h), x2 = __dmul_rn(double(nz), gp.h);
    for (int b = 0; b < gp.n_bc; ++b) {
      const Boundary& bc = gp.bc[b];
      if (bc.kind == 0) {
        double sd = __dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(x0, -bc.point[0]), bc.normal[0]),
                                        __dmul_rn(__dadd_rn(x1, -bc.point[1]), bc.normal[1])),
                              __dmul_rn(__dadd_rn(x2, -bc.point[2]), bc.normal[2]));
        if (sd <= 0.0) coulomb_project(v0, v1, v2, bc.normal[0], bc.normal[1], bc.normal[2], bc.mu);
      } else if (__dadd_rn(x2, -col.zs) <= 0.0) {
        coulomb_project(v0, v1, v2, col.n0, col.n1, col.n2, bc.mu);
      }
    }
  }
  o0 = float(v0);
  o1 = float(v1);
  o2 = float(v2);
}
__device__ inline void grid_node(const GridParams& gp, int nx, int ny, int nz, double m, double p0, double p1,
                                 double p2, double f0, double f1, double f2, float& o0, float& o1, float& o2) {
  Column col;
  column_terrain(gp, nx, ny, col);
  grid_node_col(gp, col, nx, ny, nz, m, p0, p1, p2, f0, f1, f2, o0, o1, o2);
}

__device__ inline void err_report(unsigned long long* err, uint32_t code, uint64_t particle) {
  atomicMin(err, (unsigned long long)err_word(code, particle));
}


// CV = 0: series + Jacobi, inlined (ordered regime); 1: series + moderate-
// strain path + Jacobi, inlined, path voted per warp (MODE 2 above); 2: the same compiled once, out of line, so
// every deterministic kernel variant (both work-item layouts) runs the same
// machine code and bitwise results do not depend on the layout choice
// (inlined copies may contract multiply-adds differently).
// By-value argument and result (registers under the device ABI) instead of
// pointers to the caller's arrays, which would force them to local memory.
struct HenckyIO {
  float H[9];
  float tau[6];
  float J;
  int ok;
};
static __device__ __noinline__ HenckyIO hencky_dp_shared(HenckyIO io, const Material& mat, bool project) {
  io.ok = hencky_dp_body<1>(io.H, mat, project, io.tau, io.J) ? 1 : 0;
  return io;
}
template <int CV = 0>
__device__ __forceinline__ bool hencky_dp(float H[9], const Material& mat, bool project, float tau[6], float& J) {
  if (CV == 2) {
    HenckyIO io;
#pragma unroll
    for (int q = 0; q < 9; ++q) io.H[q] = H[q];
    io = hencky_dp_shared(io, mat, project);
#pragma unroll
    for (int q = 0; q < 9; ++q) H[q] = io.H[q];
#pragma unroll
    for (int q = 0; q < 6; ++q) tau[q] = io.tau[q];
    J = io.J;
    return io.ok != 0;
  }
  return hencky_dp_body<CV == 1 ? 2 : 0>(H, mat, project, tau, J);
}

}  // namespace smpm
