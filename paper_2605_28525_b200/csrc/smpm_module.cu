// Module-level GPU entry points: the reference's hash table, grid build and
// transfer functions as stand-alone kernels (sparse_hash.py, grid_index.py,
// solver.py:863-924, materials.py:250-267).  They share every device function
// with the fused step (smpm_common.cuh) and back the phase-level parity tests.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../../include/smpm.h"
#include "smpm_common.cuh"
#include "smpm_internal.h"

using namespace smpm;

namespace {
thread_local char g_err2[512] = "";
#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      snprintf(g_err2, sizeof(g_err2), "%s failed: %s", #call, cudaGetErrorString(e_));            \
      smpm_internal_set_error(g_err2);                                                             \
      return SMPM_ERR_CUDA;                                                                        \
    }                                                                                              \
  } while (0)

inline cudaStream_t st(void* s) { return (cudaStream_t)s; }

HashView view(const smpm_hash_desc* h) {
  HashView v;
  v.keys = h->keys;
  v.vals = h->vals;
  v.mask = uint32_t(h->n_slots - 1);
  v.cap_blocks = h->cap_blocks;
  v.counter = h->counter;
  v.overflow = h->overflow;
  v.active_keys = h->active_keys;
  v.slot_of_rank = h->slot_of_rank;
  return v;
}

int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

// ------------------------------------------------------------------ hash
__global__ void k_hash_clear(HashView h, uint64_t n_slots) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_slots; i += uint64_t(gridDim.x) * blockDim.x) {
    h.keys[i] = EMPTY_KEY;
    h.vals[i] = EMPTY_VAL;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *h.counter = 0;
    *h.overflow = 0;
  }
}

__global__ void k_hash_insert_many(HashView h, const uint64_t* __restrict__ packed, int64_t n, uint32_t* ranks,
                                   uint8_t* fresh) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    bool f = false;
    uint32_t r = hash_insert(h, packed[i], &f);
    ranks[i] = r;
    if (fresh) fresh[i] = f ? 1 : 0;
  }
}

__global__ void k_hash_lookup_many(HashView h, const uint64_t* __restrict__ packed, int64_t n, uint32_t* ranks) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    ranks[i] = hash_lookup(h.keys, h.vals, h.mask, packed[i]);
}

// _insert_particle_blocks (sparse_hash.py:170-191).  first_pos records the
// smallest (particle, corner) encounter per slot: the reference's serial
// build assigns ranks in exactly that order (loops bi, bj, bk nested).
__global__ void k_insert_particle_blocks(HashView h, const double* __restrict__ x, int64_t n, double inv_h,
                                         unsigned long long* first_pos, unsigned long long* err) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    int b[3];
    float d;
    bool ok = true;
    for (int a = 0; a < 3; ++a) ok = ok && axis_base(x[3 * p + a], inv_h, b[a], d) && axis_in_key_range(b[a]);
    if (!ok) {
      err_report(err, ERR_KEY_RANGE, p);
      continue;
    }
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = b[a] >> 2;
      hi[a] = (b[a] + 2) >> 2;
    }
    int c = 0;
    for (int bi = lo[0]; bi <= hi[0]; ++bi)
      for (int bj = lo[1]; bj <= hi[1]; ++bj)
        for (int bk = lo[2]; bk <= hi[2]; ++bk, ++c) {
          uint64_t key = pack_key(bi, bj, bk);
          uint32_t r = hash_insert(h, key);
          if (first_pos && r != EMPTY_VAL) {
            // locate the slot again (the key is present now)
            uint32_t s = uint32_t(mix64(key)) & h.mask;
            while (h.keys[s] != key) s = (s + 1) & h.mask;
            atomicMin(&first_pos[s], (unsigned long long)(p * 8 + c));
          }
        }
  }
}

__global__ void k_active_blocks(const uint64_t* __restrict__ active_keys, int64_t nb, int32_t* blocks) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < nb; r += int64_t(gridDim.x) * blockDim.x) {
    int bi, bj, bk;
    unpack_key(active_keys[r], bi, bj, bk);
    blocks[3 * r] = bi;
    blocks[3 * r + 1] = bj;
    blocks[3 * r + 2] = bk;
  }
}

// ------------------------------------------------------ LSD radix sort
// Stable sort of (u64 key, u32 value) pairs, 8-bit digits.  Used to put block
// ranks in canonical order (deterministic mode); not on the timed path.
constexpr int RS_TILE = 4096;
constexpr int RS_T = 256;

__global__ void k_rs_hist(const uint64_t* __restrict__ keys, const uint32_t* nptr, int shift, uint32_t* hist,
                          int ntiles_max) {
  __shared__ uint32_t hs[256];
  const uint32_t n = *nptr;
  const int ntiles = (n + RS_TILE - 1) / RS_TILE;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    hs[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < RS_TILE; i += RS_T) {
      uint32_t j = tile * RS_TILE + i;
      if (j < n) atomicAdd(&hs[(keys[j] >> shift) & 255], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * ntiles_max + tile] = hs[threadIdx.x];
    __syncthreads();
  }
}

// exclusive scan over hist[digit][tile] (digit-major, ntiles used columns)
__global__ void k_rs_scan(uint32_t* hist, const uint32_t* nptr, int ntiles_max) {
  __shared__ uint32_t sh[32];
  const uint32_t n = *nptr;
  const int ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int total = 256 * ntiles;
  uint32_t carry = 0;
  for (int base = 0; base < total; base += blockDim.x) {
    int i = base + threadIdx.x;
    uint32_t v = 0;
    int d = 0, t = 0;
    if (i < total) {
      d = i / ntiles;
      t = i % ntiles;
      v = hist[d * ntiles_max + t];
    }
    uint32_t x = v;
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t s = lane < int(blockDim.x / 32) ? sh[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      sh[lane] = s;
    }
    __syncthreads();
    uint32_t pre = (w ? sh[w - 1] : 0) + x - v;
    uint32_t tot = sh[blockDim.x / 32 - 1];
    if (i < total) hist[d * ntiles_max + t] = carry + pre;
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RS_T) k_rs_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                     uint64_t* kout, uint32_t* vout, const uint32_t* nptr, int shift,
                                                     const uint32_t* hist, int ntiles_max) {
  __shared__ uint32_t running[256];
  __shared__ uint32_t wcount[8][256];
  const uint32_t n = *nptr;
  const int ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    running[threadIdx.x] = hist[threadIdx.x * ntiles_max + tile];
    for (int round = 0; round < RS_TILE / RS_T; ++round) {
      for (int q = 0; q < 8; ++q) wcount[q][threadIdx.x] = 0;
      __syncthreads();
      uint32_t j = tile * RS_TILE + round * RS_T + threadIdx.x;
      bool valid = j < n;
      uint64_t k = valid ? kin[j] : 0;
      uint32_t d = valid ? uint32_t((k >> shift) & 255) : 256u + lane;  // invalid lanes: unique
      uint32_t peers = __match_any_sync(0xffffffffu, d);
      uint32_t rin = __popc(peers & ((1u << lane) - 1));
      if (valid && rin == 0) wcount[w][d] = __popc(peers);
      __syncthreads();
      if (valid) {
        uint32_t pos = running[d] + rin;
        for (int q = 0; q < w; ++q) pos += wcount[q][d];
        kout[pos] = k;
        vout[pos] = vin[j];
      }
      __syncthreads();
      uint32_t add = 0;
      for (int q = 0; q < 8; ++q) add += wcount[q][threadIdx.x];
      running[threadIdx.x] += add;
      __syncthreads();
    }
  }
}

__global__ void k_canon_prep(HashView h, int mode, const unsigned long long* first_pos, uint64_t* sk, uint32_t* sv) {
  const uint32_t n = min(*h.counter, h.cap_blocks);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    sk[r] = mode == 0 ? h.active_keys[r] : first_pos[h.slot_of_rank[r]];
    sv[r] = r;
  }
}

__global__ void k_canon_apply(HashView h, const uint32_t* __restrict__ order, uint64_t* tmp_keys,
                              uint32_t* tmp_slots) {
  const uint32_t n = min(*h.counter, h.cap_blocks);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t old = order[i];
    tmp_keys[i] = h.active_keys[old];
    tmp_slots[i] = h.slot_of_rank[old];
  }
}

__global__ void k_canon_write(HashView h, const uint64_t* tmp_keys, const uint32_t* tmp_slots) {
  const uint32_t n = min(*h.counter, h.cap_blocks);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    h.active_keys[i] = tmp_keys[i];
    h.slot_of_rank[i] = tmp_slots[i];
    h.vals[tmp_slots[i]] = i;
  }
}

// ------------------------------------------------------------ transfers
struct Stencil {
  int base[3];
  float d[3];
  float w[3][3], g[3][3];
};

__device__ inline bool stencil_of(const double* x, double inv_h, Stencil& s) {
  for (int a = 0; a < 3; ++a) {
    if (!axis_base(x[a], inv_h, s.base[a], s.d[a])) return false;
    bspline(s.d[a], s.w[a], s.g[a]);
  }
  return true;
}

__device__ inline uint32_t node_slot(const HashView& h, int n0, int n1, int n2) {
  uint32_t r = hash_lookup(h.keys, h.vals, h.mask, pack_key(n0 >> 2, n1 >> 2, n2 >> 2));
  if (r == EMPTY_VAL) return EMPTY_VAL;
  return r * 64 + uint32_t(((n0 & 3) << 4) | ((n1 & 3) << 2) | (n2 & 3));
}

__global__ void k_bspline(const double* __restrict__ x, int64_t n, double inv_h, int64_t* base, double* w,
                          double* dw) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    Stencil s;
    if (!stencil_of(&x[3 * p], inv_h, s)) continue;
    for (int a = 0; a < 3; ++a) {
      base[3 * p + a] = s.base[a];
      for (int o = 0; o < 3; ++o) {
        w[9 * p + 3 * a + o] = s.w[a][o];
        dw[9 * p + 3 * a + o] = double(s.g[a][o]) * inv_h;
      }
    }
  }
}

// p2g + grid_forces (solver.py:309-453), thread per particle, fp32 atomics
__global__ void k_p2g(HashView h, double inv_h, double hh, float g0, float g1, float g2, int64_t n,
                      const double* __restrict__ x, const double* __restrict__ v, const double* __restrict__ C,
                      const double* __restrict__ m, const double* __restrict__ sigma, const double* __restrict__ jac,
                      const double* __restrict__ V0, float* mass, float* mom, float* force, unsigned long long* err) {
  const float hf = float(hh), ih = float(inv_h);
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    Stencil s;
    if (!stencil_of(&x[3 * p], inv_h, s)) {
      err_report(err, ERR_KEY_RANGE, p);
      continue;
    }
    float mp = float(m[p]);
    float pv[3], c[9], sg[9];
    float vol = 0.f;
    if (mass || mom)
      for (int a = 0; a < 3; ++a) pv[a] = float(v[3 * p + a]);
    if (mom)
      for (int q = 0; q < 9; ++q) c[q] = float(C[9 * p + q]);
    if (force) {
      vol = float(V0[p] * jac[p]);
      for (int q = 0; q < 9; ++q) sg[q] = float(sigma[9 * p + q]);
    }
    for (int oi = 0; oi < 3; ++oi)
      for (int oj = 0; oj < 3; ++oj)
        for (int ok = 0; ok < 3; ++ok) {
          uint32_t idx = node_slot(h, s.base[0] + oi, s.base[1] + oj, s.base[2] + ok);
          if (idx == EMPTY_VAL) {
            err_report(err, ERR_INACTIVE, p);
            continue;
          }
          float wk = s.w[0][oi] * s.w[1][oj] * s.w[2][ok];
          float wm = wk * mp;
          if (mass) atomicAdd(&mass[idx], wm);
          if (mom) {
            float dx0 = (float(oi) - s.d[0]) * hf, dx1 = (float(oj) - s.d[1]) * hf, dx2 = (float(ok) - s.d[2]) * hf;
            for (int a = 0; a < 3; ++a)
              atomicAdd(&mom[3 * idx + a], wm * (pv[a] + c[3 * a] * dx0 + c[3 * a + 1] * dx1 + c[3 * a + 2] * dx2));
          }
          if (force) {
            float gx = s.g[0][oi] * s.w[1][oj] * s.w[2][ok] * ih;
            float gy = s.w[0][oi] * s.g[1][oj] * s.w[2][ok] * ih;
            float gz = s.w[0][oi] * s.w[1][oj] * s.g[2][ok] * ih;
            float gg[3] = {g0, g1, g2};
            for (int a = 0; a < 3; ++a)
              atomicAdd(&force[3 * idx + a],
                        -vol * (sg[3 * a] * gx + sg[3 * a + 1] * gy + sg[3 * a + 2] * gz) + wm * gg[a]);
          }
        }
  }
}

__global__ void k_grid_update(GridParams gp, int64_t n_nodes, float* mass, float* vel, const float* force,
                              const int32_t* __restrict__ blocks) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_nodes; c += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = c >> 6;
    int l = int(c & 63);
    float o0, o1, o2;
    grid_node(gp, blocks[3 * r] * 4 + (l >> 4), blocks[3 * r + 1] * 4 + ((l >> 2) & 3), blocks[3 * r + 2] * 4 + (l & 3),
              mass[c], vel[3 * c], vel[3 * c + 1], vel[3 * c + 2], force[3 * c], force[3 * c + 1], force[3 * c + 2],
              o0, o1, o2);
    vel[3 * c] = o0;
    vel[3 * c + 1] = o1;
    vel[3 * c + 2] = o2;
  }
}

// _g2p (solver.py:628-732)
__global__ void k_g2p(HashView h, double inv_h, double hh, double dt, int64_t n, double* x, double* v, double* C,
                      double* F, const float* __restrict__ vel, unsigned long long* err) {
  const float hf = float(hh), ih = float(inv_h);
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    Stencil s;
    if (!stencil_of(&x[3 * p], inv_h, s)) {
      err_report(err, ERR_KEY_RANGE, p);
      continue;
    }
    float vv[3] = {0, 0, 0}, B[9] = {0}, A[9] = {0};
    for (int oi = 0; oi < 3; ++oi)
      for (int oj = 0; oj < 3; ++oj)
        for (int ok = 0; ok < 3; ++ok) {
          uint32_t idx = node_slot(h, s.base[0] + oi, s.base[1] + oj, s.base[2] + ok);
          if (idx == EMPTY_VAL) {
            err_report(err, ERR_INACTIVE, p);
            continue;
          }
          float wk = s.w[0][oi] * s.w[1][oj] * s.w[2][ok];
          float dxs[3] = {(float(oi) - s.d[0]) * hf, (float(oj) - s.d[1]) * hf, (float(ok) - s.d[2]) * hf};
          float gr[3] = {s.g[0][oi] * s.w[1][oj] * s.w[2][ok] * ih, s.w[0][oi] * s.g[1][oj] * s.w[2][ok] * ih,
                         s.w[0][oi] * s.w[1][oj] * s.g[2][ok] * ih};
          for (int a = 0; a < 3; ++a) {
            float gv = vel[3 * idx + a];
            vv[a] += wk * gv;
            for (int b = 0; b < 3; ++b) {
              B[3 * a + b] += wk * gv * dxs[b];
              A[3 * a + b] += gv * gr[b];
            }
          }
        }
    const float dinv = 4.0f * ih * ih;
    float Ho[9];  // H = F - I: F <- F + dt a F  <=>  H <- H + dt a (I + H)
    for (int q = 0; q < 9; ++q) Ho[q] = float(F[9 * p + q] - ((q == 0 || q == 4 || q == 8) ? 1.0 : 0.0));
    for (int a = 0; a < 3; ++a) {
      v[3 * p + a] = vv[a];
      for (int b = 0; b < 3; ++b) {
        C[9 * p + 3 * a + b] = B[3 * a + b] * dinv;
        const float hn = Ho[3 * a + b] + float(dt) * (A[3 * a + b] + (A[3 * a] * Ho[b] + A[3 * a + 1] * Ho[3 + b] +
                                                                    A[3 * a + 2] * Ho[6 + b]));
        F[9 * p + 3 * a + b] = double(hn) + (a == b ? 1.0 : 0.0);
      }
      x[3 * p + a] = __dadd_rn(x[3 * p + a], __dmul_rn(dt, double(vv[a])));
    }
  }
}

__global__ void k_stress(const Material* __restrict__ mats, int n_mat, int64_t n, double* F, double* sigma,
                         double* jac, const int64_t* __restrict__ mat_id, unsigned long long* err) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    float Fl[9], tau[6], J;  // H = F - I
    for (int q = 0; q < 9; ++q) Fl[q] = float(F[9 * p + q] - ((q == 0 || q == 4 || q == 8) ? 1.0 : 0.0));
    int64_t mid = mat_id[p];
    Material m = mats[(mid >= 0 && mid < n_mat) ? mid : 0];
    // moderate-strain path as in the late-time fused kernel (its Jacobi
    // fallback beyond), so module-level parity covers both
    if (!hencky_dp<1>(Fl, m, true, tau, J)) {
      err_report(err, ERR_DEGENERATE_F, p);
      continue;
    }
    for (int q = 0; q < 9; ++q) F[9 * p + q] = double(Fl[q]) + ((q == 0 || q == 4 || q == 8) ? 1.0 : 0.0);
    jac[p] = J;
    const int map[9] = {0, 3, 4, 3, 1, 5, 4, 5, 2};
    float iJ = 1.0f / J;
    for (int q = 0; q < 9; ++q) sigma[9 * p + q] = tau[map[q]] * iJ;
  }
}

// count_active_nodes: per particle and corner block, OR the stencil nodes
// that fall in that block into its 64-bit node mask
__global__ void k_node_masks(HashView h, const double* __restrict__ x, int64_t n, double inv_h, uint64_t* nodemask) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    int b[3];
    float d;
    bool ok = true;
    for (int a = 0; a < 3; ++a) ok = ok && axis_base(x[3 * p + a], inv_h, b[a], d);
    if (!ok) continue;
    for (int c = 0; c < 8; ++c) {
      int bb[3] = {(b[0] >> 2) + (c >> 2), (b[1] >> 2) + ((c >> 1) & 1), (b[2] >> 2) + (c & 1)};
      uint64_t mk = 0;
      for (int oi = 0; oi < 3; ++oi)
        for (int oj = 0; oj < 3; ++oj)
          for (int ok2 = 0; ok2 < 3; ++ok2) {
            int n0 = b[0] + oi, n1 = b[1] + oj, n2 = b[2] + ok2;
            if ((n0 >> 2) == bb[0] && (n1 >> 2) == bb[1] && (n2 >> 2) == bb[2])
              mk |= 1ull << (((n0 & 3) << 4) | ((n1 & 3) << 2) | (n2 & 3));
          }
      if (!mk) continue;
      uint32_t r = hash_lookup(h.keys, h.vals, h.mask, pack_key(bb[0], bb[1], bb[2]));
      if (r < h.cap_blocks) atomicOr((unsigned long long*)&nodemask[r], (unsigned long long)mk);
    }
  }
}

__global__ void k_popcount(const uint64_t* __restrict__ masks, const uint32_t* nptr, uint32_t cap,
                           unsigned long long* out) {
  uint32_t n = min(*nptr, cap);
  unsigned long long s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += __popcll(masks[i]);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

}  // namespace

extern "C" {

int smpm_hash_clear(const smpm_hash_desc* h, void* stream) {
  k_hash_clear<<<grid_for(int64_t(h->n_slots)), 256, 0, st(stream)>>>(view(h), h->n_slots);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_hash_insert_many(const smpm_hash_desc* h, const uint64_t* packed, int64_t n, uint32_t* ranks, uint8_t* fresh,
                          void* stream) {
  if (n <= 0) return SMPM_OK;
  k_hash_insert_many<<<grid_for(n), 256, 0, st(stream)>>>(view(h), packed, n, ranks, fresh);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_hash_lookup_many(const smpm_hash_desc* h, const uint64_t* packed, int64_t n, uint32_t* ranks, void* stream) {
  if (n <= 0) return SMPM_OK;
  k_hash_lookup_many<<<grid_for(n), 256, 0, st(stream)>>>(view(h), packed, n, ranks);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_insert_particle_blocks(const smpm_hash_desc* h, const double* x, int64_t n, double inv_h,
                                uint64_t* first_pos, unsigned long long* err, void* stream) {
  if (n <= 0) return SMPM_OK;
  k_insert_particle_blocks<<<grid_for(n), 256, 0, st(stream)>>>(view(h), x, n, inv_h,
                                                               (unsigned long long*)first_pos, err);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_hash_canonicalize(const smpm_hash_desc* h, int mode, const uint64_t* first_pos, void* scratch, void* stream) {
  const uint32_t cap = h->cap_blocks;
  const int ntiles_max = int((cap + RS_TILE - 1) / RS_TILE);
  char* p = (char*)scratch;
  uint64_t* ka = (uint64_t*)p;
  p += size_t(cap) * 8;
  uint64_t* kb = (uint64_t*)p;
  p += size_t(cap) * 8;
  uint32_t* va = (uint32_t*)p;
  p += size_t(cap) * 4;
  uint32_t* vb = (uint32_t*)p;
  p += size_t(cap) * 4;
  uint32_t* hist = (uint32_t*)p;  // 256 * ntiles_max (<= cap/16 words)
  HashView v = view(h);
  cudaStream_t s = st(stream);
  k_canon_prep<<<grid_for(cap), 256, 0, s>>>(v, mode, (const unsigned long long*)first_pos, ka, va);
  const uint32_t* nptr = h->counter;
  int g = std::max(1, std::min(ntiles_max, 148 * 4));
  for (int pass = 0; pass < 8; ++pass) {
    int shift = 8 * pass;
    k_rs_hist<<<g, RS_T, 0, s>>>(ka, nptr, shift, hist, ntiles_max);
    k_rs_scan<<<1, 1024, 0, s>>>(hist, nptr, ntiles_max);
    k_rs_scatter<<<g, RS_T, 0, s>>>(ka, va, kb, vb, nptr, shift, hist, ntiles_max);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  // va: old ranks in canonical order; reuse kb / vb as temporaries
  k_canon_apply<<<grid_for(cap), 256, 0, s>>>(v, va, kb, vb);
  k_canon_write<<<grid_for(cap), 256, 0, s>>>(v, kb, vb);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_hash_active_blocks(const smpm_hash_desc* h, int64_t n_blocks, int32_t* blocks, void* stream) {
  if (n_blocks <= 0) return SMPM_OK;
  k_active_blocks<<<grid_for(n_blocks), 256, 0, st(stream)>>>(h->active_keys, n_blocks, blocks);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_bspline(const double* x, int64_t n, double h, int64_t* base, double* w, double* dw, void* stream) {
  if (n <= 0) return SMPM_OK;
  k_bspline<<<grid_for(n), 256, 0, st(stream)>>>(x, n, 1.0 / h, base, w, dw);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_p2g(const smpm_hash_desc* h, const smpm_stencil_params* sp, int64_t n, const double* x, const double* v,
             const double* C, const double* m, const double* sigma, const double* jac, const double* V0, float* mass,
             float* mom, float* force, unsigned long long* err, void* stream) {
  if (n <= 0) return SMPM_OK;
  k_p2g<<<grid_for(n), 256, 0, st(stream)>>>(view(h), sp->inv_h, sp->h, float(sp->gravity[0]), float(sp->gravity[1]),
                                            float(sp->gravity[2]), n, x, v, C, m, sigma, jac, V0, mass, mom, force,
                                            err);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_grid_update(const smpm_grid_params* g, int64_t n_nodes, float* mass, float* vel, const float* force,
                     const int32_t* active_blocks, void* stream) {
  if (n_nodes <= 0) return SMPM_OK;
  cudaStream_t s = st(stream);
  GridParams gp;
  gp.h = g->h;
  gp.dt = g->dt;
  gp.mass_floor = g->mass_floor;
  for (int a = 0; a < 3; ++a) gp.gravity[a] = g->gravity[a];
  gp.n_bc = g->n_bc;
  Boundary* dbc = nullptr;
  double* dhf = nullptr;
  std::vector<Boundary> hb(std::max(1, g->n_bc));
  for (int i = 0; i < g->n_bc; ++i) {
    hb[i].kind = g->bc[i].kind;
    hb[i].mu = g->bc[i].mu;
    for (int a = 0; a < 3; ++a) {
      hb[i].point[a] = g->bc[i].point[a];
      hb[i].normal[a] = g->bc[i].normal[a];
    }
  }
  CK(cudaMallocAsync(&dbc, hb.size() * sizeof(Boundary), s));
  CK(cudaMemcpyAsync(dbc, hb.data(), hb.size() * sizeof(Boundary), cudaMemcpyHostToDevice, s));
  gp.bc = dbc;
  gp.hf = Heightfield{nullptr, 0, 0, 0, 0, 1};
  if (g->hf_data) {
    size_t nb = size_t(g->hf_nx * g->hf_ny) * 8;
    CK(cudaMallocAsync(&dhf, nb, s));
    CK(cudaMemcpyAsync(dhf, g->hf_data, nb, cudaMemcpyHostToDevice, s));
    gp.hf = Heightfield{dhf, int(g->hf_nx), int(g->hf_ny), g->hf_x0, g->hf_y0, g->hf_cell};
  }
  k_grid_update<<<grid_for(n_nodes), 256, 0, s>>>(gp, n_nodes, mass, vel, force, active_blocks);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));  // host vectors above go out of scope
  CK(cudaFreeAsync(dbc, s));
  if (dhf) CK(cudaFreeAsync(dhf, s));
  return SMPM_OK;
}

int smpm_g2p(const smpm_hash_desc* h, const smpm_stencil_params* sp, double dt, int64_t n, double* x, double* v,
             double* C, double* F, const float* vel, unsigned long long* err, void* stream) {
  if (n <= 0) return SMPM_OK;
  k_g2p<<<grid_for(n), 256, 0, st(stream)>>>(view(h), sp->inv_h, sp->h, dt, n, x, v, C, F, vel, err);
  CK(cudaGetLastError());
  return SMPM_OK;
}

int smpm_stress(const smpm_material* mats, int32_t n_mat, int64_t n, double* F, double* sigma, double* jac,
                const int64_t* mat_id, unsigned long long* err, void* stream) {
  if (n <= 0) return SMPM_OK;
  cudaStream_t s = st(stream);
  std::vector<Material> hm(std::max(1, n_mat));
  for (int i = 0; i < n_mat; ++i) {
    hm[i].mu = float(mats[i].mu);
    hm[i].lam = float(mats[i].lam);
    hm[i].alpha = float(mats[i].alpha);
    hm[i].ratio = float((3.0 * mats[i].lam + 2.0 * mats[i].mu) / (2.0 * mats[i].mu));
    hm[i].kind = mats[i].kind;
  }
  Material* dm = nullptr;
  CK(cudaMallocAsync(&dm, hm.size() * sizeof(Material), s));
  CK(cudaMemcpyAsync(dm, hm.data(), hm.size() * sizeof(Material), cudaMemcpyHostToDevice, s));
  k_stress<<<grid_for(n), 256, 0, s>>>(dm, n_mat, n, F, sigma, jac, mat_id, err);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  CK(cudaFreeAsync(dm, s));
  return SMPM_OK;
}

int smpm_count_active_nodes(const smpm_hash_desc* h, const double* x, int64_t n, double inv_h, uint64_t* nodemask,
                            unsigned long long* err, uint64_t* count_out, void* stream) {
  cudaStream_t s = st(stream);
  int rc = smpm_hash_clear(h, stream);
  if (rc) return rc;
  CK(cudaMemsetAsync(nodemask, 0, size_t(h->cap_blocks) * 8, s));
  k_insert_particle_blocks<<<grid_for(n), 256, 0, s>>>(view(h), x, n, inv_h, nullptr, err);
  k_node_masks<<<grid_for(n), 256, 0, s>>>(view(h), x, n, inv_h, nodemask);
  unsigned long long* dcount = nullptr;
  CK(cudaMallocAsync(&dcount, 8, s));
  CK(cudaMemsetAsync(dcount, 0, 8, s));
  k_popcount<<<grid_for(h->cap_blocks), 256, 0, s>>>(nodemask, h->counter, h->cap_blocks, dcount);
  CK(cudaGetLastError());
  unsigned long long c = 0;
  CK(cudaMemcpyAsync(&c, dcount, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaFreeAsync(dcount, s));
  *count_out = c;
  return SMPM_OK;
}

}  // extern "C"
