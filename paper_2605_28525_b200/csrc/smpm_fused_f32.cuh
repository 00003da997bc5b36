// Fast-mode fused step kernel: G2P -> F -> advection -> next stress -> next
// keys -> next P2G, with the P2G accumulated per cell in registers.
// Included by smpm_sim.cu after k_g2p2g (shares FusedArgs, ItemInfo and the
// helpers); the deterministic mode keeps k_g2p2g (int64 fixed point).
//
// Reference: the P2G it replaces is the fused scatter of
// /root/reference/pkg/src/sparsempm/solver.py:456-575 (per particle, 27 nodes,
// 7 fields, one atomic per field per node).  Here a work item (up to RCAP = 512
// particles of one block, slot-major) runs in three phases, three barriers:
//
//   A   all threads start the next item's velocity-arena prefetch; per
//       particle: G2P from the smem velocity arena, F update, advection,
//       Hencky/DP stress of the next step, record store, next-step keys; the
//       P2G operands (cell offset d, m, v, C, N = -V0 tau / h: 24 floats, laid
//       out so every pair the scatter multiplies is an aligned float2) go to a
//       per-particle stash (the particle's own record stage slot), and the
//       slot is pushed onto its base cell's list (atomicExch on the list head;
//       the first particle of a cell appends the cell to the task list).
//   S   a task = (non-empty base cell, x offset i) walks the cell's list and
//       accumulates its 9 nodes x 7 fields in registers (fp32, packed FFMA2:
//       over k = 0,1 per field, over fields at k = 2), then adds them to the
//       split fixed-point smem arena: ~1/8 of an atomic pair per
//       particle-node-field instead of one.  Warp 7 inserts the item's touched
//       blocks into the next step's table meanwhile.
//   F   flush: bins, cell counts, red.global.add.v4.f32 of the arena nodes;
//       records of the next item are fetched (cp.async) into the stage.
//
// Grid sums carry fp32 precision relative to each node's own magnitude: the
// arena is int32 hi/lo fixed point (2^42 of range) with per-item scales, no
// global scale, no scale replays.

#ifndef SMPM_ABL
#define SMPM_ABL 0  // timing ablations (results wrong): 1 no scatter tasks, 2 no stress, 4 no flush, 8 no gather
#endif
constexpr uint32_t RCAP = 512;   // particles per work item (two per thread)
constexpr int NSTASH = 6;        // float4 per stashed particle
constexpr int NACELL = 216;      // arena base cells (6^3: the block +- 1 cell)
constexpr int TASK_WARPS = 7;    // warps running scatter tasks (warp 7 inserts blocks)
constexpr uint32_t LEND = 0xFFFFu;  // end of a cell list

struct __align__(16) FusedSmemF {
  float4 st[2][NSTASH][CTA];      // per particle slot: record chunks 0..4 (stage), then the P2G stash
  float4 garena[2][GATH_N];       // double-buffered velocity arena
  int ahi[NF][SCAT_N];            // split fixed-point arena (m, p0..2, f0..2): value * S = hi * 2^20 + lo
  int alo[NF][SCAT_N];
  uint32_t kc[SCAT_N];            // cell sums added per arena node (> 0: active; the magic-number bias)
  uint32_t bnd[2][3];             // item maxima of the per-particle contribution bounds (m, p, f), by item parity
  uint32_t cnt[SCAT_N];           // particles binned per arena base cell (next table's cell counts)
  uint32_t head[NACELL];          // list head per arena base cell (stash slot kk * CTA + tid, LEND: empty)
  uint16_t nxt[2 * CTA];          // list link per stash slot
  uint16_t tcell[NACELL];         // non-empty base cells (scatter tasks), in arrival order
  uint32_t ntask;
  uint32_t rank[27];
  uint32_t posr[3][2][CTA];       // sorted positions of the thread's particles (ring: items i, i+1, i+2)
  uint32_t icnt[3][2];            // (particle count, first sorted position) of the ring's blocks
  uint32_t binr[2][CTA];          // bins of the item awaiting its ranks
  ItemInfo info[3];
  Material mats[8];
};

__device__ __forceinline__ float2 f2b(float a) { return make_float2(a, a); }
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}

// Adds the pair x * S to two arena words as hi * 2^20 + lo (four native int32
// reds, no carries: |lo| <= 2^19).  t = x S is an fp32 value below 2^45, so
// both parts are exact (magic-number rounding: h is t / 2^20 rounded to an
// integer, kept below 2^22 by the scale choice; L = t - 2^20 H is exact in an
// FFMA and rounded to an integer by the second magic).  Both words are biased
// by MAGIC_BITS; the flush removes the bias with the count kc.
__device__ __forceinline__ void arena_add_pair(int* hi0, int* lo0, int* hi1, int* lo1, float2 x, float2 S) {
  const float2 t = __fmul2_rn(x, S);
  const float2 h = __ffma2_rn(t, f2b(9.5367431640625e-07f), f2b(MAGIC));  // 2^-20
  const float2 hf = __fadd2_rn(h, f2b(-MAGIC));
  const float2 l = __fadd2_rn(__ffma2_rn(hf, f2b(-1048576.0f), t), f2b(MAGIC));
  sred(hi0, __float_as_int(h.x));
  sred(hi1, __float_as_int(h.y));
  sred(lo0, __float_as_int(l.x));
  sred(lo1, __float_as_int(l.y));
}
// Power-of-two item scale for contribution bound b (bits of a non-negative
// float): S = 2^(32-e) for b in [2^e, 2^(e+1)), so a cell sum of <= RCAP = 2^9
// bounds times S stays below 2^42; iS = 1/S exactly.  b = 0: S = 1.
__device__ __forceinline__ void item_scale(uint32_t bbits, float& S, float& iS) {
  const int e = bbits ? int((bbits >> 23) & 0xFFu) - 127 : 32;
  const int s = max(-100, min(100, 32 - e));
  S = __uint_as_float(uint32_t(127 + s) << 23);
  iS = __uint_as_float(uint32_t(127 - s) << 23);
}
__device__ __forceinline__ void arena_add_one(int* hi, int* lo, float x, float S) {
  const float t = x * S;
  const float h = fmaf(t, 9.5367431640625e-07f, MAGIC);
  const float hf = h - MAGIC;
  const float l = fmaf(-hf, 1048576.0f, t) + MAGIC;
  sred(hi, __float_as_int(h));
  sred(lo, __float_as_int(l));
}

template <bool GATHER, int CV>
__global__ void __launch_bounds__(CTA, SMPM_MINB) k_g2p2g_f32(FusedArgs A) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smraw[];
  FusedSmemF& sm = *reinterpret_cast<FusedSmemF*>(smraw);
  if (*A.B.halt) return;  // a batched step that must not run (smpm_sim_run)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < A.n_mat && i < 8; i += CTA) sm.mats[i] = A.mats[i];
  const uint32_t n_items = A.stB->n_items;
  const double dt = GATHER ? A.stB->dt : 0.0;
  const float ih = A.ihf;
  const float hf_ = A.hf;
  uint32_t vmax2_local = 0;
  {
    int* zh = &sm.ahi[0][0];
    int* zl = &sm.alo[0][0];
    for (int i = tid; i < NF * SCAT_N; i += CTA) zh[i] = zl[i] = 0;
    if (tid < 6) sm.bnd[tid / 3][tid % 3] = 0;
    for (int i = tid; i < SCAT_N; i += CTA) {
      sm.kc[i] = 0;
      sm.cnt[i] = 0;
    }
    for (int i = tid; i < NACELL; i += CTA) sm.head[i] = LEND;
    if (tid == 0) {
      sm.ntask = 0;
    }
  }
  // sorted positions of the thread's particles of an item: slot-major ranges
  // of RCAP (k_bin's wide placement), positions first + t and first + 256 + t
  // (count, start): the block's particle count and first sorted position (the
  // level table's block start, k_scan2), from icnt[ring]
  auto slots = [&](const ItemInfo& inf, int ring) {
    const uint32_t cnt = sm.icnt[ring][0], start = sm.icnt[ring][1];
    const uint32_t first = inf.g() * RCAP;
    const uint32_t n = inf.r() != BAD_KEY && cnt > first ? min(cnt - first, RCAP) : 0u;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t j = CTA * kk + tid;
      sm.posr[ring][kk][tid] = j < n ? start + first + j : NOPOS;
    }
  };
  // ---- prime: metadata of items 0..2, neighbour ranks of items 0 and 1,
  // positions of items 0 and 1, records and velocity arena of item 0
  if (tid == 0) fetch_item(A, n_items, 0, sm.info[0], false);
  if (tid == 1) fetch_item(A, n_items, 1, sm.info[1], false);
  if (tid == 2) fetch_item(A, n_items, 2, sm.info[2], false);
  __syncthreads();
  uint32_t src1a = 0, src1b = 0;  // storage indices of item i+1's particles
  {
    const ItemInfo& i0 = sm.info[0];
    const ItemInfo& i1 = sm.info[1];
    if (GATHER && tid < 8 && i0.r() != BAD_KEY) sm.info[0].nbr[tid] = A.B.nbr8[size_t(i0.r()) * 8 + tid];
    if (GATHER && tid >= 8 && tid < 16 && i1.r() != BAD_KEY)
      sm.info[1].nbr[tid - 8] = A.B.nbr8[size_t(i1.r()) * 8 + tid - 8];
    if (tid >= 16 && tid < 18) {
      const ItemInfo& ii = sm.info[tid - 16];
      if (ii.r() != BAD_KEY) {
        sm.icnt[tid - 16][0] = A.B.block_total[ii.r()];
        sm.icnt[tid - 16][1] = A.B.cell_off[size_t(ii.r()) * 64 + 32];
      }
    }
  }
  __syncthreads();
  {
    slots(sm.info[0], 0);
    if (GATHER) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint32_t ps = sm.posr[0][kk][tid];
        if (ps != NOPOS) {
          const float4* g = A.src.rec + size_t(A.perm[ps]) * 8;
#pragma unroll
          for (int q = 0; q < GCH; ++q) cp_async16(&sm.st[kk][q][tid], &g[q]);
        }
      }
    }
  }
  __syncthreads();
  if (GATHER && sm.info[0].r() != BAD_KEY) prefetch_arena(sm.garena[0], A, sm.info[0], tid, CTA);
  cp_async_commit();
  int buf = 0, c = 0;
  uint32_t kf = 3;  // schedule index of the next item to fetch

  while (true) {
    cp_async_wait_all();
    __syncthreads();  // [B1] records and velocity arena of item i landed; item i-1 flushed
    const ItemInfo& cur = sm.info[c];
    const int c1r = c == 2 ? 0 : c + 1, c2r = c == 0 ? 2 : c - 1;
    const ItemInfo& nxt = sm.info[c1r];
    const ItemInfo& nn = sm.info[c2r];
    if (cur.r() == BAD_KEY) break;
    int B0, B1, B2;
    cur.block(B0, B1, B2);
    // velocity arena of item i+1 (its neighbour ranks arrived with item i-1's
    // flush), sorted positions and source indices of its particles (consumed
    // by this item's flush)
    if (GATHER && nxt.r() != BAD_KEY) prefetch_arena(sm.garena[buf ^ 1], A, nxt, tid, CTA);
    cp_async_commit();
    slots(nxt, c1r);
    {
      const uint32_t pa = sm.posr[c1r][0][tid], pb = sm.posr[c1r][1][tid];
      src1a = pa != NOPOS ? A.perm[pa] : 0u;
      src1b = pb != NOPOS ? A.perm[pb] : 0u;
    }
    float bmx[3] = {0.f, 0.f, 0.f};  // contribution bounds of the thread's stashed particles

    // ================================================================ A
#pragma unroll 1
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t pos = sm.posr[c][kk][tid];
      const bool valid = pos != NOPOS;
      float4 c0, c1, c2, c3, c4, c5, c6, c7;
      if (valid) {
        if (GATHER) {
          c0 = sm.st[kk][0][tid];
          c1 = sm.st[kk][1][tid];
          c2 = sm.st[kk][2][tid];
          c3 = sm.st[kk][3][tid];
          c4 = sm.st[kk][4][tid];
        } else {
          const float4* g = A.src.rec + size_t(A.perm[pos]) * 8;
          c0 = g[0];
          c1 = g[1];
          c2 = g[2];
          c3 = g[3];
          c4 = g[4];
          c5 = g[5];
          c6 = g[6];
          c7 = g[7];
        }
      }
      uint32_t binv = BIN_SKIP;
      if (valid) {
        double xn[3];
        float vn[3], Cn[9], M[6], d1[3];
        int nb[3], ab[3];
        bool ok = true, far = false;
        int mig = -1;
        xn[0] = __hiloint2double(__float_as_int(c0.y), __float_as_int(c0.x));
        xn[1] = __hiloint2double(__float_as_int(c0.w), __float_as_int(c0.z));
        xn[2] = __hiloint2double(__float_as_int(c1.y), __float_as_int(c1.x));
        const float m = c1.z;
        const float V0 = c1.w;
        float F[9] = {c2.x, c2.y, c2.z, c2.w, c3.x, c3.y, c3.z, c3.w, c4.x};
        const uint32_t pm = __float_as_uint(c4.y);
        const uint32_t pidv = pm & PID_MASK;
        const int mt = int(pm >> 29);
        if (GATHER && !(SMPM_ABL & 8)) {
          // ---- G2P (solver.py:628-732), as k_g2p2g
          int lb[3];
          float d[3], w[3][3], g[3][3];
          const int Bb[3] = {B0, B1, B2};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            int bs;
            axis_base(xn[a], A.inv_h, bs, d[a]);
            lb[a] = bs - 4 * Bb[a];
            bspline(d[a], w[a], g[a]);
          }
          const float4* ga = sm.garena[buf];
          float2 Pz[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) Pz[k] = make_float2(w[2][k], w[2][k] * (float(k) - d[2]));
          float2 P0[3], GW0[3], W1D[3];
#pragma unroll
          for (int o = 0; o < 3; ++o) {
            P0[o] = make_float2(w[0][o], w[0][o] * (float(o) - d[0]));
            GW0[o] = make_float2(g[0][o], w[0][o]);
            W1D[o] = make_float2(w[1][o], w[1][o] * (float(o) - d[1]));
          }
          const float2 Z2 = make_float2(0.f, 0.f);
          float2 Vxy = Z2, Bx = Z2, By = Z2, Bz = Z2, Ax2 = Z2, Ay2 = Z2, Az2 = Z2;
          float2 VB = Z2, AB = Z2, BA = Z2;
          float a21 = 0.f;
#pragma unroll
          for (int oi = 0; oi < 3; ++oi) {
#pragma unroll
            for (int oj = 0; oj < 3; ++oj) {
              float2 Sxy = Z2, Txy = Z2, Uxy = Z2, TU2 = Z2;
              float S2 = 0.f;
              const int gi = lb[0] + oi, gj = lb[1] + oj;
#pragma unroll
              for (int ok = 0; ok < 3; ++ok) {
                const float4 q = ga[gaddr(gi, gj, lb[2] + ok)];
                const float2 qxy = make_float2(q.x, q.y);
                Sxy = __ffma2_rn(qxy, make_float2(Pz[ok].x, Pz[ok].x), Sxy);
                Txy = __ffma2_rn(qxy, make_float2(Pz[ok].y, Pz[ok].y), Txy);
                Uxy = __ffma2_rn(qxy, make_float2(g[2][ok], g[2][ok]), Uxy);
                TU2 = __ffma2_rn(make_float2(q.z, q.z), make_float2(Pz[ok].y, g[2][ok]), TU2);
                S2 = fmaf(q.z, Pz[ok].x, S2);
              }
              const float2 WD = __fmul2_rn(P0[oi], make_float2(w[1][oj], w[1][oj]));
              const float2 AD = __fmul2_rn(GW0[oi], W1D[oj]);
              const float wij = WD.x, Ay = w[0][oi] * g[1][oj];
              Vxy = __ffma2_rn(Sxy, make_float2(wij, wij), Vxy);
              Bx = __ffma2_rn(Sxy, make_float2(WD.y, WD.y), Bx);
              By = __ffma2_rn(Sxy, make_float2(AD.y, AD.y), By);
              Bz = __ffma2_rn(Txy, make_float2(wij, wij), Bz);
              Ax2 = __ffma2_rn(Sxy, make_float2(AD.x, AD.x), Ax2);
              Ay2 = __ffma2_rn(Sxy, make_float2(Ay, Ay), Ay2);
              Az2 = __ffma2_rn(Uxy, make_float2(wij, wij), Az2);
              VB = __ffma2_rn(make_float2(S2, S2), WD, VB);
              AB = __ffma2_rn(make_float2(S2, S2), AD, AB);
              BA = __ffma2_rn(TU2, make_float2(wij, wij), BA);
              a21 = fmaf(Ay, S2, a21);
            }
          }
          const float cs = 4.0f * ih;
          Cn[0] = Bx.x * cs;
          Cn[1] = By.x * cs;
          Cn[2] = Bz.x * cs;
          Cn[3] = Bx.y * cs;
          Cn[4] = By.y * cs;
          Cn[5] = Bz.y * cs;
          Cn[6] = VB.y * cs;
          Cn[7] = AB.y * cs;
          Cn[8] = BA.x * cs;
          vn[0] = Vxy.x;
          vn[1] = Vxy.y;
          vn[2] = VB.x;
          const float dth = float(dt) * ih;
          float A9[9] = {Ax2.x * dth, Ay2.x * dth, Az2.x * dth, Ax2.y * dth, Ay2.y * dth,
                         Az2.y * dth, AB.x * dth,  a21 * dth,   BA.y * dth};
          float Fn[9];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
              Fn[3 * i + j] =
                  F[3 * i + j] + (A9[3 * i + j] + (A9[3 * i] * F[j] + A9[3 * i + 1] * F[3 + j] + A9[3 * i + 2] * F[6 + j]));
#pragma unroll
          for (int q = 0; q < 9; ++q) F[q] = Fn[q];
          xn[0] = __dadd_rn(xn[0], __dmul_rn(dt, double(vn[0])));
          xn[1] = __dadd_rn(xn[1], __dmul_rn(dt, double(vn[1])));
          xn[2] = __dadd_rn(xn[2], __dmul_rn(dt, double(vn[2])));
        } else if (SMPM_ABL & 8) {
          vn[0] = vn[1] = vn[2] = 0.f;
          for (int q = 0; q < 9; ++q) Cn[q] = 0.f;
        } else {
          vn[0] = c4.z;
          vn[1] = c4.w;
          vn[2] = c5.x;
          Cn[0] = c5.y;
          Cn[1] = c5.z;
          Cn[2] = c5.w;
          Cn[3] = c6.x;
          Cn[4] = c6.y;
          Cn[5] = c6.z;
          Cn[6] = c6.w;
          Cn[7] = c7.x;
          Cn[8] = c7.y;
        }
        // ---- stress of the next step (materials.py:169-238)
        float tau[6], J;
        const Material& mat = sm.mats[mt];
        if (SMPM_ABL & 2) {
          tau[0] = F[0] * mat.mu; tau[1] = F[4] * mat.mu; tau[2] = F[8] * mat.mu; tau[3] = tau[4] = tau[5] = 0.f;
        } else if (!hencky_dp<CV>(F, mat, A.project != 0, tau, J)) {
          err_report(A.err, ERR_DEGENERATE_F, pidv);
          ok = false;
          tau[0] = tau[1] = tau[2] = tau[3] = tau[4] = tau[5] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) M[q] = V0 * tau[q];
        {  // ---- the particle record at its sorted position
          float4* o = A.dst.rec + size_t(pos) * 8;
          int2 x0 = make_int2(__double2loint(xn[0]), __double2hiint(xn[0]));
          int2 x1 = make_int2(__double2loint(xn[1]), __double2hiint(xn[1]));
          int2 x2 = make_int2(__double2loint(xn[2]), __double2hiint(xn[2]));
          o[0] = make_float4(__int_as_float(x0.x), __int_as_float(x0.y), __int_as_float(x1.x), __int_as_float(x1.y));
          o[1] = make_float4(__int_as_float(x2.x), __int_as_float(x2.y), m, V0);
          o[2] = make_float4(F[0], F[1], F[2], F[3]);
          o[3] = make_float4(F[4], F[5], F[6], F[7]);
          o[4] = make_float4(F[8], __uint_as_float(pm), vn[0], vn[1]);
          o[5] = make_float4(vn[2], Cn[0], Cn[1], Cn[2]);
          o[6] = make_float4(Cn[3], Cn[4], Cn[5], Cn[6]);
          o[7] = make_float4(Cn[7], Cn[8], 0.f, 0.f);
        }
        const float vv = vn[0] * vn[0] + vn[1] * vn[1] + vn[2] * vn[2];
        vmax2_local = max(vmax2_local, __float_as_uint(vv));
        // ---- next step's keys
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (!isfinite(xn[a])) {
            if (ok) err_report(A.err, ERR_NONFINITE_X, pidv);
            ok = false;
          } else if (!axis_base(xn[a], A.inv_h, nb[a], d1[a]) || !axis_in_key_range(nb[a])) {
            if (ok) err_report(A.err, ERR_KEY_RANGE, pidv);
            ok = false;
          }
        }
        if (ok) {
          ab[0] = nb[0] - (4 * B0 - 1);
          ab[1] = nb[1] - (4 * B1 - 1);
          ab[2] = nb[2] - (4 * B2 - 1);
          far = ab[0] < 0 || ab[0] > 5 || ab[1] < 0 || ab[1] > 5 || ab[2] < 0 || ab[2] > 5;
          const int nbx = nb[0] >> 2;
          mig = nbx < A.bx0 ? 0 : (nbx >= A.bx1 ? 1 : -1);
          if (mig >= 0) {
            // leaves this rank's slab: scattered here, binned by the neighbour
            const uint32_t slot = atomicAdd(&A.mig_count[mig], 1u);
            if (slot < A.mig_cap) {
              const float4* src4 = A.dst.rec + size_t(pos) * 8;
              float4* o4 = A.mig[mig] + size_t(slot) * 8;
#pragma unroll
              for (int c8 = 0; c8 < 8; ++c8) o4[c8] = src4[c8];
            } else {
              err_report(A.err, ERR_CAPACITY, pidv);
            }
          }
        }
        if (ok && !far) {
          // ---- stash the P2G operands (this slot's record stage is consumed):
          // pairs the scatter multiplies sit in aligned float2 halves
          //   s0 (dx, dy, dz, m)  s1 (v0, v1, C00, C10)  s2 (v2, C20, C01, C11)
          //   s3 (C02, C12, C21, C22)  s4 (N00, N01, N01, N11)  s5 (N02, N12, N22, -)
          // with C row-major and N = -M / h (M = V0 tau symmetric: xx yy zz xy xz yz)
          const uint32_t ci = uint32_t((ab[0] * 6 + ab[1]) * 6 + ab[2]);
          const float nh = -ih;
          sm.st[kk][0][tid] = make_float4(d1[0], d1[1], d1[2], m);
          sm.st[kk][1][tid] = make_float4(vn[0], vn[1], Cn[0], Cn[3]);
          sm.st[kk][2][tid] = make_float4(vn[2], Cn[6], Cn[1], Cn[4]);
          sm.st[kk][3][tid] = make_float4(Cn[2], Cn[5], Cn[7], Cn[8]);
          sm.st[kk][4][tid] = make_float4(M[0] * nh, M[3] * nh, M[3] * nh, M[1] * nh);
          sm.st[kk][5][tid] = make_float4(M[4] * nh, M[5] * nh, M[2] * nh, 0.f);
          const uint32_t slot = uint32_t(kk * CTA + tid);
          const uint32_t prev = atomicExch(&sm.head[ci], slot);
          sm.nxt[slot] = uint16_t(prev);
          if (prev == LEND) sm.tcell[atomicAdd(&sm.ntask, 1u)] = uint16_t(ci);
          // contribution bounds, worst case over the cell offset (|w| <= 0.75^3,
          // |dx_a| <= 1.5 h, |grad w_a| <= 0.75^2 / h): the item's fixed-point scales
          // (coarse: the split arena has 2^42 of range, the bound only keeps
          // the cell sums inside it)
          float cm = 0.f, fm = 0.f, cs = 0.f;
#pragma unroll
          for (int a = 0; a < 9; ++a) cs += fabsf(Cn[a]);
#pragma unroll
          for (int a = 0; a < 6; ++a) fm += fabsf(M[a]);
          cm = fmaxf(fmaxf(fabsf(vn[0]), fabsf(vn[1])), fabsf(vn[2])) + (1.5f * hf_) * cs;
          bmx[0] = fmaxf(bmx[0], m * 0.421875f);
          bmx[1] = fmaxf(bmx[1], m * 0.421875f * cm);
          bmx[2] = fmaxf(bmx[2], fm * 0.5625f * ih);
          if (mig < 0) {
            atomicAdd(&sm.cnt[aaddr(ab[0], ab[1], ab[2])], 1u);
            binv = BIN_ARENA | uint32_t((ab[0] << 6) | (ab[1] << 3) | ab[2]);
          } else {
            binv = MIG_KEY;
          }
        } else if (ok && far) {
          scatter_global(A, nb, d1, m, vn, Cn, M, binv, mig < 0, 1.f, 1.f, 1.f);
        } else {
          binv = BAD_KEY;
        }
      }
      sm.binr[kk][tid] = valid ? binv : BIN_SKIP;
    }
    {
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const uint32_t b = __reduce_max_sync(0xffffffffu, __float_as_uint(bmx[f]));
        if (lane == 0 && b) atomicMax(&sm.bnd[buf][f], b);
      }
    }
    __syncthreads();  // [B2] stash, cell lists, touched blocks and bounds of item i

    // ================================================================ S
    if (warp < TASK_WARPS) {
      const uint32_t nt = (SMPM_ABL & 1) ? 0u : sm.ntask;
      float Sg[3], iSg;
#pragma unroll
      for (int f = 0; f < 3; ++f) item_scale(sm.bnd[buf][f], Sg[f], iSg);
#pragma unroll 1
      for (uint32_t t = tid; t < 3 * nt; t += TASK_WARPS * 32) {
        const uint32_t oi = t / nt;
        const uint32_t cc = sm.tcell[t - oi * nt];
        const int a0 = int(cc / 36), a1 = int((cc / 6) % 6), a2 = int(cc % 6);
        // x weight of offset oi as a function of dx: t = dx - xc, w = wa + wb t^2, g = wg t
        const float4 xw = A.xw[oi];
        const float xc = xw.x, wa = xw.y, wb = xw.z, wg = xw.w;
        const float oih = float(oi) * hf_;
        // node (oi, j, k) accumulators: k = 0, 1 packed per field; k = 2
        // packed over fields: (m, p2), (p0, p1), (f0, f1), f2
        const float2 Z2 = make_float2(0.f, 0.f);
        float2 m01[3], p01[3][3], f01[3][3], mp2[3], pp2[3], ff2[3];
        float f22[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          m01[j] = mp2[j] = pp2[j] = ff2[j] = Z2;
          f22[j] = 0.f;
#pragma unroll
          for (int a = 0; a < 3; ++a) p01[a][j] = f01[a][j] = Z2;
        }
        uint32_t sl = sm.head[cc];
#pragma unroll 1
        while (sl != LEND) {
          const float4* sp = &sm.st[sl >> 8][0][sl & (CTA - 1)];
          sl = sm.nxt[sl];
          const float4 s0 = sp[0], s1 = sp[CTA], s2 = sp[2 * CTA], s3 = sp[3 * CTA], s4 = sp[4 * CTA],
                       s5 = sp[5 * CTA];
          const float tx = s0.x - xc;
          const float wx = fmaf(wb, tx * tx, wa), gx = wg * tx;
          float wy[3], gy[3], wz[3], gz[3];
          bspline(s0.y, wy, gy);
          bspline(s0.z, wz, gz);
          // momentum m w (v + C dx), dx = h (o - d): per node
          //   wz_k R_a(j) + wz_k tz_k T_a(j), R_a = W (u_a + C_a1 ty_j), T_a = W C_a2,
          //   u_a = v_a + C_a0 tx, W = m wx wy_j;
          // force N grad w (N = -M / h, grad in cell units): per node
          //   wz_k P_a(j) + gz_k Q_a(j), P_a = N_a0 gx wy_j + N_a1 wx gy_j, Q_a = N_a2 wx wy_j
          const float txh = fmaf(-s0.x, hf_, oih);
          const float2 u01 = __ffma2_rn(make_float2(s1.z, s1.w), f2b(txh), make_float2(s1.x, s1.y));
          const float u2 = fmaf(s2.y, txh, s2.x);
          const float X = s0.w * wx;
          const float2 MG01 = __fmul2_rn(make_float2(s4.x, s4.y), f2b(gx));
          const float2 MW01 = __fmul2_rn(make_float2(s4.z, s4.w), f2b(wx));
          const float2 MQ01 = __fmul2_rn(make_float2(s5.x, s5.y), f2b(wx));
          const float MG2 = s5.x * gx, MW2 = s5.y * wx, MQ2 = s5.z * wx;
          const float tz0 = -s0.z * hf_;
          const float2 z1 = make_float2(wz[0], wz[1]);
          const float2 z2 = __fmul2_rn(z1, make_float2(tz0, tz0 + hf_));
          const float z22 = wz[2] * (tz0 + 2.0f * hf_);
          const float2 gz01 = make_float2(gz[0], gz[1]);
          const float ty0 = -s0.y * hf_;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const float tyh = ty0 + float(j) * hf_;
            const float W = X * wy[j];
            const float2 R01 = __fmul2_rn(__ffma2_rn(make_float2(s2.z, s2.w), f2b(tyh), u01), f2b(W));
            const float2 WR2 = make_float2(W, W * fmaf(s3.z, tyh, u2));
            const float2 T01 = __fmul2_rn(make_float2(s3.x, s3.y), f2b(W));
            const float T2 = W * s3.w;
            const float2 P01 = __ffma2_rn(MG01, f2b(wy[j]), __fmul2_rn(MW01, f2b(gy[j])));
            const float P2 = fmaf(MG2, wy[j], MW2 * gy[j]);
            const float2 Q01 = __fmul2_rn(MQ01, f2b(wy[j]));
            const float Q2 = MQ2 * wy[j];
            m01[j] = __ffma2_rn(z1, f2b(W), m01[j]);
            p01[0][j] = __ffma2_rn(z2, f2b(T01.x), __ffma2_rn(z1, f2b(R01.x), p01[0][j]));
            p01[1][j] = __ffma2_rn(z2, f2b(T01.y), __ffma2_rn(z1, f2b(R01.y), p01[1][j]));
            p01[2][j] = __ffma2_rn(z2, f2b(T2), __ffma2_rn(z1, f2b(WR2.y), p01[2][j]));
            f01[0][j] = __ffma2_rn(gz01, f2b(Q01.x), __ffma2_rn(z1, f2b(P01.x), f01[0][j]));
            f01[1][j] = __ffma2_rn(gz01, f2b(Q01.y), __ffma2_rn(z1, f2b(P01.y), f01[1][j]));
            f01[2][j] = __ffma2_rn(gz01, f2b(Q2), __ffma2_rn(z1, f2b(P2), f01[2][j]));
            mp2[j] = __ffma2_rn(WR2, f2b(wz[2]), mp2[j]);
            mp2[j].y = fmaf(T2, z22, mp2[j].y);
            pp2[j] = __ffma2_rn(T01, f2b(z22), __ffma2_rn(R01, f2b(wz[2]), pp2[j]));
            ff2[j] = __ffma2_rn(Q01, f2b(gz[2]), __ffma2_rn(P01, f2b(wz[2]), ff2[j]));
            f22[j] = fmaf(Q2, gz[2], fmaf(P2, wz[2], f22[j]));
          }
        }
        // add the task's 9 nodes to the arena (fixed point, the item's scales:
        // a cell sum is at most RCAP bounds, kept below 2^42), and K
        const float2 Smm = f2b(Sg[0]), Spp = f2b(Sg[1]), Sff = f2b(Sg[2]), Smp = make_float2(Sg[0], Sg[1]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int d0 = aaddr(a0 + int(oi), a1 + j, a2), d1 = d0 + 1, d2 = d0 + 2;
          arena_add_pair(&sm.ahi[0][d0], &sm.alo[0][d0], &sm.ahi[0][d1], &sm.alo[0][d1], m01[j], Smm);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            arena_add_pair(&sm.ahi[1 + a][d0], &sm.alo[1 + a][d0], &sm.ahi[1 + a][d1], &sm.alo[1 + a][d1], p01[a][j],
                           Spp);
            arena_add_pair(&sm.ahi[4 + a][d0], &sm.alo[4 + a][d0], &sm.ahi[4 + a][d1], &sm.alo[4 + a][d1], f01[a][j],
                           Sff);
          }
          arena_add_pair(&sm.ahi[0][d2], &sm.alo[0][d2], &sm.ahi[3][d2], &sm.alo[3][d2], mp2[j], Smp);
          arena_add_pair(&sm.ahi[1][d2], &sm.alo[1][d2], &sm.ahi[2][d2], &sm.alo[2][d2], pp2[j], Spp);
          arena_add_pair(&sm.ahi[4][d2], &sm.alo[4][d2], &sm.ahi[5][d2], &sm.alo[5][d2], ff2[j], Sff);
          arena_add_one(&sm.ahi[6][d2], &sm.alo[6][d2], f22[j], Sg[2]);
          atomicAdd(&sm.kc[d0], 1u);
          atomicAdd(&sm.kc[d1], 1u);
          atomicAdd(&sm.kc[d2], 1u);
        }
      }
    } else {
      // warp 7: the blocks the item's stencils touch (from its non-empty base
      // cells), inserted into the next step's table
      const uint32_t nt = sm.ntask;
      uint32_t tm = 0;
      for (uint32_t e = lane; e < nt; e += 32) {
        const uint32_t cc = sm.tcell[e];
        tm |= touched27(axis_blocks(int(cc / 36)), axis_blocks(int((cc / 6) % 6)), axis_blocks(int(cc % 6)));
      }
      tm = __reduce_or_sync(0xffffffffu, tm);
      if (lane < 27) {
        uint32_t rk = BAD_KEY;
        if ((tm >> lane) & 1u) {
          const int di = lane / 9 - 1, dj = (lane / 3) % 3 - 1, dk = lane % 3 - 1;
          // dense backend: a stencil node outside the declared domain (solver.py:1053-1058)
          if (B0 + di < A.dbox_lo[0] || B0 + di > A.dbox_hi[0] || B1 + dj < A.dbox_lo[1] ||
              B1 + dj > A.dbox_hi[1] || B2 + dk < A.dbox_lo[2] || B2 + dk > A.dbox_hi[2])
            err_report(A.err, ERR_INACTIVE, 0);
          rk = hash_insert(A.S.hv, pack_key(B0 + di, B1 + dj, B2 + dk));
          if (rk >= A.S.hv.cap_blocks) rk = BAD_KEY;
        }
        sm.rank[lane] = rk;
      }
    }
    __syncthreads();  // [B3] arena and ranks of item i complete; the stash is free

    // ================================================================ F
    // records of item i+1 into the stage (overlaps the flush)
    if (GATHER) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        if (sm.posr[c1r][kk][tid] != NOPOS) {
          const float4* g = A.src.rec + size_t(kk ? src1b : src1a) * 8;
#pragma unroll
          for (int q = 0; q < GCH; ++q) cp_async16(&sm.st[kk][q][tid], &g[q]);
        }
      }
    }
    if (tid == 0) fetch_item(A, n_items, kf, sm.info[c], true);  // item i+3 -> this item's ring slot
    // neighbour ranks and particle range of item i+2 (used from item i+1's start)
    if (nn.r() != BAD_KEY) {
      if (GATHER && tid >= 32 && tid < 34)
        cp_async16(&sm.info[c2r].nbr[4 * (tid - 32)], A.B.nbr8 + size_t(nn.r()) * 8 + 4 * (tid - 32));
      if (tid == 34) cp_async4(&sm.icnt[c2r][0], A.B.block_total + nn.r());
      if (tid == 35) cp_async4(&sm.icnt[c2r][1], A.B.cell_off + size_t(nn.r()) * 64 + 32);
    }
    cp_async_commit();
    // bins of item i (positions from ring slot c)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t bv = sm.binr[kk][tid];
      if (bv == BIN_SKIP) continue;
      uint32_t out = bv;
      if (bv >= BIN_ARENA && bv < BIN_ARENA + 512u) {
        const int q0 = int((bv >> 6) & 7u), q1 = int((bv >> 3) & 7u), q2 = int(bv & 7u);
        const uint32_t rk = sm.rank[((q0 + 3) >> 2) * 9 + ((q1 + 3) >> 2) * 3 + ((q2 + 3) >> 2)];
        const uint32_t lc = (((q0 + 3) & 3) << 4) | (((q1 + 3) & 3) << 2) | ((q2 + 3) & 3);
        out = rk == BAD_KEY ? OVF_KEY : rk * 64 + lc;
      }
      A.bin_out[sm.posr[c][kk][tid]] = out;
    }
    for (int nd = tid; nd < 216; nd += CTA) {
      const int i = nd / 36, j = (nd / 6) % 6, k = nd % 6;
      const int ad = aaddr(i, j, k);
      const uint32_t cc = sm.cnt[ad];
      if (cc) {
        sm.cnt[ad] = 0;
        const uint32_t rq2 = sm.rank[((i + 3) >> 2) * 9 + ((j + 3) >> 2) * 3 + ((k + 3) >> 2)];
        const uint32_t lc = (((i + 3) & 3) << 4) | (((j + 3) & 3) << 2) | ((k + 3) & 3);
        if (rq2 != BAD_KEY) atomicAdd(&A.S.cell_count[rq2 * 64 + lc], cc);
      }
      sm.head[nd] = LEND;
    }
    float iS[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      float S_;
      item_scale(sm.bnd[buf][f], S_, iS[f]);
    }
    if (tid < 3) sm.bnd[buf ^ 1][tid] = 0;  // the next item's (item i-1 is done with them)
    for (int nd = tid; nd < 512; nd += CTA) {
      const int i = nd >> 6, j = (nd >> 3) & 7, k = nd & 7;
      const int ad = aaddr(i, j, k);
      const uint32_t K = sm.kc[ad];
      if (!K || (SMPM_ABL & 4)) continue;
      float vals[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int bias = int(K * MAGIC_BITS);  // mod 2^32: the true sums fit in int32
        vals[f] = fmaf(float(sm.ahi[f][ad] - bias), 1048576.0f, float(sm.alo[f][ad] - bias)) *
                  iS[f == 0 ? 0 : (f < 4 ? 1 : 2)];
        sm.ahi[f][ad] = 0;
        sm.alo[f][ad] = 0;
      }
      sm.kc[ad] = 0;
      const uint32_t rk = sm.rank[((i + 3) >> 2) * 9 + ((j + 3) >> 2) * 3 + ((k + 3) >> 2)];
      if (rk == BAD_KEY) continue;
      const size_t node = size_t(rk) * 64 + ((((i + 3) & 3) << 4) | (((j + 3) & 3) << 2) | ((k + 3) & 3));
      red_v4(&A.acc[2 * node], vals[0], vals[1], vals[2], vals[3]);
      red_v4(&A.acc[2 * node + 1], vals[4], vals[5], vals[6], float(K));  // .w > 0: active node (n_active)
    }
    if (tid == 0) sm.ntask = 0;
    ++kf;
    buf ^= 1;
    c = c1r;
  }
  vmax2_local = __reduce_max_sync(0xffffffffu, vmax2_local);
  if (lane == 0 && vmax2_local) atomicMax(&A.stS->vmax2_bits, vmax2_local);
  if (blockIdx.x == 0 && tid < 3) A.stS->scale_inv[tid] = 0.f;  // fp32-grade arena: no global fixed-point scales
}
