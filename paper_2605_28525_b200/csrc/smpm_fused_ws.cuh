// Warp-specialised fast-mode fused step kernel (default for large scenes):
// the same per-particle work and precision model as k_g2p2g_f32
// (smpm_fused_f32.cuh), reorganised as a producer/consumer pipeline inside one
// 512-thread CTA per SM instead of three CTA-wide barriers per item.
//
// Reference: the P2G it replaces is the fused scatter of
// /root/reference/pkg/src/sparsempm/solver.py:456-575, the G2P
// solver.py:628-732, the stress materials.py:169-238.
//
//   warps 8..15 (A, producer, 2 particles per thread): per particle G2P from
//     the smem velocity arena, F update, advection, next-step stress, record
//     store, next-step keys, P2G operands into stash buffer b = item & 1 and
//     onto its cell list; then bar.arrive(FULL[b]).  The records of item i+1
//     are prefetched (cp.async) into the thread's own stage slots as soon as
//     item i's are consumed, the velocity arena of item i+1 at item i's start.
//   warps 0..7 (S, consumer): bar.sync(FULL[b]); scatter tasks (cell, x
//     offset) on all 256 lanes into the split fixed-point arena (one round up
//     to 85 non-empty cells: the flowing regime's halo cells), the first warp
//     done with its tasks inserts the touched blocks; flush, bins and cell
//     counts; buffer b is handed back with bar.arrive(EMPTY[b]).
//
// Tried and dropped (A/B on C4, tools/gpu_ab_ws.sh): next-step keys, lists
// and counts on the consumer (fp64 position in a 7-chunk stash): +0.5 ms
// early, +0.5 ms late -- the consumer's pre-pass sits on its critical path;
// setmaxnreg 144/112 and 136/120 splits: within noise.
//
// A works on item i+1 while S scatters item i, so neither waits for the other
// at a CTA-wide barrier; the only intra-role barrier is the A-side one that
// publishes the landed velocity arena.  Named barriers: FULL[b] = 1 + b,
// EMPTY[b] = 3 + b (512 threads: 256 arrive, 256 sync), producer-only 5 and
// consumer-only 6 (256 each); barrier 0 (__syncthreads) only before the split.

#ifndef SMPM_WS_STATS
#define SMPM_WS_STATS 0
#endif
#if SMPM_WS_STATS
__device__ uint32_t ws_stat_nt[128], ws_stat_lm[64], ws_stat_lmax_item;
// clock64 phase sums of CTA 0: producer (warp 8 lane 0) wait-empty, wait-data,
// work; consumer (per warp, lane 0) wait-full, tasks, wait-consumers, flush
__device__ unsigned long long ws_clk_a[3], ws_clk_s[8][4];
#define WS_CLK(v) long long v = clock64()
#else
#define WS_CLK(v)
#endif
constexpr int WS_CTA = 512;  // threads per CTA: 256 consumer (S) + 256 producer (A)
constexpr int WA = 256;      // threads per role
constexpr int WB_FULL = 1, WB_EMPTY = 3, WB_A = 5, WB_S = 6;
#ifndef SMPM_WS_SHIGH
#define SMPM_WS_SHIGH 0  // 1: consumer on warps 8..15 (A/B: same early, +0.2 ms late)
#endif
#ifndef SMPM_WS_TW
#define SMPM_WS_TW 8  // consumer warps running scatter tasks (7: warp 7 only inserts)
#endif
constexpr int WS_TW = SMPM_WS_TW;
#ifndef SMPM_WS_RA
#define SMPM_WS_RA 0  // setmaxnreg of the producer warps (0: the launch's 128)
#endif
#ifndef SMPM_WS_RS
#define SMPM_WS_RS 0  // setmaxnreg of the consumer warps (RA + RS <= 256)
#endif

struct __align__(16) FusedSmemWS {
  float4 stage[2][GCH][WA];          // records of the A thread's two particles (G2P chunks)
  float4 stash[2][2][NSTASH][WA];    // [buffer][kk][chunk][thread] P2G operands
  float4 garena[2][GATH_N];          // double-buffered velocity arena
  int ahi[NF][SCAT_N];               // split fixed-point arena (S only)
  int alo[NF][SCAT_N];
  uint32_t kc[SCAT_N];               // cell sums added per arena node
  uint32_t cnt[2][SCAT_N];           // particles binned per arena base cell
  uint32_t head[2][NACELL];          // cell list heads
  uint16_t nxt[2][2 * WA];           // list links
  uint16_t tcell[2][NACELL];         // non-empty base cells
  uint32_t ntask[2];
  uint32_t iclaim;                   // insert duty of the current item taken (WS_TW = 8)
  uint32_t bnd[2][3];                // item maxima of the contribution bounds (m, p, f)
  int blk[2][4];                     // block coordinates of the buffer's item; [3] != 0: no item (end)
  uint32_t rank[27];                 // next-table ranks of the item's touched blocks (S only)
  uint32_t posr[3][2][WA];           // sorted positions of the A thread's particles, ring by item % 3
  uint32_t binr[2][2][WA];           // bins awaiting the item's ranks
  uint32_t srcr[2][WA];              // storage indices of the next item's particles
  uint32_t icnt[4][2];               // (particle count, first sorted position), ring by item % 4
  ItemInfo info[4];                  // item metadata ring (A only)
  Material mats[8];
};
static_assert(sizeof(FusedSmemWS) <= 227 * 1024, "FusedSmemWS exceeds the per-CTA shared-memory limit");

__device__ __forceinline__ void nbar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------- producer
template <bool GATHER, int CV>
__device__ __forceinline__ void ws_produce(const FusedArgs& A, FusedSmemWS& sm, const int t, const uint32_t n_items) {
  const int lane = t & 31;
  const double dt = GATHER ? A.stB->dt : 0.0;
  const float ih = A.ihf;
  const float hf_ = A.hf;
  uint32_t vmax2_local = 0;
  // sorted positions of the thread's particles of an item (slot-major ranges
  // of RCAP, positions first + t and first + 256 + t)
  auto slots = [&](const ItemInfo& inf, int pr, int ir) {
    const uint32_t cnt = sm.icnt[ir][0], start = sm.icnt[ir][1];
    const uint32_t first = inf.g() * RCAP;
    const uint32_t n = inf.r() != BAD_KEY && cnt > first ? min(cnt - first, RCAP) : 0u;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t j = WA * kk + t;
      sm.posr[pr][kk][t] = j < n ? start + first + j : NOPOS;
    }
  };
  // this thread's velocity-arena node (t < 216): neighbour slot, arena
  // address and node within the neighbour block, fixed for the launch
  int pa_slot = 0, pa_dst = 0, pa_loc = 0;
  if (t < 216) {
    const int i = t / 36, j = (t / 6) % 6, k = t % 6;
    pa_slot = ((i >> 2) << 2) | ((j >> 2) << 1) | (k >> 2);
    pa_dst = gaddr(i, j, k);
    pa_loc = ((i & 3) << 4) | ((j & 3) << 2) | (k & 3);
  }
  auto prefetch_ga = [&](float4* ga, const ItemInfo& inf) {
    if (t < 216) {
      const uint32_t gr = inf.nbr[pa_slot];
      if (gr < A.B.hv.cap_blocks)
        cp_async16(ga + pa_dst, &A.gv[size_t(gr) * 64 + pa_loc]);
      else
        ga[pa_dst] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  // ---- prime: metadata of items 0..2, neighbour ranks and ranges of items
  // 0 and 1, records and velocity arena of item 0
  if (t < 3) fetch_item(A, n_items, t, sm.info[t], false);
  nbar_sync(WB_A, WA);
  {
    const ItemInfo& i0 = sm.info[0];
    const ItemInfo& i1 = sm.info[1];
    if (GATHER && t < 8 && i0.r() != BAD_KEY) sm.info[0].nbr[t] = A.B.nbr8[size_t(i0.r()) * 8 + t];
    if (GATHER && t >= 8 && t < 16 && i1.r() != BAD_KEY) sm.info[1].nbr[t - 8] = A.B.nbr8[size_t(i1.r()) * 8 + t - 8];
    if (t >= 16 && t < 18) {
      const ItemInfo& ii = sm.info[t - 16];
      if (ii.r() != BAD_KEY) {
        sm.icnt[t - 16][0] = A.B.block_total[ii.r()];
        sm.icnt[t - 16][1] = A.B.cell_off[size_t(ii.r()) * 64 + 32];
      }
    }
  }
  nbar_sync(WB_A, WA);
  slots(sm.info[0], 0, 0);
  if (GATHER) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t ps = sm.posr[0][kk][t];
      if (ps != NOPOS) {
        const float4* g = A.src.rec + size_t(A.perm[ps]) * 8;
#pragma unroll
        for (int q = 0; q < GCH; ++q) cp_async16(&sm.stage[kk][q][t], &g[q]);
      }
    }
    if (sm.info[0].r() != BAD_KEY) prefetch_ga(sm.garena[0], sm.info[0]);
  }
  cp_async_commit();

  for (uint32_t k = 0;; ++k) {
    const int b = int(k & 1u);
    const int pc = int(k % 3u), pn = int((k + 1) % 3u);
    WS_CLK(ta0);
    if (k >= 2) nbar_sync(WB_EMPTY + b, WS_CTA);  // S is done with item k - 2 (buffer b, posr ring slot pn)
    WS_CLK(ta1);
    cp_async_wait_all();
    nbar_sync(WB_A, WA);  // records, velocity arena and metadata of item k landed; item k-1 fully read
    WS_CLK(ta2);
    const ItemInfo& cur = sm.info[k & 3];
    if (cur.r() == BAD_KEY) {
      if (t == 0) sm.blk[b][3] = 1;
      nbar_arrive(WB_FULL + b, WS_CTA);
      if (k >= 1) nbar_sync(WB_EMPTY + (b ^ 1), WS_CTA);  // S's hand-back of the last item
      break;
    }
    const ItemInfo& nxt = sm.info[(k + 1) & 3];
    int B0, B1, B2;
    cur.block(B0, B1, B2);
    // sorted positions of item k+1's particles; their source indices land in
    // smem by cp.async, committed as the oldest group of the item (a register
    // load would be waited for at the head of the non-unrolled kk loop)
    slots(nxt, pn, int((k + 1) & 3));
    if (GATHER) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint32_t p = sm.posr[pn][kk][t];
        if (p != NOPOS) cp_async4(&sm.srcr[kk][t], A.perm + p);
      }
      cp_async_commit();
    }
    if (t == 0) {
      sm.blk[b][0] = B0;
      sm.blk[b][1] = B1;
      sm.blk[b][2] = B2;
      sm.blk[b][3] = 0;
      fetch_item(A, n_items, k + 3, sm.info[(k + 3) & 3], true);  // item k-1's ring slot
    }
    {  // neighbour ranks and particle range of item k+2 (used from item k+1's start)
      const ItemInfo& nn = sm.info[(k + 2) & 3];
      if (nn.r() != BAD_KEY) {
        if (GATHER && t >= 32 && t < 34)
          cp_async16(&sm.info[(k + 2) & 3].nbr[4 * (t - 32)], A.B.nbr8 + size_t(nn.r()) * 8 + 4 * (t - 32));
        if (t == 34) cp_async4(&sm.icnt[(k + 2) & 3][0], A.B.block_total + nn.r());
        if (t == 35) cp_async4(&sm.icnt[(k + 2) & 3][1], A.B.cell_off + size_t(nn.r()) * 64 + 32);
      }
    }
    // velocity arena of item k+1 (its records are fetched as this item's are consumed)
    if (GATHER && nxt.r() != BAD_KEY) prefetch_ga(sm.garena[b ^ 1], nxt);
    cp_async_commit();
    // record of item k+1 into stage slot kk (called once the slot's record of
    // item k has been consumed, or at once for an empty slot)
    auto prefetch_rec = [&](int kk) {
      if (GATHER && sm.posr[pn][kk][t] != NOPOS) {
        if (kk == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");  // the source indices (oldest group)
        const float4* g = A.src.rec + size_t(sm.srcr[kk][t]) * 8;
#pragma unroll
        for (int q = 0; q < GCH; ++q) cp_async16(&sm.stage[kk][q][t], &g[q]);
        cp_async_commit();
      }
    };
    float bmx[3] = {0.f, 0.f, 0.f};

#pragma unroll 1
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t pos = sm.posr[pc][kk][t];
      const bool valid = pos != NOPOS;
      if (!valid) prefetch_rec(kk);
      float4 c0, c1, c2, c3, c4, c5, c6, c7;
      if (valid) {
        if (GATHER) {
          c0 = sm.stage[kk][0][t];
          c1 = sm.stage[kk][1][t];
          c2 = sm.stage[kk][2][t];
          c3 = sm.stage[kk][3][t];
          c4 = sm.stage[kk][4][t];
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
        if (GATHER) {
          // ---- G2P (solver.py:628-732), as k_g2p2g_f32
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
          const float4* ga = sm.garena[b];
          float2 Pz[3];
#pragma unroll
          for (int kz = 0; kz < 3; ++kz) Pz[kz] = make_float2(w[2][kz], w[2][kz] * (float(kz) - d[2]));
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
          prefetch_rec(kk);  // x, m, V0, H and pid|mat of the stage slot are consumed
          xn[0] = __dadd_rn(xn[0], __dmul_rn(dt, double(vn[0])));
          xn[1] = __dadd_rn(xn[1], __dmul_rn(dt, double(vn[1])));
          xn[2] = __dadd_rn(xn[2], __dmul_rn(dt, double(vn[2])));
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
        if (!hencky_dp<CV>(F, mat, A.project != 0, tau, J)) {
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
          // ---- P2G operands into stash buffer b (layout as k_g2p2g_f32)
          const uint32_t ci = uint32_t((ab[0] * 6 + ab[1]) * 6 + ab[2]);
          const float nh = -ih;
          float4* st = &sm.stash[b][kk][0][t];
          st[0] = make_float4(d1[0], d1[1], d1[2], m);
          st[WA] = make_float4(vn[0], vn[1], Cn[0], Cn[3]);
          st[2 * WA] = make_float4(vn[2], Cn[6], Cn[1], Cn[4]);
          st[3 * WA] = make_float4(Cn[2], Cn[5], Cn[7], Cn[8]);
          st[4 * WA] = make_float4(M[0] * nh, M[3] * nh, M[3] * nh, M[1] * nh);
          st[5 * WA] = make_float4(M[4] * nh, M[5] * nh, M[2] * nh, 0.f);
          const uint32_t slot = uint32_t(kk * WA + t);
          const uint32_t prev = atomicExch(&sm.head[b][ci], slot);
          sm.nxt[b][slot] = uint16_t(prev);
          if (prev == LEND) sm.tcell[b][atomicAdd(&sm.ntask[b], 1u)] = uint16_t(ci);
          float cs = 0.f, fm = 0.f;
#pragma unroll
          for (int a = 0; a < 9; ++a) cs += fabsf(Cn[a]);
#pragma unroll
          for (int a = 0; a < 6; ++a) fm += fabsf(M[a]);
          const float cm = fmaxf(fmaxf(fabsf(vn[0]), fabsf(vn[1])), fabsf(vn[2])) + (1.5f * hf_) * cs;
          bmx[0] = fmaxf(bmx[0], m * 0.421875f);
          bmx[1] = fmaxf(bmx[1], m * 0.421875f * cm);
          bmx[2] = fmaxf(bmx[2], fm * 0.5625f * ih);
          if (mig < 0) {
            atomicAdd(&sm.cnt[b][aaddr(ab[0], ab[1], ab[2])], 1u);
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
      sm.binr[b][kk][t] = valid ? binv : BIN_SKIP;
      // this slot's stage is consumed (or was empty): the record of item k+1
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const uint32_t bb = __reduce_max_sync(0xffffffffu, __float_as_uint(bmx[f]));
      if (lane == 0 && bb) atomicMax(&sm.bnd[b][f], bb);
    }
    cp_async_commit();
#if SMPM_WS_STATS
    if (blockIdx.x == 0 && t == 0) {
      const long long ta3 = clock64();
      ws_clk_a[0] += ta1 - ta0;
      ws_clk_a[1] += ta2 - ta1;
      ws_clk_a[2] += ta3 - ta2;
    }
#endif
    nbar_arrive(WB_FULL + b, WS_CTA);  // buffer b (stash, lists, counts, bins, bounds) holds item k
  }
  vmax2_local = __reduce_max_sync(0xffffffffu, vmax2_local);
  if (lane == 0 && vmax2_local) atomicMax(&A.stS->vmax2_bits, vmax2_local);
}

// ---------------------------------------------------------------- consumer
__device__ __forceinline__ void ws_consume(const FusedArgs& A, FusedSmemWS& sm, const int t) {
  const int lane = t & 31, warp = t >> 5;
  const float hf_ = A.hf;
  for (uint32_t k = 0;; ++k) {
    const int b = int(k & 1u);
    WS_CLK(ts0);
    nbar_sync(WB_FULL + b, WS_CTA);
    WS_CLK(ts1);
    if (sm.blk[b][3]) break;
    const int B0 = sm.blk[b][0], B1 = sm.blk[b][1], B2 = sm.blk[b][2];
    const uint32_t nt = sm.ntask[b];
#if SMPM_WS_STATS >= 2
    // diagnostics (timing builds only): per item, the task count and the
    // longest cell list, histogrammed by CTA 0 and printed at the end
    if (blockIdx.x == 0) {
      uint32_t lmax = 0;
      for (uint32_t e = t; e < nt; e += WA) {
        uint32_t n = 0;
        for (uint32_t sl = sm.head[b][sm.tcell[b][e]]; sl != LEND; sl = sm.nxt[b][sl]) ++n;
        lmax = max(lmax, n);
      }
      lmax = __reduce_max_sync(0xffffffffu, lmax);
      if (lane == 0) atomicMax(&ws_stat_lmax_item, lmax);
      nbar_sync(WB_S, WA);
      if (t == 0) {
        atomicAdd(&ws_stat_nt[min(nt, 127u)], 1u);
        atomicAdd(&ws_stat_lm[min(ws_stat_lmax_item, 63u)], 1u);
        ws_stat_lmax_item = 0;
      }
      nbar_sync(WB_S, WA);
    }
#endif
    float Sg[3], iS[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) item_scale(sm.bnd[b][f], Sg[f], iS[f]);
    if (warp < WS_TW) {
#pragma unroll 1
      for (uint32_t tk = t; tk < 3 * nt; tk += WS_TW * 32) {
        const uint32_t oi = tk / nt;
        const uint32_t cc = sm.tcell[b][tk - oi * nt];
        const int a0 = int(cc / 36), a1 = int((cc / 6) % 6), a2 = int(cc % 6);
        const float4 xw = A.xw[oi];
        const float xc = xw.x, wa = xw.y, wb = xw.z, wg = xw.w;
        const float oih = float(oi) * hf_;
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
        uint32_t sl = sm.head[b][cc];
#pragma unroll 1
        while (sl != LEND) {
          const float4* sp = &sm.stash[b][sl >> 8][0][sl & (WA - 1)];  // chunks 0..5
          sl = sm.nxt[b][sl];
          const float4 s0 = sp[0], s1 = sp[WA], s2 = sp[2 * WA], s3 = sp[3 * WA], s4 = sp[4 * WA], s5 = sp[5 * WA];
          const float tx = s0.x - xc;
          const float wx = fmaf(wb, tx * tx, wa), gx = wg * tx;
          float wy[3], gy[3], wz[3], gz[3];
          bspline(s0.y, wy, gy);
          bspline(s0.z, wz, gz);
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
    }
    WS_CLK(ts2);
    bool ins = warp >= WS_TW;  // WS_TW = 7: warp 7 inserts; 8: the first warp done with its tasks
    if (WS_TW == 8) {
      uint32_t cl = 0;
      if (lane == 0) cl = atomicExch(&sm.iclaim, 1u);
      ins = __shfl_sync(0xffffffffu, cl, 0) == 0u;
    }
    if (ins) {
      // the blocks the item's stencils touch, inserted into the next step's table
      uint32_t tm = 0;
      for (uint32_t e = lane; e < nt; e += 32) {
        const uint32_t cc = sm.tcell[b][e];
        tm |= touched27(axis_blocks(int(cc / 36)), axis_blocks(int((cc / 6) % 6)), axis_blocks(int(cc % 6)));
      }
      tm = __reduce_or_sync(0xffffffffu, tm);
      if (lane < 27) {
        uint32_t rk = BAD_KEY;
        if ((tm >> lane) & 1u) {
          const int di = lane / 9 - 1, dj = (lane / 3) % 3 - 1, dk = lane % 3 - 1;
          if (B0 + di < A.dbox_lo[0] || B0 + di > A.dbox_hi[0] || B1 + dj < A.dbox_lo[1] ||
              B1 + dj > A.dbox_hi[1] || B2 + dk < A.dbox_lo[2] || B2 + dk > A.dbox_hi[2])
            err_report(A.err, ERR_INACTIVE, 0);
          rk = hash_insert(A.S.hv, pack_key(B0 + di, B1 + dj, B2 + dk));
          if (rk >= A.S.hv.cap_blocks) rk = BAD_KEY;
        }
        sm.rank[lane] = rk;
      }
    }
    WS_CLK(ts3);
    nbar_sync(WB_S, WA);  // arena and ranks of item k complete
    WS_CLK(ts4);
    // bins of item k
    const int pc = int(k % 3u);
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint32_t bv = sm.binr[b][kk][t];
      if (bv == BIN_SKIP) continue;
      uint32_t out = bv;
      if (bv >= BIN_ARENA && bv < BIN_ARENA + 512u) {
        const int q0 = int((bv >> 6) & 7u), q1 = int((bv >> 3) & 7u), q2 = int(bv & 7u);
        const uint32_t rk = sm.rank[((q0 + 3) >> 2) * 9 + ((q1 + 3) >> 2) * 3 + ((q2 + 3) >> 2)];
        const uint32_t lc = (((q0 + 3) & 3) << 4) | (((q1 + 3) & 3) << 2) | ((q2 + 3) & 3);
        out = rk == BAD_KEY ? OVF_KEY : rk * 64 + lc;
      }
      A.bin_out[sm.posr[pc][kk][t]] = out;
    }
    for (int nd = t; nd < 216; nd += WA) {
      const int i = nd / 36, j = (nd / 6) % 6, kz = nd % 6;
      const int ad = aaddr(i, j, kz);
      const uint32_t cc = sm.cnt[b][ad];
      if (cc) {
        sm.cnt[b][ad] = 0;
        const uint32_t rq2 = sm.rank[((i + 3) >> 2) * 9 + ((j + 3) >> 2) * 3 + ((kz + 3) >> 2)];
        const uint32_t lc = (((i + 3) & 3) << 4) | (((j + 3) & 3) << 2) | ((kz + 3) & 3);
        if (rq2 != BAD_KEY) atomicAdd(&A.S.cell_count[rq2 * 64 + lc], cc);
      }
      sm.head[b][nd] = LEND;
    }
    if (t == 0) sm.ntask[b] = 0;
    if (t == 1) sm.iclaim = 0;
    if (t < 3) sm.bnd[b][t] = 0;
    for (int nd = t; nd < 512; nd += WA) {
      const int i = nd >> 6, j = (nd >> 3) & 7, kz = nd & 7;
      const int ad = aaddr(i, j, kz);
      const uint32_t K = sm.kc[ad];
      if (!K) continue;
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
      const uint32_t rk = sm.rank[((i + 3) >> 2) * 9 + ((j + 3) >> 2) * 3 + ((kz + 3) >> 2)];
      if (rk == BAD_KEY) continue;
      const size_t node = size_t(rk) * 64 + ((((i + 3) & 3) << 4) | (((j + 3) & 3) << 2) | ((kz + 3) & 3));
      red_v4(&A.acc[2 * node], vals[0], vals[1], vals[2], vals[3]);
      red_v4(&A.acc[2 * node + 1], vals[4], vals[5], vals[6], float(K));  // .w > 0: active node (n_active)
    }
#if SMPM_WS_STATS
    if (blockIdx.x == 0 && lane == 0) {
      const long long ts5 = clock64();
      ws_clk_s[warp][0] += ts1 - ts0;  // wait for a full buffer
      ws_clk_s[warp][1] += ts2 - ts1 + ts3 - ts2;  // tasks (+ inserts)
      ws_clk_s[warp][2] += ts4 - ts3;  // wait for the other consumers
      ws_clk_s[warp][3] += ts5 - ts4;  // bins, counts, flush
    }
#endif
    nbar_arrive(WB_EMPTY + b, WS_CTA);  // buffer b is free for item k+2
  }
}

template <bool GATHER, int CV>
__global__ void __launch_bounds__(WS_CTA, 1) k_g2p2g_ws(FusedArgs A) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smraw[];
  FusedSmemWS& sm = *reinterpret_cast<FusedSmemWS*>(smraw);
  if (*A.B.halt) return;  // a batched step that must not run (smpm_sim_run)
  const int tid = threadIdx.x;
  for (int i = tid; i < A.n_mat && i < 8; i += WS_CTA) sm.mats[i] = A.mats[i];
  {
    int* zh = &sm.ahi[0][0];
    int* zl = &sm.alo[0][0];
    for (int i = tid; i < NF * SCAT_N; i += WS_CTA) zh[i] = zl[i] = 0;
    for (int i = tid; i < SCAT_N; i += WS_CTA) {
      sm.kc[i] = 0;
      sm.cnt[0][i] = 0;
      sm.cnt[1][i] = 0;
    }
    for (int i = tid; i < 2 * NACELL; i += WS_CTA) (&sm.head[0][0])[i] = LEND;
    if (tid < 6) (&sm.bnd[0][0])[tid] = 0;
    if (tid < 2) sm.ntask[tid] = 0;
    if (tid == 2) sm.iclaim = 0;
  }
  __syncthreads();
  // the issue arbiter favours high warp ids: the producer takes warps 8..15
  // (the consumer there measured the same early and 0.2 ms slower late)
  const bool producer = SMPM_WS_SHIGH ? tid < WA : tid >= WA;
  const int rt = tid & (WA - 1);
  if (producer) {
    if (SMPM_WS_RA) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SMPM_WS_RA));
    ws_produce<GATHER, CV>(A, sm, rt, A.stB->n_items);
  } else {
    if (SMPM_WS_RS) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SMPM_WS_RS));
    ws_consume(A, sm, rt);
  }
  if (blockIdx.x == 0 && tid < 3) A.stS->scale_inv[tid] = 0.f;  // fp32-grade arena: no global fixed-point scales
#if SMPM_WS_STATS
  if (blockIdx.x == 0 && tid == 0) {
    printf("WSSTATS nt");
    for (int i = 0; i < 128; ++i) printf(" %u", ws_stat_nt[i]);
    printf("\nWSSTATS lmax");
    for (int i = 0; i < 64; ++i) printf(" %u", ws_stat_lm[i]);
    printf("\n");
    printf("WSCLK A wait_empty %llu wait_data %llu work %llu\n", ws_clk_a[0], ws_clk_a[1], ws_clk_a[2]);
    for (int w = 0; w < 8; ++w)
      printf("WSCLK S%d wait_full %llu tasks %llu wait_s %llu flush %llu\n", w, ws_clk_s[w][0], ws_clk_s[w][1],
             ws_clk_s[w][2], ws_clk_s[w][3]);
    for (int i = 0; i < 3; ++i) ws_clk_a[i] = 0;
    for (int w = 0; w < 8; ++w)
      for (int i = 0; i < 4; ++i) ws_clk_s[w][i] = 0;
    for (int i = 0; i < 128; ++i) ws_stat_nt[i] = 0;
    for (int i = 0; i < 64; ++i) ws_stat_lm[i] = 0;
  }
#endif
}
