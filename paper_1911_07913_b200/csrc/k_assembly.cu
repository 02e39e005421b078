// Level-0 system matrix H = M + dt^2 d2Phi/dx2 on B200 (objective.hpp:318-363).
//
// Stage 1 (one thread per particle): virtual F -> SVD -> dP/dF projected in the diagonal
//   space -> one 1008-byte record per particle: the 27 W_k = F^nT grad w_k, then kappa*T as
//   its 45 unique entries (hot_particle.cuh: kRecW, kRecT, tslot).
// Stage 2 (one warp per row, rows from a work counter): gather over the 27 neighbouring
//   particle bins, records staged by the bulk-copy engine, the per-particle rank-3 block
//   updates on the fp64 tensor cores (DMMA), accumulated into the row's upper-triangle slots
//   in shared memory (fixed order, no atomics).  Each unordered block pair is computed once by
//   the row with the smaller index and written together with its transpose, so block (i,j) ==
//   block(j,i)^T exactly (the reference's symmetry_error() == 0 invariant).  The mass diagonal
//   and the Dirichlet projection (objective.hpp:133-144) are fused into the write-out.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "hot_async.cuh"
#include "hot_internal.h"
#include "hot_particle.cuh"

namespace hotb200 {

namespace {

constexpr int kAsmWarps = 4;
constexpr int kUpper = 63;  // slots 62..124

/// Per particle (bin order) one record of kRecStride doubles (1008 B = 63 x 16 B): W (27 x 3),
/// W_k = F^nT grad w_k (0 where w_k = 0), then kappa*T's 45 unique entries (T is symmetric).
constexpr int kTPacked = 45;
constexpr int kTensorStride = kRecStride;

/// Records are written through a per-warp shared-memory transpose: each lane computes its
/// particle's values, then the warp writes the 32 records part by part, consecutive lanes on
/// consecutive addresses (a thread-per-particle store pattern puts every lane on its own line).
constexpr int kTWarps = 4;
template <int MINB>
__global__ void __launch_bounds__(kTWarps * 32, MINB) k_particle_tensors(ParticlesView P, GridView g, double dx, double dt,
                                                                   const DevMaterial* __restrict__ mats,
                                                                   const double* __restrict__ u,
                                                                   const double* __restrict__ svd_in, int project,
                                                                   double* __restrict__ Tu, int* bad, long long plo,
                                                                   long long phi) {
  __shared__ double stage[kTWarps][32][kTPacked];
  const long long n = P.n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nchunks = (phi - plo + 31) / 32;
  for (long long ch = blockIdx.x * (long long)kTWarps + wib; ch < nchunks; ch += (long long)gridDim.x * kTWarps) {
    const long long p = plo + ch * 32 + lane;
    if (p < phi) {
      const int mat = __ldg(P.mat + p);
      const double vol = __ldg(P.vol + p);
      M3 U, V, Fn;
      double s[3];
      bool ok = true;
      if (svd_in) {  // SVD of the virtual F at this dv, stored by the energy evaluation
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          U.m[k] = __ldg(svd_in + k * n + p);
          V.m[k] = __ldg(svd_in + (12 + k) * n + p);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) s[k] = __ldg(svd_in + (9 + k) * n + p);
      } else {
        M3 F;
        ok = virtual_F(P, p, g, dx, dt, u, F, Fn);
        if (ok) svd3(F, U, s, V);
        else atomicExch(bad, 1);
      }
      if (ok) {
        const DevMaterial mt = mats[mat];
        double T[45];
        fcr_dpdf_projected(U, s, V, mt.mu, mt.lambda, dt * dt * vol, project != 0, T);
#pragma unroll
        for (int q = 0; q < kTPacked; ++q) stage[wib][lane][tperm(q)] = T[q];  // T slot tslot(r, c)
      }
    }
    __syncwarp();
    const int cnt = (int)min(32LL, phi - plo - ch * 32);
    for (int t = 0; t < cnt; ++t) {
      double* out = Tu + (plo + ch * 32 + t) * kTensorStride + kRecT;
      out[lane] = stage[wib][t][lane];
      if (lane < kTPacked - 32) out[32 + lane] = stage[wib][t][32 + lane];
    }
    __syncwarp();
  }
}

/// The record's W part: W_k = F^nT grad w_k for the 27 stencil nodes (grid.hpp:58-73,
/// objective.hpp:337-339); nodes with zero weight get W = 0, which is how the reference skips
/// them (transfer.hpp:36-37).  A separate light kernel (the T kernel is register bound).
constexpr int kWWarps = 4;
__global__ void __launch_bounds__(kWWarps * 32) k_particle_W(ParticlesView P, double dx, double* __restrict__ Tu, long long plo,
                                                             long long phi) {
  __shared__ double stage[kWWarps][32][27 + 1];  // one x-plane (9 positions) of the warp's 32 records
  const long long n = P.n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nchunks = (phi - plo + 31) / 32;
  for (long long ch = blockIdx.x * (long long)kWWarps + wib; ch < nchunks; ch += (long long)gridDim.x * kWWarps) {
    const long long p = plo + ch * 32 + lane;
    const bool live = p < phi;
    double Fn[9];
    Axis3 ax[3];
    if (live) {
      double xs[3];
#pragma unroll
      for (int k = 0; k < 9; ++k) Fn[k] = __ldg(P.F + k * n + p);
#pragma unroll
      for (int a = 0; a < 3; ++a) xs[a] = __ldg(P.x + a * n + p);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double c = xs[a] / dx;
        axis_weights(c, stencil_base_1d(c), ax[a]);
        axis_dw_over_dx(ax[a], dx);
      }
    }
    const int cnt = (int)min(32LL, phi - plo - ch * 32);
#pragma unroll 1
    for (int k0 = 0; k0 < 3; ++k0) {
      if (live) {
        const double w0 = k0 == 0 ? ax[0].w[0] : (k0 == 1 ? ax[0].w[1] : ax[0].w[2]);
        const double dw0 = k0 == 0 ? ax[0].dw[0] : (k0 == 1 ? ax[0].dw[1] : ax[0].dw[2]);
#pragma unroll
        for (int kk = 0; kk < 9; ++kk) {
          const int k1 = kk / 3, k2 = kk % 3;
          const double w1 = ax[1].w[k1], w2 = ax[2].w[k2];
          double W[3] = {0.0, 0.0, 0.0};
          if (w0 * w1 * w2 > 0.0) {
            const double g0 = dw0 * w1 * w2, g1 = ax[1].dw[k1] * w0 * w2, g2 = ax[2].dw[k2] * w0 * w1;
#pragma unroll
            for (int q = 0; q < 3; ++q) W[q] = Fn[q] * g0 + Fn[3 + q] * g1 + Fn[6 + q] * g2;
          }
#pragma unroll
          for (int q = 0; q < 3; ++q) stage[wib][lane][3 * kk + q] = W[q];
        }
      }
      __syncwarp();
      for (int t = 0; t < cnt; ++t)
        if (lane < 27) Tu[(plo + ch * 32 + t) * kTensorStride + kRecW + 27 * k0 + lane] = stage[wib][t][lane];
      __syncwarp();
    }
  }
}

__global__ void k_fill_cols(LevelView L, int* __restrict__ cols, unsigned long long* __restrict__ active) {
  const int R = L.radius, P = level_pitch(R), S = level_slots(R), W = 2 * R + 1;
  unsigned long long cnt = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)L.n * P;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / P), s = (int)(t % P);
    int c = -1;
    if (s < S)
      c = dense_lookup(L.map, L.coords[3 * i] + s / (W * W) - R, L.coords[3 * i + 1] + (s / W) % W - R,
                       L.coords[3 * i + 2] + s % W - R);
    cols[t] = c;
    cnt += c >= 0 ? 1 : 0;
  }
  // active-slot count of the level (algorithmic bytes of the profile), one atomic per warp
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(active, cnt);
}

/// Row gather (objective.hpp:331-357), one warp per row i.  A particle p of a bin whose stencil
/// holds i at position a contributes to the row's upper-triangle block at stencil position k
///   C_k[c][e] += sum_g W_k[g] M[c][e][g],   M[c][e][g] = sum_f W_a[f] T[(3c+f),(3e+g)].
/// Per particle that is a rank-3 update of the (upper positions) x (ce) block, which runs on the
/// fp64 tensor cores (DMMA m8n8k4): M-dim = upper positions (tiles of 8), N-dim = ce 0..7, K = g
/// (3, padded to 4 with a zero row of B).  The ninth column ce = 8 would waste a whole second
/// N tile, so it goes to the FMA pipe instead: each lane accumulates A[k][g] * M[8][g] and the
/// four g lanes are summed once per bin pair.  Every lane computes its own B-fragment entry
/// M[ce][g] (3 FMA from the staged T and W_a), so M never goes through shared memory.
///
/// Bin offset o and its mirror 26-o are walked together (their upper position counts add up to
/// 28), both bins' particles staged by the bulk-copy engine (one cp.async.bulk per bin chunk,
/// mbarrier completion, double buffered one chunk ahead).  The tile counts of a pair are
/// template constants, so the per-particle loop has no tile branches.  Each (pair, lane) block
/// accumulates in registers and is folded into the row's shared accumulator once per pair (bin
/// o's lanes, then the mirror's: fixed order, no atomics).
// CH particles per bin per stage; AW warps per CTA (4 x 2, launch_assemble_rows)
template <int CH>
constexpr int asm_stage() { return 2 * CH * kTensorStride; }  // doubles: [bin of pair][particle][...]
template <int CH>
constexpr int asm_warp_doubles() { return 2 * asm_stage<CH>() + kUpper * 9 + 1 + 2 + 28; }  // + pad + 2 mbarriers + pair table
template <int AW, int CH>
constexpr int asm_smem() { return AW * asm_warp_doubles<CH>() * 8; }
constexpr unsigned kParticleBytes = kTensorStride * 8;  // 1008 = 63 x 16
static_assert(asm_warp_doubles<1>() % 2 == 0 && asm_warp_doubles<2>() % 2 == 0 && asm_warp_doubles<3>() % 2 == 0,
              "16-byte aligned per-warp smem");

/// S(o) = 25 o0 + 5 o1 + o2 of a stencil position, and kmin(o): the first stencil position k of
/// the bin at offset o whose slot S(k) + S(o) is in the row's upper triangle (>= 62).
struct Kmin27 {
  int S[27], kmin[27];
  constexpr Kmin27() : S(), kmin() {
    for (int o = 0; o < 27; ++o) S[o] = 25 * (o / 9) + 5 * ((o / 3) % 3) + o % 3;
    for (int o = 0; o < 27; ++o) {
      int k = 0;
      while (k < 27 && S[k] + S[o] < kDiagSlot) ++k;
      kmin[o] = k;
    }
  }
};
constexpr Kmin27 kKmin27{};
__constant__ int c_S27[27] = {
#define HOT_S(o) (25 * ((o) / 9) + 5 * (((o) / 3) % 3) + (o) % 3)
    HOT_S(0),  HOT_S(1),  HOT_S(2),  HOT_S(3),  HOT_S(4),  HOT_S(5),  HOT_S(6),  HOT_S(7),  HOT_S(8),
    HOT_S(9),  HOT_S(10), HOT_S(11), HOT_S(12), HOT_S(13), HOT_S(14), HOT_S(15), HOT_S(16), HOT_S(17),
    HOT_S(18), HOT_S(19), HOT_S(20), HOT_S(21), HOT_S(22), HOT_S(23), HOT_S(24), HOT_S(25), HOT_S(26)};
#undef HOT_S
__constant__ int c_kmin27[27] = {
    kKmin27.kmin[0],  kKmin27.kmin[1],  kKmin27.kmin[2],  kKmin27.kmin[3],  kKmin27.kmin[4],  kKmin27.kmin[5],
    kKmin27.kmin[6],  kKmin27.kmin[7],  kKmin27.kmin[8],  kKmin27.kmin[9],  kKmin27.kmin[10], kKmin27.kmin[11],
    kKmin27.kmin[12], kKmin27.kmin[13], kKmin27.kmin[14], kKmin27.kmin[15], kKmin27.kmin[16], kKmin27.kmin[17],
    kKmin27.kmin[18], kKmin27.kmin[19], kKmin27.kmin[20], kKmin27.kmin[21], kKmin27.kmin[22], kKmin27.kmin[23],
    kKmin27.kmin[24], kKmin27.kmin[25], kKmin27.kmin[26]};

/// D = A B + D on the fp64 tensor cores: m8n8k4, A row-major (lane: row lane/4, col lane%4),
/// B column-major (lane: row lane%4, col lane/4), C/D (lane: row lane/4, cols 2(lane%4)+{0,1}).
__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

/// One bin of a pair, one particle: B-fragment entries from the staged T and W_a, then the
/// DMMA tiles (ce 0..7) and the FMA column (ce 8).  Lanes g < 3 form M[ce = qm][g]; the g = 3
/// pad lanes qm < 3 form M[8][qm] in the same loads, and a shuffle hands M[8][g] to the lanes of
/// column g.  `valid` = the slot holds a particle of this bin (stale slots hold finite data of an
/// earlier particle and get B = 0).
template <int NT>
__device__ __forceinline__ void asm_particle(const double* __restrict__ P, int wa, const int (&tb)[3], int src8,
                                             bool valid, const int (&oA)[4], double (&C)[4][2], double (&E)[4]) {
  const double w0 = P[wa], w1 = P[wa + 1], w2 = P[wa + 2];
  const double raw = w0 * P[tb[0]] + w1 * P[tb[1]] + w2 * P[tb[2]];
  const double m8raw = __shfl_sync(0xffffffffu, raw, src8);
  const double b = valid ? raw : 0.0;
  const double m8 = valid ? m8raw : 0.0;
#pragma unroll
  for (int mt = 0; mt < NT; ++mt) {
    const double a = P[oA[mt]];
    dmma_f64(C[mt], a, b);
    E[mt] = fma(a, m8, E[mt]);
  }
}

/// Fold one bin's register blocks into the row accumulator (upper slots su = S(k) + S(o) - 62).
template <int NT>
__device__ __forceinline__ void asm_fold(double* acc, int kmin, int So, int qm, int qk, double (&C)[4][2],
                                         double (&E)[4]) {
#pragma unroll
  for (int mt = 0; mt < NT; ++mt) {
    double e = E[mt];
    e += __shfl_xor_sync(0xffffffffu, e, 1);
    e += __shfl_xor_sync(0xffffffffu, e, 2);
    const int k = kmin + 8 * mt + qm;
    if (k <= 26) {
      const int su = 25 * (k / 9) + 5 * ((k / 3) % 3) + k % 3 + So - kDiagSlot;
      acc[su * 9 + 2 * qk] += C[mt][0];
      acc[su * 9 + 2 * qk + 1] += C[mt][1];
      if (qk == 0) acc[su * 9 + 8] += e;
    }
  }
}

template <int AW, int CH>
__global__ void __launch_bounds__(AW * 32) k_assemble_rows(BinsView bins, GridView g, LevelView L,
                                                                   const double* __restrict__ Tu,
                                                                   unsigned int* __restrict__ row_counter) {
  extern __shared__ __align__(16) double asm_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // per warp: staging [2 buffers][asm_stage<CH>()] | acc [kUpper*9] | pad | mbarriers [2] | pair table
  double* base = asm_smem + (size_t)wid * asm_warp_doubles<CH>();
  double* Sbuf = base;
  double* acc = base + 2 * asm_stage<CH>();
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(acc + kUpper * 9 + 1);
  int* PT = reinterpret_cast<int*>(acc + kUpper * 9 + 1 + 2);  // [14][pb1, n1, pb2, n2]
  for (int q = lane; q < 2 * asm_stage<CH>(); q += 32) Sbuf[q] = 0.0;  // stale slots must hold finite data
  __syncwarp();
  if (lane == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar + 1, 1);
    mbar_fence_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before the bulk copies
  }
  __syncwarp();
  unsigned phase = 0;  // bit b: parity of the next completion of buffer b
  const int qk = lane & 3, qm = lane >> 2;
  // lane's load f: M[ce = qm][g = qk] needs T[(3c+f),(3e+g)]; the g = 3 pad lanes qm < 3 load
  // T[(6+f),(6+qm)] (the ce = 8 column), the other pad lanes repeat a neighbour's address
  int tb[3];
  {
    const int c = qm / 3, e = qm % 3;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      if (qk < 3) tb[f] = kRecT + tslot(3 * c + f, 3 * e + qk);
      else if (qm < 4) tb[f] = kRecT + tslot(6 + f, 6 + min(qm, 2));
      else tb[f] = kRecT + tslot(3 * c + f, 3 * e + 2);
    }
  }
  const bool lane_g = qk < 3;
  const int src8 = 4 * min(qk, 2) + 3;  // the pad lane holding M[8][g]
  // rows are handed out in index order (a work counter), so the
  // rows in flight stay a narrow band and their particle bins stay in L2
  auto next_row = [&]() {
    int r = 0;
    if (lane == 0) r = (int)atomicAdd(row_counter, 1u);
    return L.lo + __shfl_sync(0xffffffffu, r, 0);
  };
  for (int i = next_row(); i < L.hi; i = next_row()) {
    for (int k = lane; k < kUpper * 9; k += 32) acc[k] = 0.0;
    // the write-out's column ids and Dirichlet flags, loaded now so their latency hides under
    // the gather: slot s = lane + 32 j (zero fill), upper slot 62 + lane + 32 j
    const int* crow = L.cols + (long long)i * kSlotPitch;
    int zc[kSlotPitch / 32], uc[2];
    bool ud[2];
#pragma unroll
    for (int j = 0; j < kSlotPitch / 32; ++j) zc[j] = lane + 32 * j < kSlots ? __ldg(crow + lane + 32 * j) : -1;
#pragma unroll
    for (int j = 0; j < 2; ++j) uc[j] = lane + 32 * j < kUpper ? __ldg(crow + kDiagSlot + lane + 32 * j) : -1;
#pragma unroll
    for (int j = 0; j < 2; ++j) ud[j] = uc[j] >= 0 && g.dir[uc[j]] != 0;
    const bool di = g.dir[i] != 0;
    const double mi = g.mass[i];
    const int ci0 = L.coords[3 * i], ci1 = L.coords[3 * i + 1], ci2 = L.coords[3 * i + 2];
    // lane o < 27 resolves bin offset o (bin node = i + o - 1): first particle and count
    int my_pb = 0, my_np = 0;
    if (lane < 27) {
      const int j = dense_lookup(L.map, ci0 + lane / 9 - 1, ci1 + (lane / 3) % 3 - 1, ci2 + lane % 3 - 1);
      if (j >= 0) {
        my_pb = __ldg(bins.start + j);
        my_np = __ldg(bins.start + j + 1) - my_pb;
      }
    }
    // pair q < 14: bins q and 26-q (q = 13: the centre bin alone); its table row in shared memory
    {
      const int pb2 = __shfl_sync(0xffffffffu, my_pb, 26 - min(lane, 26));
      const int n2 = __shfl_sync(0xffffffffu, my_np, 26 - min(lane, 26));
      if (lane < 14) {
        PT[4 * lane] = my_pb;
        PT[4 * lane + 1] = my_np;
        PT[4 * lane + 2] = pb2;
        PT[4 * lane + 3] = lane < 13 ? n2 : 0;
      }
      __syncwarp();
    }
    // lane 0 runs the bulk-copy producer one chunk ahead along (pair, c0)
    int pq_n = 0, c0_n = 0;  // next chunk to issue (lane 0)
    auto advance = [&]() {   // lane 0: move (pq_n, c0_n) to the next non-empty chunk
      c0_n += CH;
      while (pq_n < 14 && c0_n >= max(PT[4 * pq_n + 1], PT[4 * pq_n + 3])) {
        ++pq_n;
        c0_n = 0;
      }
    };
    auto issue = [&](int buf) {  // lane 0: one bulk copy per bin and chunk
      const int pb1 = PT[4 * pq_n], n1 = PT[4 * pq_n + 1], pb2 = PT[4 * pq_n + 2], n2 = PT[4 * pq_n + 3];
      const int k1 = max(0, min(CH, n1 - c0_n)), k2 = max(0, min(CH, n2 - c0_n));
      const unsigned mb = smem_u32(mbar + buf);
      double* dst = Sbuf + buf * asm_stage<CH>();
      mbar_expect_tx(mb, (k1 + k2) * kParticleBytes);
      if (k1) bulk_g2s(dst, Tu + (long long)(pb1 + c0_n) * kRecStride, k1 * kParticleBytes, mb);
      if (k2)
        bulk_g2s(dst + CH * kRecStride, Tu + (long long)(pb2 + c0_n) * kRecStride, k2 * kParticleBytes, mb);
    };
    if (lane == 0) {
      pq_n = 0;
      c0_n = -CH;
      advance();
      if (pq_n < 14) issue(0);
      advance();
    }
    int buf = 0;
    for (int pq = 0; pq < 14; ++pq) {
      const int n1 = PT[4 * pq + 1], n2 = PT[4 * pq + 3];
      const int nmax = max(n1, n2);
      if (nmax == 0) continue;
      // bin b's upper stencil positions: the suffix k >= kmin_b (slot S(k) + S(o_b) >= 62,
      // S(v) = 25 v0 + 5 v1 + v2); o_0 = pq, o_1 = 26 - pq (S(o_1) = 62 - S(o_0)); the row sits
      // at stencil position 26 - o_b of the bin's particles
      const int So0 = c_S27[pq], So1 = 62 - So0;
      const int kmin0 = c_kmin27[pq], kmin1 = pq == 13 ? 27 : c_kmin27[26 - pq];  // the centre bin has no mirror
      const int wa0 = kRecW + 3 * (26 - pq), wa1 = kRecW + 3 * pq;
      auto run = [&](auto nt0c, auto nt1c) {
        constexpr int NT0 = decltype(nt0c)::value, NT1 = decltype(nt1c)::value;
        double C0[4][2], C1[4][2], E0[4], E1[4];
        int oA0[4], oA1[4];  // A fragment W_k[g]: k clamped to 26 (rows past 26 are never folded)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          C0[mt][0] = C0[mt][1] = C1[mt][0] = C1[mt][1] = E0[mt] = E1[mt] = 0.0;
          oA0[mt] = kRecW + 3 * min(kmin0 + 8 * mt + qm, 26) + min(qk, 2);
          oA1[mt] = kRecW + 3 * min(kmin1 + 8 * mt + qm, 26) + min(qk, 2);
        }
        for (int c0 = 0; c0 < nmax; c0 += CH) {
          if (lane == 0) {
            if (pq_n < 14) issue(buf ^ 1);
            advance();
          }
          mbar_wait(smem_u32(mbar + buf), (phase >> buf) & 1u);
          phase ^= 1u << buf;
          const double* S = Sbuf + buf * asm_stage<CH>();
#pragma unroll 1
          for (int t = 0; t < CH; ++t) {
            asm_particle<NT0>(S + t * kTensorStride, wa0, tb, src8, lane_g && c0 + t < n1, oA0, C0, E0);
            if (NT1 > 0)
              asm_particle<NT1>(S + (CH + t) * kTensorStride, wa1, tb, src8, lane_g && c0 + t < n2, oA1,
                                C1, E1);
          }
          __syncwarp();  // buffer buf is refilled by the next iteration's issue
          buf ^= 1;
        }
        // fold the pair's accumulators into the row: bin 0, then the mirror bin
        asm_fold<NT0>(acc, kmin0, So0, qm, qk, C0, E0);
        __syncwarp();
        if (NT1 > 0) asm_fold<NT1>(acc, kmin1, So1, qm, qk, C1, E1);
        __syncwarp();
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I3 = std::integral_constant<int, 3>;
      using I4 = std::integral_constant<int, 4>;
      // tile counts ceil((27 - kmin) / 8) per bin: (1,4) pq 0-2, (1,3) 3-7, (2,3) 8-10, (2,2) 11-12, (2,0) 13
      if (pq < 3) run(I1{}, I4{});
      else if (pq < 8) run(I1{}, I3{});
      else if (pq < 11) run(I2{}, I3{});
      else if (pq < 13) run(I2{}, I2{});
      else run(I2{}, I0{});
    }
    // write-out: upper slots + transposed mirror, mass diagonal, Dirichlet projection
#pragma unroll
    for (int j = 0; j < kSlotPitch / 32; ++j) {  // inactive / pad slots hold zeros
      if (zc[j] < 0)
#pragma unroll
        for (int k = 0; k < 9; ++k) __stcs(L.H + ((long long)i * 9 + k) * kSlotPitch + lane + 32 * j, 0.0);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int u = lane + 32 * j, s = kDiagSlot + u;
      const int col = uc[j];
      if (col < 0) continue;
      double C[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) C[k] = acc[u * 9 + k];
      const bool zero = di || ud[j];
      if (s == kDiagSlot) {
        if (di) {
#pragma unroll
          for (int k = 0; k < 9; ++k) C[k] = (k % 4 == 0) ? 1.0 : 0.0;
        } else {  // symmetrise (objective.hpp:349-351), then the mass diagonal
          const double t01 = 0.5 * (C[1] + C[3]), t02 = 0.5 * (C[2] + C[6]), t12 = 0.5 * (C[5] + C[7]);
          C[1] = C[3] = t01;
          C[2] = C[6] = t02;
          C[5] = C[7] = t12;
          C[0] += mi;
          C[4] += mi;
          C[8] += mi;
        }
      } else if (zero) {
#pragma unroll
        for (int k = 0; k < 9; ++k) C[k] = 0.0;
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) __stcs(L.H + ((long long)i * 9 + k) * kSlotPitch + s, C[k]);
      if (s != kDiagSlot) {
        const int sm = kSlots - 1 - s;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) __stcs(L.H + ((long long)col * 9 + 3 * r + c) * kSlotPitch + sm, C[3 * c + r]);
      }
    }
    __syncwarp();
  }
}

int agrid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

void launch_particle_tensors(const ParticlesView& P, GridView g, double dx, double dt, const DevMaterial* mats,
                             const double* u, const double* svd_in, int project, double* Tu, int* bad_flag,
                             cudaStream_t s, long long plo, long long phi) {
  if (phi < 0) phi = P.n;
  if (phi <= plo) return;
  const long long chunks = (phi - plo + 31) / 32;
  // min CTAs per SM 1 (253 registers): cfg2 tensors phase 0.419 ms per step against 0.434 /
  // 0.495 / 0.672 ms at 3 / 4 / 6 (register caps that spill)
  const int tgrid_ = (int)std::min<long long>((chunks + kTWarps - 1) / kTWarps, 16LL * num_sms());
  k_particle_tensors<1><<<tgrid_, kTWarps * 32, 0, s>>>(P, g, dx, dt, mats, u, svd_in, project, Tu, bad_flag, plo, phi);
  k_particle_W<<<(int)std::min<long long>((chunks + kWWarps - 1) / kWWarps, 32LL * num_sms()), kWWarps * 32, 0, s>>>(
      P, dx, Tu, plo, phi);
  count_launches(2);
}

void launch_fill_cols(LevelView L, unsigned long long* active, cudaStream_t s) {
  cudaMemsetAsync(active, 0, sizeof(unsigned long long), s);
  if (L.n == 0) return;
  k_fill_cols<<<agrid((long long)L.n * level_pitch(L.radius), 256), 256, 0, s>>>(L, const_cast<int*>(L.cols), active);
  count_launches(1);
}

void launch_assemble_rows(const ParticlesView& P, BinsView bins, GridView g, LevelView L, double dx,
                          const double* Tu, unsigned int* row_counter, cudaStream_t s) {
  if (L.hi <= L.lo) return;
  (void)dx;
  (void)P;
  // 4 warps x 2 particles per bin chunk (cfg2 assembly per step: 4x2 3.56 ms, 2x2 3.54, 4x1
  // 3.55, 6x1 3.73, 8x1 3.93, 4x3 3.92); a resident grid taking rows from the work counter
  constexpr int AW = 4, CH = 2;
  const int resident = resident_blocks((const void*)k_assemble_rows<AW, CH>, AW * 32, asm_smem<AW, CH>());
  cudaMemsetAsync(row_counter, 0, sizeof(unsigned int), s);
  const long long blocks = std::min<long long>(resident, ((long long)(L.hi - L.lo) + AW - 1) / AW);
  k_assemble_rows<AW, CH><<<(int)blocks, AW * 32, asm_smem<AW, CH>(), s>>>(bins, g, L, Tu, row_counter);
  count_launches(1);
}

}  // namespace hotb200
