// Level-0 system matrix H = M + dt^2 d2Phi/dx2 on B200 (objective.hpp:318-363).
//
// Stage 1 (one thread per particle): virtual F -> SVD -> dP/dF projected in the diagonal
//   space -> one 1008-byte record per particle: the 27 W_k = F^nT grad w_k, then kappa*T as
//   its 45 unique entries (hot_particle.cuh: kRecW, kRecT, tslot).
// Stage 2, by bins (the default; k_bin_pairs + k_row_gather below): every particle of a bin has
//   the same 27 stencil nodes, so the bin's sums over its particles for the 378 unordered
//   stencil-position pairs are formed ONCE, as DMMA tiles on the fp64 tensor cores (records
//   staged by the bulk-copy engine, the result bulk-stored to a ring of bins); then one warp per
//   row adds the segments of its 27 bins in a fixed order (no atomics) and writes the row.
//   Each unordered block pair is written together with its transpose, so block (i,j) ==
//   block(j,i)^T exactly (the reference's symmetry_error() == 0 invariant).  The mass diagonal
//   and the Dirichlet projection (objective.hpp:133-144) are fused into the write-out.
// Stage 2, by row tiles (HOT_ASM=tiles; k_assemble_tiles): one warp per row gathers over the 27
//   neighbouring bins and forms the per-particle rank-3 block updates per (row, particle).
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
        double mu, la;
        particle_lame(mt, P.Jp, p, mu, la);
        double T[45];
        model_dpdf_projected(U, s, V, mu, la, mt.elasticity, dt * dt * vol, project != 0, T);
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

/// Column ids of every slot (-1 inactive): one warp per row, its coordinates loaded once and the
/// row's dense-map lookups issued together (a thread per (row, slot) chained two dependent L2
/// round trips per slot: 0.18 ms per cfg2 level 0).
template <int R>
__global__ void __launch_bounds__(256) k_fill_cols(LevelView L, int* __restrict__ cols,
                                                   unsigned long long* __restrict__ active) {
  constexpr int P = level_pitch(R), S = level_slots(R), W = 2 * R + 1;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  for (int i = gw; i < L.n; i += nw) {
    const int x = L.coords[3 * i], y = L.coords[3 * i + 1], z = L.coords[3 * i + 2];
    int c[P / 32];
#pragma unroll
    for (int j = 0; j < P / 32; ++j) {
      const int sl = lane + 32 * j;
      c[j] = sl < S ? dense_lookup(L.map, x + sl / (W * W) - R, y + (sl / W) % W - R, z + sl % W - R) : -1;
    }
#pragma unroll
    for (int j = 0; j < P / 32; ++j) {
      cols[(long long)i * P + lane + 32 * j] = c[j];
      cnt += c[j] >= 0 ? 1 : 0;
    }
  }
  // active-slot count of the level (algorithmic bytes of the profile), one atomic per warp
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0 && cnt) atomicAdd(active, cnt);
}

/// Level-0 assembly (objective.hpp:318-363), row tiles fed by a producer warp.
///
/// A tile is T consecutive level-0 rows (T consumer warps, one row each).  Rows are sorted
/// lexicographically, so a tile's rows usually share (x, y) and run along z; every particle bin
/// their stencils reach is bulk-copied into shared memory ONCE per tile and consumed by every
/// tile row whose 27-stencil it touches (up to 3 of them), instead of once per row.
///
/// Groups.  Consecutive tile rows with the same (x, y) and z steps of at most 3 form a group; the
/// producer stages, per group, the 9 bin columns (x + dx, y + dy) over z in [zfirst-1, zlast+1]
/// (each column is a contiguous particle range: bins are node-ordered), and only that group's
/// rows consume them.  So every row sees each of its 27 bins exactly once, in a fixed order
/// (column-major, z ascending, particles in storage order): the row sums are deterministic and
/// independent of the tiling (the slab-sharded assembly stays bitwise equal to one GPU).
///
/// Per (row i, particle p of a bin whose stencil holds i at position a) the row's upper blocks
/// k >= a (slot S(k) - S(a) above the diagonal, S(v) = 25 v0 + 5 v1 + v2) get the rank-3 update
///   C_k[c][e] += sum_g W_k[g] M[c][e][g],   M[c][e][g] = sum_f W_a[f] T[(3c+f),(3e+g)],
/// on the fp64 tensor cores (DMMA m8n8k4: M-dim = upper positions k in tiles of 8, N-dim =
/// ce 0..7, K = g padded to 4); the ninth column ce = 8 goes to the FMA pipe.  Each lane forms its
/// own B-fragment entry M[ce][g] from three staged T entries and W_a.
///
/// Pipeline: a ring of S slots of up to CP particle records (CP x 1008 B each).  The producer
/// warp's lane 0 fills a slot with one bulk copy of a bin chunk, the slot's metadata and an
/// mbarrier arrive.expect_tx; the T consumer warps wait on the slot's full barrier (suspending
/// in hardware, not spinning) and release it on its empty barrier.  The consumers' particle loop
/// is unrolled over CP with a warp-uniform exit at the chunk's count, so every load uses an
/// immediate offset from a per-chunk base.  The register accumulators of a (bin, row) are
/// folded into the row's shared accumulator once per bin, in a fixed order (no atomics).
///
/// Tuning (cfg2, level-0 assembly per step, tools/asm_variants.sh; the old one-row-per-warp
/// kernel took 5.73 ms): CP x S = 8 x 4 5.29 ms, 8 x 5 5.93, 8 x 6 5.88, 4 x 8 5.79, 16 x 2
/// 6.97; T = 2 / 8 rows per tile 8.4 / 7.7 ms against 6.6 at T = 4 (CP 4); register caps for
/// more CTAs per SM spill and lose (6.3-6.7 ms); two accumulator chains per chunk 6.0 vs 5.84.
#ifndef HOT_ASM_T
#define HOT_ASM_T 4
#endif
#ifndef HOT_ASM_CP
#define HOT_ASM_CP 8
#endif
#ifndef HOT_ASM_S
#define HOT_ASM_S 4
#endif
constexpr int kAsmT = HOT_ASM_T;          // rows (consumer warps) per tile
constexpr int kAsmCP = HOT_ASM_CP;        // particle records per ring slot
constexpr int kAsmS = HOT_ASM_S;          // ring slots
#ifndef HOT_ASM_UNROLL
#define HOT_ASM_UNROLL 4
#endif
constexpr int kAsmUnroll = HOT_ASM_UNROLL;  // particle-loop unroll of a ring slot
constexpr int kAsmSpan = 3 * kAsmT + 2;   // z extent of a group's bin columns, at most
constexpr unsigned kRecBytes = kTensorStride * 8;  // 1008 = 63 x 16
enum : int { kSlotData = 0, kSlotTileEnd = 1, kSlotStop = 2 };
struct AsmMeta {
  int kind, tile, group, col, bz, last, cnt, pad1;
};
constexpr size_t kAsmRingBytes = (size_t)kAsmS * kAsmCP * kRecBytes;
constexpr size_t kAsmAccBytes = (size_t)kAsmT * kUpper * 9 * 8;
constexpr size_t kAsmBarBytes = (size_t)2 * kAsmS * 8;
constexpr size_t kAsmMetaBytes = (size_t)kAsmS * sizeof(AsmMeta);
constexpr size_t kAsmTableBytes = (size_t)9 * kAsmSpan * 2 * 4;
constexpr size_t kAsmSmem = kAsmRingBytes + kAsmAccBytes + kAsmBarBytes + kAsmMetaBytes + kAsmTableBytes;
static_assert(kAsmRingBytes % 16 == 0 && kAsmAccBytes % 16 == 0, "16-byte aligned regions");

/// Group start (index within the tile) of tile row w: rows w' < w with the same (x, y) and z
/// steps of at most 3 belong to the same group.  Both sides of the pipeline call this.
__device__ __forceinline__ int asm_group_of(const LevelView& L, int r0, int w) {
  int g = w;
  while (g > 0) {
    const int* c1 = L.coords + 3 * (r0 + g);
    const int* c0 = c1 - 3;
    if (c0[0] != c1[0] || c0[1] != c1[1] || c1[2] - c0[2] > 3) break;
    --g;
  }
  return g;
}

/// D = A B + D on the fp64 tensor cores: m8n8k4, A row-major (lane: row lane/4, col lane%4),
/// B column-major (lane: row lane%4, col lane/4), C/D (lane: row lane/4, cols 2(lane%4)+{0,1}).
__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

/// One ring slot (CP records) for a row at stencil position a = kmin: B-fragment entries from the
/// staged T and W_a, then NT DMMA tiles (ce 0..7) and the FMA column (ce 8).  Lanes g < 3 form
/// M[ce = qm][g]; the g = 3 pad lanes qm < 3 form M[8][qm] in the same loads, and a shuffle hands
/// M[8][g] to the lanes of column g.  gmask zeroes the pad lanes' B row and FMA term.
template <int NT>
__device__ __forceinline__ void asm_chunk(const double* __restrict__ S, int kmin, const int (&tb)[3], int src8,
                                          double gmask, int qm, int qk, double (&C)[4][2], double (&E)[4], int cnt) {
  const double* pw = S + kRecW + 3 * kmin;
  const double* pt0 = S + tb[0];
  const double* pt1 = S + tb[1];
  const double* pt2 = S + tb[2];
  const double* pa[4];
#pragma unroll
  for (int mt = 0; mt < NT; ++mt) pa[mt] = S + kRecW + 3 * min(kmin + 8 * mt + qm, 26) + min(qk, 2);
#pragma unroll kAsmUnroll
  for (int t = 0; t < kAsmCP; ++t) {
    if (t >= cnt) break;  // warp-uniform: the slot's record count
    const int o = t * kTensorStride;
    const double w0 = pw[o], w1 = pw[o + 1], w2 = pw[o + 2];
    const double raw = w0 * pt0[o] + w1 * pt1[o] + w2 * pt2[o];
    const double m8 = __shfl_sync(0xffffffffu, raw, src8) * gmask;
    const double b = raw * gmask;
#pragma unroll
    for (int mt = 0; mt < NT; ++mt) {
      const double av = pa[mt][o];
      dmma_f64(C[mt], av, b);
      E[mt] = fma(av, m8, E[mt]);
    }
  }
}

/// Fold a (bin, row)'s register blocks into the row accumulator (upper slot su = S(k) - S(a)),
/// then clear them.
template <int NT>
__device__ __forceinline__ void asm_fold(double* acc, int kmin, int qm, int qk, double (&C)[4][2], double (&E)[4]) {
  const int Sa = 25 * (kmin / 9) + 5 * ((kmin / 3) % 3) + kmin % 3;
#pragma unroll
  for (int mt = 0; mt < NT; ++mt) {
    double e = E[mt];
    e += __shfl_xor_sync(0xffffffffu, e, 1);
    e += __shfl_xor_sync(0xffffffffu, e, 2);
    const int k = kmin + 8 * mt + qm;
    if (k <= 26) {
      const int su = 25 * (k / 9) + 5 * ((k / 3) % 3) + k % 3 - Sa;
      acc[su * 9 + 2 * qk] += C[mt][0];
      acc[su * 9 + 2 * qk + 1] += C[mt][1];
      if (qk == 0) acc[su * 9 + 8] += e;
    }
    C[mt][0] = C[mt][1] = E[mt] = 0.0;
  }
}

/// The row's write-out: upper slots + transposed mirror, mass diagonal, symmetrised diagonal
/// block (objective.hpp:349-351), Dirichlet projection (objective.hpp:133-144); inactive and pad
/// slots hold zeros.  zc / uc / ud / di / mi were loaded when the row's tile started.
/// Matrix store: streaming (evict-first) where nothing else competes for L2, default policy
/// where the partially written lower-half lines must outlive a stream of loads (k_row_gather).
template <bool STREAM>
__device__ __forceinline__ void asm_store(double* p, double v) {
  if (STREAM)
    __stcs(p, v);
  else
    *p = v;
}

template <bool STREAM = true>
__device__ __forceinline__ void asm_write_row(const LevelView& L, int i, int lane, const double* acc,
                                              const int (&zc)[kSlotPitch / 32], const int (&uc)[2],
                                              const bool (&ud)[2], bool di, double mi) {
#pragma unroll
  for (int j = 0; j < kSlotPitch / 32; ++j) {
    if (zc[j] < 0)
#pragma unroll
      for (int k = 0; k < 9; ++k) asm_store<STREAM>(L.H + ((long long)i * 9 + k) * kSlotPitch + lane + 32 * j, 0.0);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int u = lane + 32 * j, sl = kDiagSlot + u;
    const int col = uc[j];
    if (col < 0) continue;
    double Cb[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Cb[k] = acc[u * 9 + k];
    const bool zero = di || ud[j];
    if (sl == kDiagSlot) {
      if (di) {
#pragma unroll
        for (int k = 0; k < 9; ++k) Cb[k] = (k % 4 == 0) ? 1.0 : 0.0;
      } else {
        const double t01 = 0.5 * (Cb[1] + Cb[3]), t02 = 0.5 * (Cb[2] + Cb[6]), t12 = 0.5 * (Cb[5] + Cb[7]);
        Cb[1] = Cb[3] = t01;
        Cb[2] = Cb[6] = t02;
        Cb[5] = Cb[7] = t12;
        Cb[0] += mi;
        Cb[4] += mi;
        Cb[8] += mi;
      }
    } else if (zero) {
#pragma unroll
      for (int k = 0; k < 9; ++k) Cb[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) asm_store<STREAM>(L.H + ((long long)i * 9 + k) * kSlotPitch + sl, Cb[k]);
    if (sl != kDiagSlot) {
      const int sm = kSlots - 1 - sl;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) asm_store<STREAM>(L.H + ((long long)col * 9 + 3 * r + c) * kSlotPitch + sm, Cb[3 * c + r]);
    }
  }
}

/// mbarrier wait that suspends the warp in hardware between probes instead of spinning (the
/// spin loop's YIELD / TRYWAIT / BRA otherwise steal issue slots from the compute warps).
__device__ __forceinline__ void mbar_wait_sleep(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          bar),
      "r"(parity), "r"(100000)
      : "memory");

}

/// Non-blocking probe of an mbarrier phase.
__device__ __forceinline__ bool mbar_test(unsigned bar, unsigned parity) {
  unsigned done;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(done)
               : "r"(bar), "r"(parity)
               : "memory");
  return done != 0;
}

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

#ifdef HOT_ASM_MINB
#define HOT_ASM_BOUNDS __launch_bounds__((kAsmT + 1) * 32, HOT_ASM_MINB)
#else
#define HOT_ASM_BOUNDS __launch_bounds__((kAsmT + 1) * 32)
#endif
__global__ void HOT_ASM_BOUNDS k_assemble_tiles(BinsView bins, GridView g, LevelView L,
                                                                      const double* __restrict__ Tu,
                                                                      unsigned int* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char asm_sm[];
  double* ring = reinterpret_cast<double*>(asm_sm);
  double* accs = reinterpret_cast<double*>(asm_sm + kAsmRingBytes);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(asm_sm + kAsmRingBytes + kAsmAccBytes);
  unsigned long long* empty = full + kAsmS;
  AsmMeta* meta = reinterpret_cast<AsmMeta*>(asm_sm + kAsmRingBytes + kAsmAccBytes + kAsmBarBytes);
  int* table = reinterpret_cast<int*>(asm_sm + kAsmRingBytes + kAsmAccBytes + kAsmBarBytes + kAsmMetaBytes);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kAsmS; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, kAsmT);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int ntiles = (L.hi - L.lo + kAsmT - 1) / kAsmT;

  if (wid == kAsmT) {  // ------------------------------------------------ producer warp
    int it = 0;        // slots issued (lane 0 counts; broadcast after each group)
    auto acquire = [&]() {  // lane 0: wait until slot it % S is free again
      const int slot = it % kAsmS;
      mbar_wait_sleep(smem_u32(empty + slot), ((it / kAsmS) & 1) ^ 1);
      return slot;
    };
    for (;;) {
      int t = 0;
      if (lane == 0) t = (int)atomicAdd(tile_counter, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) break;
      const int r0 = L.lo + t * kAsmT;
      const int nr = min(kAsmT, L.hi - r0);
      for (int w = 0; w < nr; ++w) {
        if (asm_group_of(L, r0, w) != w) continue;  // w starts a group
        int wl = w;
        while (wl + 1 < nr && asm_group_of(L, r0, wl + 1) == w) ++wl;
        const int x = L.coords[3 * (r0 + w)], y = L.coords[3 * (r0 + w) + 1];
        const int zlo = L.coords[3 * (r0 + w) + 2] - 1;
        const int span = L.coords[3 * (r0 + wl) + 2] + 1 - zlo + 1;
        // bin table of the group: (first particle, count) per (column, z), warp-parallel lookups
        for (int e = lane; e < 9 * span; e += 32) {
          const int col = e / span, z = zlo + e % span;
          const int j = dense_lookup(L.map, x + col / 3 - 1, y + col % 3 - 1, z);
          int st = 0, cnt = 0;
          if (j >= 0) {
            st = __ldg(bins.start + j);
            cnt = __ldg(bins.start + j + 1) - st;
          }
          table[2 * e] = st;
          table[2 * e + 1] = cnt;
        }
        __syncwarp();
        if (lane == 0) {
          for (int e = 0; e < 9 * span; ++e) {
            const int st = table[2 * e], cnt = table[2 * e + 1];
            for (int c0 = 0; c0 < cnt; c0 += kAsmCP) {
              const int slot = acquire();
              const int k = min(kAsmCP, cnt - c0);
              meta[slot] = AsmMeta{kSlotData, t, w, e / span, zlo + e % span, c0 + kAsmCP >= cnt ? 1 : 0, k, 0};
              const unsigned mb = smem_u32(full + slot);
              double* dst = ring + (size_t)slot * kAsmCP * kTensorStride;
              mbar_expect_tx(mb, k * kRecBytes);
              bulk_g2s(dst, Tu + (long long)(st + c0) * kTensorStride, k * kRecBytes, mb);
              ++it;
            }
          }
        }
        it = __shfl_sync(0xffffffffu, it, 0);
        __syncwarp();  // the table is rewritten by the next group
      }
      if (lane == 0) {  // the tile's rows are complete: write-out marker
        const int slot = acquire();
        meta[slot] = AsmMeta{kSlotTileEnd, t, 0, 0, 0, 0, 0, 0};
        mbar_arrive(smem_u32(full + slot));
        ++it;
      }
      it = __shfl_sync(0xffffffffu, it, 0);
    }
    if (lane == 0) {
      const int slot = acquire();
      meta[slot] = AsmMeta{kSlotStop, 0, 0, 0, 0, 0, 0, 0};
      mbar_arrive(smem_u32(full + slot));
    }
    return;
  }

  // ------------------------------------------------------------------- consumer warp wid
  double* acc = accs + (size_t)wid * kUpper * 9;
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
  const double gmask = qk < 3 ? 1.0 : 0.0;
  const int src8 = 4 * min(qk, 2) + 3;  // the pad lane holding M[8][g]
  double C[4][2], E[4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) C[mt][0] = C[mt][1] = E[mt] = 0.0;
  int cur = -1, row = -1, grp = 0, zr = 0;
  // write-out inputs of the current row (loaded when its tile starts, so their latency hides)
  int zc[kSlotPitch / 32], uc[2];
  bool ud[2], di = false;
  double mi = 0.0;
  for (int it = 0;; ++it) {
    const int slot = it % kAsmS;
    mbar_wait_sleep(smem_u32(full + slot), (it / kAsmS) & 1);
    const AsmMeta m = meta[slot];
    if (m.kind == kSlotStop) break;
    if (m.tile != cur) {  // a new tile: this warp's row, its group, accumulator, write-out inputs
      cur = m.tile;
      const int r0 = L.lo + cur * kAsmT;
      row = r0 + wid < L.hi ? r0 + wid : -1;
      if (row >= 0) {
        grp = asm_group_of(L, r0, wid);
        zr = L.coords[3 * row + 2];
        for (int k = lane; k < kUpper * 9; k += 32) acc[k] = 0.0;
        const int* crow = L.cols + (long long)row * kSlotPitch;
#pragma unroll
        for (int j = 0; j < kSlotPitch / 32; ++j) zc[j] = lane + 32 * j < kSlots ? __ldg(crow + lane + 32 * j) : -1;
#pragma unroll
        for (int j = 0; j < 2; ++j) uc[j] = lane + 32 * j < kUpper ? __ldg(crow + kDiagSlot + lane + 32 * j) : -1;
#pragma unroll
        for (int j = 0; j < 2; ++j) ud[j] = uc[j] >= 0 && g.dir[uc[j]] != 0;
        di = g.dir[row] != 0;
        mi = g.mass[row];
      }
      __syncwarp();
    }
    if (m.kind == kSlotData) {
      const int a2 = zr - m.bz + 1;
      if (row >= 0 && m.group == grp && a2 >= 0 && a2 <= 2) {
        // the row sits at stencil position a = (1 - dx, 1 - dy, a2) of the bin's particles
        const int kmin = 9 * (2 - m.col / 3) + 3 * (2 - m.col % 3) + a2;
        const double* S = ring + (size_t)slot * kAsmCP * kTensorStride;
        // DMMA tiles over the upper positions: ceil((27 - kmin) / 8)
        if (kmin >= 19) {
          asm_chunk<1>(S, kmin, tb, src8, gmask, qm, qk, C, E, m.cnt);
          if (m.last) asm_fold<1>(acc, kmin, qm, qk, C, E);
        } else if (kmin >= 11) {
          asm_chunk<2>(S, kmin, tb, src8, gmask, qm, qk, C, E, m.cnt);
          if (m.last) asm_fold<2>(acc, kmin, qm, qk, C, E);
        } else if (kmin >= 3) {
          asm_chunk<3>(S, kmin, tb, src8, gmask, qm, qk, C, E, m.cnt);
          if (m.last) asm_fold<3>(acc, kmin, qm, qk, C, E);
        } else {
          asm_chunk<4>(S, kmin, tb, src8, gmask, qm, qk, C, E, m.cnt);
          if (m.last) asm_fold<4>(acc, kmin, qm, qk, C, E);
        }
      }
    } else if (m.kind == kSlotTileEnd && row >= 0) {
      __syncwarp();
      asm_write_row<true>(L, row, lane, acc, zc, uc, ud, di, mi);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + slot));
  }
}

// ---------------------------------------------------------------------------------------------
// Level-0 assembly by bins (the default): pair sums per bin on the fp64 tensor cores, then a row
// gather.  DESIGN.md §4 "Level-0 assembly by bins".
//
// Every particle of bin b (stencil-centre node b) has the same 27 stencil nodes, so the bin's
// contribution to block (node a, node k), a <= k stencil positions, is one small GEMM over the
// bin's particles:
//   P_b[a][k][c][e] = sum_p sum_g W^p_k[g] * M^{p,a}[c][e][g],
//   M^{p,a}[c][e][g] = sum_f W^p_a[f] T^p[(3c+f),(3e+g)]
// (objective.hpp:322-347 regrouped).  Stage A (k_bin_pairs) computes the 378 upper pairs x 9
// entries of every bin ONCE (the row-tile kernel re-formed M per (row, particle): 27 times) as
// DMMA m8n8k4 tiles with M-dim = k, N-dim = a (8 positions), K-dim = 4 particles of one
// component g, and bulk-stores the bin's 27,216-byte result; stage B (k_row_gather) sums, per
// row, the segments of its 27 bins in a fixed order and writes the row, its transposes, the mass
// diagonal and the Dirichlet projection (asm_write_row).  No atomics; every sum has a fixed
// order that does not depend on the row range, so slab-sharded assembly stays bitwise equal.
//
// Pair layout of a bin: segment of position a at pair_seg_off(a), entry (k - a) * 9 + (3c + e):
// the part of a bin one row needs is contiguous, (27 - a) * 72 bytes, and 16-byte aligned.
__host__ __device__ constexpr int pair_off(int a) { return 27 * a - a * (a - 1) / 2; }
static_assert(pair_off(27) == 378, "upper pairs of 27 positions");
/// First double of position a's segment: segments of odd length (a even) are padded by one
/// double, so every segment starts on a 16-byte boundary (bulk copies).
__host__ __device__ constexpr int pair_seg_off(int a) { return 9 * pair_off(a) + (a + 1) / 2; }
__host__ __device__ constexpr int pair_seg_len(int a) { return (9 * (27 - a) + 1) & ~1; }  // doubles copied
constexpr int kPairDoubles = pair_seg_off(27);
constexpr unsigned kPairBytes = kPairDoubles * 8;  // 27,328 = 1708 x 16
static_assert(kPairDoubles == 3416 && pair_seg_off(1) == 244 && pair_seg_off(2) == 478, "padded pair layout");
/// Slot index of stencil position k in the 5^3 diagonal storage, relative to position 0.
__device__ __forceinline__ int spos(int k) { return k + 2 * (k / 3) + 10 * (k / 9); }

#ifndef HOT_BP_CP
#define HOT_BP_CP 12
#endif
#ifndef HOT_BP_S
#define HOT_BP_S 3
#endif
constexpr int kBpCP = HOT_BP_CP;  // records per ring slot (groups of 4 particles)
constexpr int kBpS = HOT_BP_S;    // ring slots
constexpr int kBpWarps = 9;  // compute warps: one block entry ce = 3c + e each
constexpr int kBpGrab = 32;  // bins per work-counter grab
struct BpMeta {
  int kind, bin, cnt, last, pad[4];
};
constexpr size_t kBpRingBytes = (size_t)kBpS * kBpCP * kRecBytes;
constexpr size_t kBpOutBytes = 2 * (size_t)kPairBytes;
constexpr size_t kBpZeroBytes = kRecBytes;
constexpr size_t kBpBarBytes = (size_t)(2 * kBpS + 4) * 8;  // ring full / empty, output full[2] / free[2]
constexpr int kBpQueue = kBpS + 5;  // > bins between the producer's push and their store (ring slots + 2 outputs + 1)
constexpr size_t kBpMetaBytes = (size_t)kBpS * sizeof(BpMeta) + kBpQueue * sizeof(int);
constexpr size_t kBpSmem = kBpRingBytes + kBpOutBytes + kBpZeroBytes + kBpBarBytes + kBpMetaBytes;
static_assert(kBpRingBytes % 16 == 0 && kBpOutBytes % 16 == 0 && kBpZeroBytes % 16 == 0, "16-byte aligned regions");

/// One compute warp of k_bin_pairs: block entry ce = wid, all ten (a tile, k tile >= a tile)
/// accumulator tiles.  Lane (qk, qm): particle 4u + qk of the group, position 8t + qm of a tile;
/// the K index of a step is the particle and the step's component g = v is the same for all
/// lanes, so a lane needs three T entries per step, and the W_a its B entries need are also its
/// A entries (W_k[v] at k = a).  Lanes past the bin's count read a record of zeros.  A finished
/// bin's tiles go to one of two output buffers in the pair layout; the warps do not wait for each
/// other: each arrives on the buffer's mbarrier and the producer warp issues the bulk store.
__device__ __forceinline__ void bp_consume(const double* ring, const double* zero_rec, double* outs,
                                           unsigned long long* full, unsigned long long* empty, const BpMeta* meta,
                                           int wid, int lane) {
  unsigned long long* ofull = empty + kBpS;
  unsigned long long* ofree = ofull + 2;
  const int qk = lane & 3, qm = lane >> 2;
  const int c = wid / 3, e = wid % 3;
  double Cc[10][2];
#pragma unroll
  for (int t = 0; t < 10; ++t) Cc[t][0] = Cc[t][1] = 0.0;
  int wofs[4], tofs[3][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) wofs[i] = kRecW + 3 * min(8 * i + qm, 26);
#pragma unroll
  for (int v = 0; v < 3; ++v)
#pragma unroll
    for (int f = 0; f < 3; ++f) tofs[v][f] = kRecT + tslot(3 * c + f, 3 * e + v);
  int nbins = 0;  // bins this CTA has finished (selects the output buffer)
  for (int it = 0;; ++it) {
    const int slot = it % kBpS;
    mbar_wait_sleep(smem_u32(full + slot), (it / kBpS) & 1);
    const BpMeta m = meta[slot];
    if (m.kind == kSlotStop) break;
    const double* S = ring + (size_t)slot * kBpCP * kTensorStride;
    const int ngroups = (m.cnt + 3) >> 2;
    for (int u = 0; u < ngroups; ++u) {
      const int p = 4 * u + qk;
      const double* R = p < m.cnt ? S + p * kTensorStride : zero_rec;
      double W[4][3];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int f = 0; f < 3; ++f) W[i][f] = R[wofs[i] + f];
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const double t0 = R[tofs[v][0]], t1 = R[tofs[v][1]], t2 = R[tofs[v][2]];
        int t = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double B = fma(W[i][2], t2, fma(W[i][1], t1, W[i][0] * t0));
#pragma unroll
          for (int kt = i; kt < 4; ++kt) dmma_f64(Cc[t++], W[kt][v], B);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(empty + slot));
    if (m.last) {
      // the bin's tiles -> its pair layout in shared memory -> one bulk store
      double* out = outs + (size_t)(nbins & 1) * kPairDoubles;
      // the store of two bins ago has read this buffer (no wait in practice)
      if (nbins >= 2) mbar_wait_sleep(smem_u32(ofree + (nbins & 1)), ((nbins >> 1) - 1) & 1);
      int t = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int kt = i; kt < 4; ++kt) {
          const int k = 8 * kt + qm;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int a = 8 * i + 2 * qk + j;
            if (a <= k && k <= 26) out[pair_seg_off(a) + 9 * (k - a) + wid] = Cc[t][j];
            Cc[t][j] = 0.0;
          }
          ++t;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ofull + (nbins & 1)));  // the producer warp stores the bin
      ++nbins;
    }
  }
}

/// Stage A.  Bins [jlo, jhi) in grabs of kBpGrab from a work counter; a bin is skipped when it
/// is empty, when its records are not in [plo, phi) (slabs), or when none of its 27 nodes is a
/// row of [rlo, rhi).  G holds ring_cap bins; bin j lives at slot j % ring_cap.
__global__ void __launch_bounds__((kBpWarps + 1) * 32, 2)
    k_bin_pairs(BinsView bins, GridView g, const double* __restrict__ Tu, double* __restrict__ G, int ring_cap, int jlo,
                int jhi, int rlo, int rhi, long long plo, long long phi, unsigned int* __restrict__ counter,
                unsigned long long* __restrict__ bins_done) {
  extern __shared__ __align__(16) unsigned char bp_sm[];
  double* ring = reinterpret_cast<double*>(bp_sm);
  double* outs = reinterpret_cast<double*>(bp_sm + kBpRingBytes);
  double* zero_rec = reinterpret_cast<double*>(bp_sm + kBpRingBytes + kBpOutBytes);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(bp_sm + kBpRingBytes + kBpOutBytes + kBpZeroBytes);
  unsigned long long* empty = full + kBpS;
  BpMeta* meta = reinterpret_cast<BpMeta*>(bp_sm + kBpRingBytes + kBpOutBytes + kBpZeroBytes + kBpBarBytes);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < kTensorStride; k += blockDim.x) zero_rec[k] = 0.0;
  unsigned long long* ofull = empty + kBpS;
  unsigned long long* ofree = ofull + 2;
  int* binq = reinterpret_cast<int*>(meta + kBpS);
  if (threadIdx.x == 0) {
    for (int q = 0; q < kBpS; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, kBpWarps);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(ofull + q, kBpWarps);
      mbar_init(ofree + q, 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // (Rotating the producer's warp slot between the CTAs of an SM, by block index or by arrival
  // order on the SM, measured no different: the schedulers are not what limits the tensor pipe.)
  const int role = wid;
  if (role == kBpWarps) {  // ------------------------------------------------ producer warp
    // Lane 0 runs both pipelines without blocking in either: record chunks into free ring slots,
    // and the bulk store of every bin whose nine columns have arrived in an output buffer.
    int it = 0;  // ring slots issued
    int nb = 0;  // bins pushed (last chunk issued); bin q's id waits in binq[q % kBpQueue]
    int ns = 0;  // bins stored
    auto pump_store = [&]() -> bool {
      if (ns >= nb || !mbar_test(smem_u32(ofull + (ns & 1)), (ns >> 1) & 1)) return false;
      double* dst = G + (size_t)(binq[ns % kBpQueue] % ring_cap) * kPairDoubles;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"(smem_u32(outs + (size_t)(ns & 1) * kPairDoubles)), "r"(kPairBytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_arrive(smem_u32(ofree + (ns & 1)));
      ++ns;
      return true;
    };
    const bool all_rows = rlo <= 0 && rhi >= g.n;
    for (;;) {
      int j0 = 0;
      if (lane == 0) j0 = jlo + kBpGrab * (int)atomicAdd(counter, 1u);
      j0 = __shfl_sync(0xffffffffu, j0, 0);
      if (j0 >= jhi) break;
      // each lane looks at one bin of the grab
      const int j = j0 + lane;
      int st = 0, cnt = 0;
      if (j < jhi) {
        st = __ldg(bins.start + j);
        cnt = __ldg(bins.start + j + 1) - st;
        if (st < plo || st + cnt > phi) cnt = 0;
        if (cnt > 0 && !all_rows) {
          const int* nb27 = g.nb27 + 27LL * j;
          int mn = j, mx = j;
          for (int e = 0; e < 13; ++e) {
            const int q = __ldg(nb27 + e);
            if (q >= 0) {
              mn = q;
              break;
            }
          }
          for (int e = 26; e > 13; --e) {
            const int q = __ldg(nb27 + e);
            if (q >= 0) {
              mx = q;
              break;
            }
          }
          if (mx < rlo || mn >= rhi) cnt = 0;
        }
      }
      for (int e = 0; e < kBpGrab; ++e) {
        const int bst = __shfl_sync(0xffffffffu, st, e), bcnt = __shfl_sync(0xffffffffu, cnt, e);
        if (lane == 0) {
          for (int c0 = 0; c0 < bcnt; c0 += kBpCP) {
            const int slot = it % kBpS;
            while (!mbar_test(smem_u32(empty + slot), ((it / kBpS) & 1) ^ 1))
              if (!pump_store()) __nanosleep(32);
            const int k = min(kBpCP, bcnt - c0);
            const int last = c0 + kBpCP >= bcnt ? 1 : 0;
            meta[slot] = BpMeta{kSlotData, j0 + e, k, last, {0, 0, 0, 0}};
            const unsigned mb = smem_u32(full + slot);
            mbar_expect_tx(mb, k * kRecBytes);
            bulk_g2s(ring + (size_t)slot * kBpCP * kTensorStride, Tu + (long long)(bst + c0) * kTensorStride,
                     k * kRecBytes, mb);
            ++it;
            if (last) {
              binq[nb % kBpQueue] = j0 + e;
              ++nb;
            }
            pump_store();
          }
        }
      }
    }
    if (lane == 0) {
      const int slot = it % kBpS;
      while (!mbar_test(smem_u32(empty + slot), ((it / kBpS) & 1) ^ 1))
        if (!pump_store()) __nanosleep(32);
      meta[slot] = BpMeta{kSlotStop, 0, 0, 0, {0, 0, 0, 0}};
      mbar_arrive(smem_u32(full + slot));
      while (ns < nb)
        if (!pump_store()) __nanosleep(64);
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      if (bins_done && nb) atomicAdd(bins_done, (unsigned long long)nb);  // profile: bins with particles
    }
    return;
  }
  bp_consume(ring, zero_rec, outs, full, empty, meta, role, lane);
}

/// Stage B.  One warp per row of [rlo, rhi) whose largest neighbour bin lies in [blo, bhi) (the
/// band whose pair sums stage A has just produced; blo < 0 and bhi > n: every row).  A CTA takes
/// kRgWarps consecutive rows at a time from a counter, in index order: consecutive rows run
/// along z, their transposes fill neighbouring slots of the same lower-half lines at about the
/// same time, and the rows in flight stay a narrow band, so those lines are completed in L2.  The row's 27 bins in neighbour-table order (x, y, z
/// ascending); the row sits at position a = 26 - e of bin e, whose segment is read in runs of up
/// to three positions k (27 doubles, contiguous both in the segment and in the row's upper slots
/// spos(k) - spos(a)); the loads of two bins are in flight before the first is added.
#ifndef RG_WARPS
#define RG_WARPS 8
#endif
#ifndef RG_MINB
#define RG_MINB 3
#endif
#ifndef RG_STREAM
#define RG_STREAM false
#endif
constexpr int kRgWarps = RG_WARPS;
/// Pair-sum load: L2 only (no L1 allocation), default L2 policy.  With the rows of a CTA
/// consecutive, the sectors two runs or two rows share are L2 hits; an evict-first hint lost them
/// (k_row_gather 2.15 against 2.01 ms).
__device__ __forceinline__ double ld_pair(const double* p) { return __ldcg(p); }
/// Runs of bin position a: run 0 = positions a .. 3 (a / 3) + 2, run r >= 1 = the three positions
/// of (k0, k1) index a / 3 + r; 9 - a / 3 runs.  The run count is warp-uniform, and a switch that
/// falls through from the last run issues exactly that many loads / adds (predicated-off
/// instructions of a fully unrolled loop cost as many issue slots as live ones).
#define RG_RUN_LOAD(r) v[r] = lane < 27 ? ld_pair(seg + 9 * (3 * (m0 + r) - a) + lane) : 0.0
__device__ __forceinline__ void rg_load(const double* __restrict__ seg, int a, int lane, double (&v)[9]) {
  const int m0 = a / 3, len0 = 9 * (3 * m0 + 3 - a);
  switch (9 - m0) {
    case 9: RG_RUN_LOAD(8); [[fallthrough]];
    case 8: RG_RUN_LOAD(7); [[fallthrough]];
    case 7: RG_RUN_LOAD(6); [[fallthrough]];
    case 6: RG_RUN_LOAD(5); [[fallthrough]];
    case 5: RG_RUN_LOAD(4); [[fallthrough]];
    case 4: RG_RUN_LOAD(3); [[fallthrough]];
    case 3: RG_RUN_LOAD(2); [[fallthrough]];
    case 2: RG_RUN_LOAD(1); [[fallthrough]];
    default: v[0] = lane < len0 ? ld_pair(seg + lane) : 0.0;
  }
}
#undef RG_RUN_LOAD
#define RG_RUN_ADD(r)                                                          \
  {                                                                            \
    const int m = m0 + r;                                                      \
    if (lane < 27) acc[9 * (5 * m + 10 * (m / 3) - Sa) + lane] += v[r];        \
  }
__device__ __forceinline__ void rg_add(double* acc, int a, int lane, const double (&v)[9]) {
  const int m0 = a / 3, len0 = 9 * (3 * m0 + 3 - a), Sa = spos(a);
  switch (9 - m0) {
    case 9: RG_RUN_ADD(8); [[fallthrough]];
    case 8: RG_RUN_ADD(7); [[fallthrough]];
    case 7: RG_RUN_ADD(6); [[fallthrough]];
    case 6: RG_RUN_ADD(5); [[fallthrough]];
    case 5: RG_RUN_ADD(4); [[fallthrough]];
    case 4: RG_RUN_ADD(3); [[fallthrough]];
    case 3: RG_RUN_ADD(2); [[fallthrough]];
    case 2: RG_RUN_ADD(1); [[fallthrough]];
    default:
      if (lane < len0) acc[lane] += v[0];
  }
}
#undef RG_RUN_ADD
__global__ void __launch_bounds__(kRgWarps * 32, RG_MINB)
    k_row_gather(BinsView bins, GridView g, LevelView L, const double* __restrict__ G, int ring_cap, int rlo, int rhi,
                 int blo, int bhi, long long plo, long long phi, unsigned int* __restrict__ counter) {
  __shared__ __align__(16) double accs[kRgWarps][kUpper * 9];
  __shared__ int s_base[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* acc = accs[wid];
  if (threadIdx.x == 0) s_base[0] = rlo + kRgWarps * (int)atomicAdd(counter, 1u);
  for (int it = 0;; ++it) {
    __syncthreads();  // s_base[it & 1] is set; everyone is done with s_base[(it + 1) & 1]
    const int base = s_base[it & 1];
    if (base >= rhi) break;
    if (threadIdx.x == 0) s_base[(it + 1) & 1] = rlo + kRgWarps * (int)atomicAdd(counter, 1u);
    const int row = base + wid;
    if (row >= rhi) continue;
    int j = -1, cnt = 0, slot = 0;
    if (lane < 27) {
      j = __ldg(g.nb27 + 27LL * row + lane);
      if (j >= 0) {
        const int st = __ldg(bins.start + j);
        cnt = __ldg(bins.start + j + 1) - st;
        if (st < plo || st + cnt > phi) cnt = 0;
        slot = j % ring_cap;
      }
    }
    const unsigned present = __ballot_sync(0xffffffffu, j >= 0);
    const int mx = __shfl_sync(0xffffffffu, j, 31 - __clz((int)present));
    if (mx < blo || mx >= bhi) continue;
    unsigned live = __ballot_sync(0xffffffffu, cnt > 0);
    for (int k = lane; k < kUpper * 9; k += 32) acc[k] = 0.0;
    int zc[kSlotPitch / 32], uc[2];
    bool ud[2];
    const int* crow = L.cols + (long long)row * kSlotPitch;
#pragma unroll
    for (int q = 0; q < kSlotPitch / 32; ++q) zc[q] = lane + 32 * q < kSlots ? __ldg(crow + lane + 32 * q) : -1;
#pragma unroll
    for (int q = 0; q < 2; ++q) uc[q] = lane + 32 * q < kUpper ? __ldg(crow + kDiagSlot + lane + 32 * q) : -1;
#pragma unroll
    for (int q = 0; q < 2; ++q) ud[q] = uc[q] >= 0 && g.dir[uc[q]] != 0;
    const bool di = g.dir[row] != 0;
    const double mi = g.mass[row];
    __syncwarp();
    while (live) {
      const int e1 = __ffs((int)live) - 1;
      live &= live - 1;
      const int e2 = live ? __ffs((int)live) - 1 : -1;
      live &= live - 1;  // no-op on 0
      const int a1 = 26 - e1, a2 = 26 - max(e2, 0);
      const double* seg1 = G + (size_t)__shfl_sync(0xffffffffu, slot, e1) * kPairDoubles + pair_seg_off(a1);
      const double* seg2 = G + (size_t)__shfl_sync(0xffffffffu, slot, max(e2, 0)) * kPairDoubles + pair_seg_off(a2);
      double v1[9], v2[9];
      rg_load(seg1, a1, lane, v1);
      if (e2 >= 0) rg_load(seg2, a2, lane, v2);
      rg_add(acc, a1, lane, v1);
      if (e2 >= 0) rg_add(acc, a2, lane, v2);
    }
    __syncwarp();
    asm_write_row<RG_STREAM>(L, row, lane, acc, zc, uc, ud, di, mi);
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
  const int blocks = agrid((long long)L.n * 32, 256);
  if (L.radius == 2)
    k_fill_cols<2><<<blocks, 256, 0, s>>>(L, const_cast<int*>(L.cols), active);
  else
    k_fill_cols<3><<<blocks, 256, 0, s>>>(L, const_cast<int*>(L.cols), active);
  count_launches(1);
}

void launch_assemble_rows(const ParticlesView& P, BinsView bins, GridView g, LevelView L, double dx,
                          const double* Tu, unsigned int* tile_counter, cudaStream_t s) {
  if (L.hi <= L.lo) return;
  (void)dx;
  (void)P;
  // a resident grid of (T consumer + 1 producer)-warp CTAs taking row tiles from a counter in
  // index order, so the tiles in flight stay a narrow band and their particle bins stay in L2
  const int resident = resident_blocks((const void*)k_assemble_tiles, (kAsmT + 1) * 32, (int)kAsmSmem);
  cudaMemsetAsync(tile_counter, 0, sizeof(unsigned int), s);
  const long long tiles = ((long long)(L.hi - L.lo) + kAsmT - 1) / kAsmT;
  const long long blocks = std::min<long long>(resident, tiles);
  k_assemble_tiles<<<(int)blocks, (kAsmT + 1) * 32, kAsmSmem, s>>>(bins, g, L, Tu, tile_counter);
  count_launches(1);
}

int asm_pair_doubles() { return kPairDoubles; }

void launch_bin_pairs(BinsView bins, GridView g, LevelView L, const double* Tu, double* G, int ring_cap, int b0, int b1,
                      long long plo, long long phi, unsigned int* counter, unsigned long long* bins_done,
                      cudaStream_t s) {
  if (b1 <= b0) return;
  const int resident = resident_blocks((const void*)k_bin_pairs, (kBpWarps + 1) * 32, (int)kBpSmem);
  cudaMemsetAsync(counter, 0, sizeof(unsigned int), s);
  const long long grabs = ((long long)(b1 - b0) + kBpGrab - 1) / kBpGrab;
  k_bin_pairs<<<(int)std::min<long long>(resident, grabs), (kBpWarps + 1) * 32, kBpSmem, s>>>(
      bins, g, Tu, G, ring_cap, b0, b1, L.lo, L.hi, plo, phi, counter, bins_done);
  count_launches(1);
}

void launch_row_gather(BinsView bins, GridView g, LevelView L, const double* G, int ring_cap, int r0, int r1, int blo,
                       int bhi, long long plo, long long phi, unsigned int* counter, cudaStream_t s) {
  if (r1 <= r0) return;
  const int resident = resident_blocks((const void*)k_row_gather, kRgWarps * 32, 0);
  cudaMemsetAsync(counter, 0, sizeof(unsigned int), s);
  const long long blocks = ((long long)(r1 - r0) + kRgWarps - 1) / kRgWarps;
  k_row_gather<<<(int)std::min<long long>(resident, blocks), kRgWarps * 32, 0, s>>>(bins, g, L, G, ring_cap, r0, r1, blo,
                                                                                   bhi, plo, phi, counter);
  count_launches(1);
}

}  // namespace hotb200
