// Node-embedding Galerkin multigrid on B200 (multigrid.hpp:14-392, pcg.hpp:17-46).
//
//   build_restriction  dense coarse flags + scan (same lexicographic order as the
//                      reference's sort/unique); the embedding weights are implicit.
//   galerkin_coarsen   two gathers, each fine block read once: X = H_f P^T per fine row
//                      (rows streamed by bulk copy), then H_c = P X per upper coarse block,
//                      written with its transpose (exactly symmetric), Dirichlet projection fused.
//   smooth_sgs         the reference's serial colour-ordered symmetric Gauss-Seidel
//                      (multigrid.hpp:298-316) reproduced exactly by a wave schedule (DESIGN.md
//                      §4.1): level 0 streams all 54 waves through one persistent bulk-copy
//                      kernel; coarse levels run as a dataflow kernel with per-row epoch flags.
//   coarse_solve/pcg   Jacobi-PCG from zero as one cooperative kernel (3 grid barriers per
//                      iteration, deterministic block reductions).
#include <cooperative_groups.h>
#include <climits>
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

#include "hot_async.cuh"
#include "hot_internal.h"

namespace cg = cooperative_groups;

namespace hotb200 {

namespace {

constexpr int kMgThreads = 256;
constexpr int kMgWarps = kMgThreads / 32;
constexpr int kUpper = 63;
constexpr int kSgsThreads = 128;  // one thread per diagonal-storage slot

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int floor_div2(int x) { return x >> 1; }  // arithmetic shift = floor

/// Coarse parents of a fine lattice coordinate along one axis and their embedding weights
/// (multigrid.hpp:63-93, embedding_entries_1d): linear: even c -> c/2 (1); odd -> floor(c/2),
/// +1 (1/2 each).  Quadratic: even c -> c/2-1, c/2, c/2+1 (1/8, 3/4, 1/8); odd -> floor(c/2),
/// +1 (1/2 each).
__device__ __forceinline__ void parents_1d(int c, int quad, int& lo, int& cnt, double w[3]) {
  if (c & 1) {
    lo = floor_div2(c);
    cnt = 2;
    w[0] = w[1] = 0.5;
  } else if (quad) {
    lo = c / 2 - 1;
    cnt = 3;
    w[0] = 0.125;
    w[1] = 0.75;
    w[2] = 0.125;
  } else {
    lo = c / 2;
    cnt = 1;
    w[0] = 1.0;
  }
}

/// Weight of the fine child 2J + d of coarse node J along one axis (0 outside the embedding).
__device__ __forceinline__ double child_w(int d, int quad) {
  if (d == 0) return quad ? 0.75 : 1.0;
  if (d == 1 || d == -1) return 0.5;
  if (quad && (d == 2 || d == -2)) return 0.125;
  return 0.0;
}

__global__ void k_mark_parents(LevelView f, DenseMap cmap, int quad, uint8_t* __restrict__ flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.n; i += gridDim.x * blockDim.x) {
    int lo[3], cnt[3];
    double w[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) parents_1d(f.coords[3 * i + a], quad, lo[a], cnt[a], w[a]);
    for (int x = 0; x < cnt[0]; ++x)
      for (int y = 0; y < cnt[1]; ++y)
        for (int z = 0; z < cnt[2]; ++z) {
          const long long l = dense_lin(cmap, lo[0] + x, lo[1] + y, lo[2] + z);
          flags[l] = 1;
        }
  }
}

/// A coarse node is Dirichlet when a fine Dirichlet node embeds into it (multigrid.hpp:151).
__global__ void k_coarse_dirichlet(LevelView f, DenseMap cmap, int quad, uint8_t* __restrict__ cdir) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.n; i += gridDim.x * blockDim.x) {
    if (!f.dir[i]) continue;
    int lo[3], cnt[3];
    double w[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) parents_1d(f.coords[3 * i + a], quad, lo[a], cnt[a], w[a]);
    for (int x = 0; x < cnt[0]; ++x)
      for (int y = 0; y < cnt[1]; ++y)
        for (int z = 0; z < cnt[2]; ++z) cdir[dense_lookup(cmap, lo[0] + x, lo[1] + y, lo[2] + z)] = 1;
  }
}

/// Galerkin triple product H_c = R H_f R^T (multigrid.hpp:162-202) in two gathers, each
/// fine block read once:
///   X[i][B] = sum_{l in ch(B)} w_lB H_f(i,l)        one warp per fine row, its 9 KB row staged
///                                                  in shared memory; 64 coarse targets
///                                                  B = floor(i/2) - 1 + [0,4)^3 per row
///   H_c(A,B) = sum_{i in ch(A)} w_iA X[i][B]        one thread per upper coarse block, then the
///                                                  block and its transpose are written once
/// (exact symmetry); Dirichlet projection (multigrid.hpp:287) fused.  Linear embedding: child
/// 2B+d of B has weight prod_a (d_a ? 1/2 : 1).
constexpr int kGalX = 64 * 9;  // doubles of X per fine row
// warps per CTA x ring stages per warp (8 x 1, launch_galerkin)


constexpr int kGalXRowBytes = 9 * kSlotPitch * 8;  // 9216: one fine row's blocks, contiguous
template <int W, int S>
constexpr int galx_smem() { return W * (S * kGalXRowBytes + S * 8); }

/// Stage 1 of the Galerkin product, HBM-streaming: each warp keeps kGalXStages fine rows in
/// flight through the bulk-copy engine (one 9 KB cp.async.bulk per row, mbarrier completion)
/// while it contracts the previous row into its 64 coarse targets.
template <int W, int S>
__global__ void __launch_bounds__(W * 32) k_galerkin_x(LevelView f, double* __restrict__ X) {
  extern __shared__ __align__(128) unsigned char gx_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  unsigned char* ring = gx_smem + (size_t)wib * S * kGalXRowBytes;
  unsigned long long* mb =
      reinterpret_cast<unsigned long long*>(gx_smem + (size_t)W * S * kGalXRowBytes) +
      wib * S;
  unsigned long long policy = 0;
  if (lane == 0) {
    policy = l2_evict_first_policy();
    for (int s = 0; s < S; ++s) mbar_init(mb + s, 1);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](int row, int s) {  // lane 0
    const unsigned bar = smem_u32(mb + s);
    mbar_expect_tx(bar, kGalXRowBytes);
    bulk_g2s_hint(ring + (size_t)s * kGalXRowBytes, f.H + (long long)row * 9 * kSlotPitch, kGalXRowBytes, bar, policy);
  };
  if (lane == 0)
    for (int s = 0; s < S; ++s)
      if (f.lo + gw + s * nw < f.hi) issue(f.lo + gw + s * nw, s);
  unsigned phase_bits = 0;
  int s = 0;
  for (int i = f.lo + gw; i < f.hi; i += nw) {
    mbar_wait(smem_u32(mb + s), (phase_bits >> s) & 1u);
    phase_bits ^= 1u << s;
    const double* H = reinterpret_cast<const double*>(ring + (size_t)s * kGalXRowBytes);
    int base[3];  // 2*(floor(c/2)-1) - c: -2 (even) or -3 (odd)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int c = __ldg(f.coords + 3 * i + a);
      base[a] = 2 * ((c >> 1) - 1) - c;
    }
    for (int tq = lane; tq < 64; tq += 32) {
      const int t0 = tq >> 4, t1 = (tq >> 2) & 3, t2 = tq & 3;
      // an even coordinate (base -2) reaches coarse targets t = 0..2 only: t = 3 would be zeros,
      // and k_galerkin_c never reads it (27 to 64 targets per row are written, not always 64)
      if ((t0 == 3 && base[0] == -2) || (t1 == 3 && base[1] == -2) || (t2 == 3 && base[2] == -2)) continue;
      double acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.0;
#pragma unroll
      for (int d0 = -1; d0 <= 1; ++d0) {
        const int f0 = 2 * t0 + d0 + base[0];
        if (f0 < -2 || f0 > 2) continue;
#pragma unroll
        for (int d1 = -1; d1 <= 1; ++d1) {
          const int f1 = 2 * t1 + d1 + base[1];
          if (f1 < -2 || f1 > 2) continue;
#pragma unroll
          for (int d2 = -1; d2 <= 1; ++d2) {
            const int f2 = 2 * t2 + d2 + base[2];
            if (f2 < -2 || f2 > 2) continue;
            const double w = (d0 ? 0.5 : 1.0) * (d1 ? 0.5 : 1.0) * (d2 ? 0.5 : 1.0);
            const int sl = 25 * (f0 + 2) + 5 * (f1 + 2) + (f2 + 2);
#pragma unroll
            for (int k = 0; k < 9; ++k) acc[k] += w * H[k * kSlotPitch + sl];  // zero when l is inactive
          }
        }
      }
      double* dst = X + (long long)i * kGalX + 9 * tq;
#pragma unroll
      for (int k = 0; k < 9; ++k) dst[k] = acc[k];
    }
    __syncwarp();  // the stage is refilled below
    if (lane == 0 && i + S * nw < f.hi) issue(i + S * nw, s);
    s = s + 1 == S ? 0 : s + 1;
  }
}

__global__ void __launch_bounds__(kMgThreads) k_galerkin_c(LevelView f, LevelView c, const double* __restrict__ X) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int A = c.lo + gw; A < c.hi; A += nw) {
    const int A0 = c.coords[3 * A], A1 = c.coords[3 * A + 1], A2 = c.coords[3 * A + 2];
    const bool dA = c.dir[A] != 0;
    // children of A (fine nodes 2A + d) and their X base offsets
    int ch[27];
#pragma unroll
    for (int t = 0; t < 27; ++t) ch[t] = dense_lookup(f.map, 2 * A0 + t / 9 - 1, 2 * A1 + (t / 3) % 3 - 1, 2 * A2 + t % 3 - 1);
    for (int s = lane; s < kSlotPitch; s += 32)
      if (s >= kSlots || c.cols[(long long)A * kSlotPitch + s] < 0)
#pragma unroll
        for (int k = 0; k < 9; ++k) __stcs(c.H + ((long long)A * 9 + k) * kSlotPitch + s, 0.0);
    for (int u = lane; u < kUpper; u += 32) {
      const int s = kDiagSlot + u;
      const int B = c.cols[(long long)A * kSlotPitch + s];
      if (B < 0) continue;
      const int O0 = s / 25 - 2, O1 = (s / 5) % 5 - 2, O2 = s % 5 - 2;
      double acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.0;
#pragma unroll
      for (int t = 0; t < 27; ++t) {
        const int i = ch[t];
        if (i < 0) continue;
        const int d0 = t / 9 - 1, d1 = (t / 3) % 3 - 1, d2 = t % 3 - 1;
        // B - (floor(i/2) - 1) per axis; floor((2A+d)/2) = A + (d < 0 ? -1 : 0)
        const int q0 = O0 + 1 - (d0 < 0 ? -1 : 0), q1 = O1 + 1 - (d1 < 0 ? -1 : 0), q2 = O2 + 1 - (d2 < 0 ? -1 : 0);
        if ((unsigned)q0 > 3u || (unsigned)q1 > 3u || (unsigned)q2 > 3u) continue;
        // child coordinate 2A + d is even when d == 0: its X has no target 3 (not written, zero)
        if ((q0 == 3 && d0 == 0) || (q1 == 3 && d1 == 0) || (q2 == 3 && d2 == 0)) continue;
        const double w = (d0 ? 0.5 : 1.0) * (d1 ? 0.5 : 1.0) * (d2 ? 0.5 : 1.0);
        const double* x = X + (long long)i * kGalX + 9 * (16 * q0 + 4 * q1 + q2);
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += w * __ldg(x + k);
      }
      double C[9];
      if (s == kDiagSlot) {
        C[0] = acc[0];
        C[4] = acc[4];
        C[8] = acc[8];
        C[1] = C[3] = acc[1];
        C[2] = C[6] = acc[2];
        C[5] = C[7] = acc[5];
        if (dA) {
#pragma unroll
          for (int k = 0; k < 9; ++k) C[k] = (k % 4 == 0) ? 1.0 : 0.0;
        }
      } else {
        const bool zero = dA || c.dir[B] != 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) C[k] = zero ? 0.0 : acc[k];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) __stcs(c.H + ((long long)A * 9 + k) * kSlotPitch + s, C[k]);
      if (s != kDiagSlot) {
        const int sm = kSlots - 1 - s;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int q = 0; q < 3; ++q) __stcs(c.H + ((long long)B * 9 + 3 * r + q) * kSlotPitch + sm, C[3 * q + r]);
      }
    }
  }
}

/// Galerkin product for the QUADRATIC node embedding (coarse radius 3, multigrid.hpp:274),
/// the same two gathers as the linear kernels:
///   X[i][t] = sum_{l in row i, B parent of l} w_lB H_f(i,l), B = base(i) + t, t in [0, RF+3)^3,
///             base_a = floor((c_a - RF) / 2) - 1      (one warp per fine row, row in smem)
///   H_c(A,B) = sum_{i = 2A + d, |d| <= 2} w_iA X[i][B - base(i)]   (one lane per upper block)
/// Children weights per axis (1/8, 1/2, 3/4, 1/2, 1/8) for d = -2..2.  A contribution always
/// lands within radius 3 (|B - A| <= |l - i| / 2 + 2 <= 3), as the reference's overflow check
/// requires (multigrid.hpp:186-188).
constexpr int kGqWarps = 4;

template <int RF>
__global__ void __launch_bounds__(kGqWarps * 32) k_galerkin_qx(LevelView f, double* __restrict__ X) {
  constexpr int P = level_pitch(RF), NSL = 2 * RF + 1, SP = RF + 3, NT = SP * SP * SP;
  extern __shared__ __align__(16) double gq_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double* H = gq_smem + (size_t)wib * 9 * P;
  for (int i = gw; i < f.n; i += nw) {
    const double* src = f.H + (long long)i * 9 * P;
    __syncwarp();
    for (int q = lane; q < 9 * P; q += 32) H[q] = __ldcs(src + q);
    __syncwarp();
    int c[3], base[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c[a] = f.coords[3 * i + a];
      base[a] = ((c[a] - RF) >> 1) - 1;
    }
    for (int t = lane; t < NT; t += 32) {
      const int B0 = base[0] + t / (SP * SP), B1 = base[1] + (t / SP) % SP, B2 = base[2] + t % SP;
      double acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.0;
      for (int d0 = -2; d0 <= 2; ++d0) {
        const int f0 = 2 * B0 + d0 - c[0];
        if (f0 < -RF || f0 > RF) continue;
        const double w0 = child_w(d0, 1);
        for (int d1 = -2; d1 <= 2; ++d1) {
          const int f1 = 2 * B1 + d1 - c[1];
          if (f1 < -RF || f1 > RF) continue;
          const double w01 = w0 * child_w(d1, 1);
          for (int d2 = -2; d2 <= 2; ++d2) {
            const int f2 = 2 * B2 + d2 - c[2];
            if (f2 < -RF || f2 > RF) continue;
            const double w = w01 * child_w(d2, 1);
            const int sl = ((f0 + RF) * NSL + (f1 + RF)) * NSL + (f2 + RF);
#pragma unroll
            for (int k = 0; k < 9; ++k) acc[k] += w * H[k * P + sl];  // zero when l is inactive
          }
        }
      }
      double* dst = X + ((long long)i * NT + t) * 9;
#pragma unroll
      for (int k = 0; k < 9; ++k) dst[k] = acc[k];
    }
  }
}

template <int RF>
__global__ void __launch_bounds__(kMgThreads) k_galerkin_qc(LevelView f, LevelView c, const double* __restrict__ X) {
  constexpr int SP = RF + 3, NT = SP * SP * SP;
  constexpr int PC = level_pitch(3), SC = level_slots(3), DC = SC / 2, UPC = SC - DC;  // 352, 343, 171, 172
  __shared__ int ch_s[kMgWarps][125];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  int* ch = ch_s[wib];
  for (int A = gw; A < c.n; A += nw) {
    const int A0 = c.coords[3 * A], A1 = c.coords[3 * A + 1], A2 = c.coords[3 * A + 2];
    const bool dA = c.dir[A] != 0;
    __syncwarp();
    for (int t = lane; t < 125; t += 32)
      ch[t] = dense_lookup(f.map, 2 * A0 + t / 25 - 2, 2 * A1 + (t / 5) % 5 - 2, 2 * A2 + t % 5 - 2);
    __syncwarp();
    for (int s = lane; s < PC; s += 32)
      if (s >= SC || c.cols[(long long)A * PC + s] < 0)
#pragma unroll
        for (int k = 0; k < 9; ++k) __stcs(c.H + ((long long)A * 9 + k) * PC + s, 0.0);
    for (int u = lane; u < UPC; u += 32) {
      const int s = DC + u;
      const int B = c.cols[(long long)A * PC + s];
      if (B < 0) continue;
      const int O0 = s / 49 - 3, O1 = (s / 7) % 7 - 3, O2 = s % 7 - 3;
      double acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.0;
      for (int t = 0; t < 125; ++t) {
        const int i = ch[t];
        if (i < 0) continue;
        const int d0 = t / 25 - 2, d1 = (t / 5) % 5 - 2, d2 = t % 5 - 2;
        // B - base(i), base_a = floor((2A + d - RF) / 2) - 1
        const int q0 = A0 + O0 - ((((2 * A0 + d0) - RF) >> 1) - 1);
        const int q1 = A1 + O1 - ((((2 * A1 + d1) - RF) >> 1) - 1);
        const int q2 = A2 + O2 - ((((2 * A2 + d2) - RF) >> 1) - 1);
        if ((unsigned)q0 >= (unsigned)SP || (unsigned)q1 >= (unsigned)SP || (unsigned)q2 >= (unsigned)SP) continue;
        const double w = child_w(d0, 1) * child_w(d1, 1) * child_w(d2, 1);
        const double* x = X + ((long long)i * NT + (q0 * SP + q1) * SP + q2) * 9;
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += w * __ldg(x + k);
      }
      double C[9];
      if (s == DC) {
        C[0] = acc[0];
        C[4] = acc[4];
        C[8] = acc[8];
        C[1] = C[3] = acc[1];
        C[2] = C[6] = acc[2];
        C[5] = C[7] = acc[5];
        if (dA) {
#pragma unroll
          for (int k = 0; k < 9; ++k) C[k] = (k % 4 == 0) ? 1.0 : 0.0;
        }
      } else {
        const bool zero = dA || c.dir[B] != 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) C[k] = zero ? 0.0 : acc[k];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) __stcs(c.H + ((long long)A * 9 + k) * PC + s, C[k]);
      if (s != DC) {
        const int sm = SC - 1 - s;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int q = 0; q < 3; ++q) __stcs(c.H + ((long long)B * 9 + 3 * r + q) * PC + sm, C[3 * q + r]);
      }
    }
  }
}

/// Level diagonal inverse (multigrid.hpp:233-240) with the singular-block check.
__global__ void k_level_dinv(LevelView L, int* singular) {
  for (int i = L.lo + blockIdx.x * blockDim.x + threadIdx.x; i < L.hi; i += gridDim.x * blockDim.x) {
    M3 D;
#pragma unroll
    for (int k = 0; k < 9; ++k)
      D.m[k] = L.H[((long long)i * 9 + k) * level_pitch(L.radius) + level_slots(L.radius) / 2];
    double det;
    const M3 Di = m3_inverse(D, &det);
    if (!(fabs(det) > 0.0)) atomicExch(singular, 1);
#pragma unroll
    for (int k = 0; k < 9; ++k) L.dinv[9 * i + k] = Di.m[k];
  }
}

/// Wave id of every row (§4.1 of DESIGN.md): level 0 the mod-3 colour; coarse levels
/// 8 * colour + 4 (x>>1) + 2 (y>>1) + (z>>1), offset by the bounding box so ids start near 0.
__global__ void k_level_waves(LevelView L, int coarse, int q, int off0, int off1, int off2, int* __restrict__ wave_of) {
  // level 0: the mod-3 colour; coarse levels, colour modulus q (2 linear, 3 quadratic) and
  // radius <= q: t = 8 * colour + 4 X + 2 Y + Z on the colour sub-lattice (X = floor(x / q))
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += gridDim.x * blockDim.x) {
    const int c0 = L.coords[3 * i], c1 = L.coords[3 * i + 1], c2 = L.coords[3 * i + 2];
    auto md = [](int v, int k) { return ((v % k) + k) % k; };
    auto fl = [](int v, int k) { return v >= 0 ? v / k : -((-v + k - 1) / k); };
    int w;
    if (!coarse) {
      w = (md(c0, 3) * 3 + md(c1, 3)) * 3 + md(c2, 3);
    } else {
      const int col = (md(c0, q) * q + md(c1, q)) * q + md(c2, q);
      w = 8 * col + 4 * (fl(c0, q) - off0) + 2 * (fl(c1, q) - off1) + (fl(c2, q) - off2);
    }
    wave_of[i] = w;
  }
}

/// Rows bucketed by wave, a STABLE counting sort (rows of a wave in ascending index order, the
/// same on every run): per block of kBucketRows rows a shared-memory histogram (no contended
/// global atomics), an exclusive scan over the wave-major (wave, block) counts, then each block
/// ranks its rows in index order (match_any within 32-row chunks, running counts in shared
/// memory).  Rows of one wave never couple, so the order inside a wave changes no value; it only
/// makes the schedule deterministic and keeps a warp's neighbouring rows together.
constexpr int kBucketRows = 256;
__global__ void k_wave_block_count(const int* __restrict__ wave_of, int n, int wmin, int nwaves, int* __restrict__ bc) {
  extern __shared__ int hist[];
  for (int w = threadIdx.x; w < nwaves; w += blockDim.x) hist[w] = 0;
  __syncthreads();
  const int lo = blockIdx.x * kBucketRows, hi = min(n, lo + kBucketRows);
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(hist + (wave_of[i] - wmin), 1);
  __syncthreads();
  for (int w = threadIdx.x; w < nwaves; w += blockDim.x) bc[(long long)w * gridDim.x + blockIdx.x] = hist[w];
  if (blockIdx.x == 0 && threadIdx.x == 0) bc[(long long)nwaves * gridDim.x] = 0;  // the scan's total slot
}
__global__ void k_wave_block_scatter(const int* __restrict__ wave_of, int n, int wmin, int nwaves,
                                     const int* __restrict__ off, int* __restrict__ rows, int base) {
  extern __shared__ int run[];  // rows of each wave this block has placed so far
  const int lane = threadIdx.x;  // one warp per block
  for (int w = lane; w < nwaves; w += 32) run[w] = 0;
  __syncwarp();
  const int lo = blockIdx.x * kBucketRows, hi = min(n, lo + kBucketRows);
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const int i = i0 + lane;
    const bool v = i < hi;
    const int w = v ? wave_of[i] - wmin : -1 - lane;  // distinct keys for idle lanes
    const unsigned mask = __match_any_sync(0xffffffffu, w);
    const int rank = __popc(mask & ((1u << lane) - 1u));
    int pos = 0;
    if (v) pos = off[(long long)w * gridDim.x + blockIdx.x] + run[w] + rank;
    __syncwarp();
    if (v && rank == 0) run[w] += __popc(mask);
    __syncwarp();
    if (v) rows[pos] = base + i;
  }
}
/// counts[w] and start[w] (exclusive, start[nwaves] = n) from the (wave, block) offsets
__global__ void k_wave_totals(const int* __restrict__ off, int nblocks, int nwaves, int* __restrict__ counts,
                              int* __restrict__ start) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= nwaves; w += gridDim.x * blockDim.x) {
    const int s0 = off[(long long)w * nblocks];
    start[w] = s0;
    if (w < nwaves) counts[w] = off[(long long)(w + 1) * nblocks] - s0;
  }
}

/// out[p] = first row whose axis-0 coordinate is >= lo0 + p (p = 0..nplanes): the rows are in
/// lexicographic order, axis 0 most significant (common.hpp:41), so a plane range is a row range.
__global__ void k_plane_starts(const int* __restrict__ coords, int n, int lo0, int nplanes, int* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= nplanes; p += gridDim.x * blockDim.x) {
    int a = 0, b = n;
    while (a < b) {
      const int m = (a + b) >> 1;
      if (coords[3 * m] < lo0 + p) a = m + 1;
      else b = m;
    }
    out[p] = a;
  }
}

/// y_i (3) = sum_s H(i,s) x_col (objective.hpp:66-77), one warp per row.  All column ids and
/// all 36 block entries a lane needs are requested before any is consumed (memory-level
/// parallelism); inactive slots hold zeros (written by assembly / Galerkin), so they are
/// multiplied by 0 instead of branched around.
template <int R>
__device__ __forceinline__ void row_product(const LevelView& L, int i, const double* __restrict__ x, int lane,
                                            double& y0, double& y1, double& y2, bool cg_load) {
  constexpr int P = level_pitch(R), NS = P / 32;
  const int* cols = L.cols + (long long)i * P;
  const double* h = L.H + (long long)i * 9 * P;
  int c[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) c[k] = __ldg(cols + lane + 32 * k);
  double xv[NS][3];
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const double* xp = x + 3 * (c[k] >= 0 ? c[k] : 0);  // inactive slots: zero block, any finite x
#pragma unroll
    for (int a = 0; a < 3; ++a) xv[k][a] = cg_load ? __ldcg(xp + a) : __ldg(xp + a);
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const int s = lane + 32 * k;
    double hv[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) hv[e] = __ldcs(h + e * P + s);
    a0 += hv[0] * xv[k][0] + hv[1] * xv[k][1] + hv[2] * xv[k][2];
    a1 += hv[3] * xv[k][0] + hv[4] * xv[k][1] + hv[5] * xv[k][2];
    a2 += hv[6] * xv[k][0] + hv[7] * xv[k][1] + hv[8] * xv[k][2];
  }
  y0 = wsum(a0);
  y1 = wsum(a1);
  y2 = wsum(a2);
}

template <int R>
__global__ void __launch_bounds__(kMgThreads) k_spmv(LevelView L, const double* __restrict__ x, double* __restrict__ y,
                                                     const double* __restrict__ b) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = L.lo + gw; i < L.hi; i += nw) {
    double y0, y1, y2;
    row_product<R>(L, i, x, lane, y0, y1, y2, false);
    if (lane == 0) {
      if (b) {
        y[3 * i] = b[3 * i] - y0;
        y[3 * i + 1] = b[3 * i + 1] - y1;
        y[3 * i + 2] = b[3 * i + 2] - y2;
      } else {
        y[3 * i] = y0;
        y[3 * i + 1] = y1;
        y[3 * i + 2] = y2;
      }
    }
  }
}

/// b_c = R r_f (multigrid.hpp:24-31) as a gather over each coarse node's fine children 2J + d
/// (|d| <= 1 linear, <= 2 quadratic), Dirichlet coarse rows zeroed (multigrid.hpp:372-376).
__global__ void k_restrict(LevelView f, LevelView c, int quad, const double* __restrict__ rf, double* __restrict__ bc) {
  const int r = quad ? 2 : 1, w1 = 2 * r + 1;
  for (int J = blockIdx.x * blockDim.x + threadIdx.x; J < c.n; J += gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (!c.dir[J]) {
      const int J0 = c.coords[3 * J], J1 = c.coords[3 * J + 1], J2 = c.coords[3 * J + 2];
      for (int t = 0; t < w1 * w1 * w1; ++t) {
        const int d0 = t / (w1 * w1) - r, d1 = (t / w1) % w1 - r, d2 = t % w1 - r;
        const int i = dense_lookup(f.map, 2 * J0 + d0, 2 * J1 + d1, 2 * J2 + d2);
        if (i < 0) continue;
        const double w = child_w(d0, quad) * child_w(d1, quad) * child_w(d2, quad);
        a0 += w * rf[3 * i];
        a1 += w * rf[3 * i + 1];
        a2 += w * rf[3 * i + 2];
      }
    }
    bc[3 * J] = a0;
    bc[3 * J + 1] = a1;
    bc[3 * J + 2] = a2;
  }
}

/// u_f += P u_c (multigrid.hpp:33-39): each fine node's embedding parents.
__global__ void k_prolong_add(LevelView f, LevelView c, int quad, const double* __restrict__ uc,
                              double* __restrict__ uf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.n; i += gridDim.x * blockDim.x) {
    int lo[3], cnt[3];
    double w[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) parents_1d(f.coords[3 * i + a], quad, lo[a], cnt[a], w[a]);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int x = 0; x < cnt[0]; ++x)
      for (int y = 0; y < cnt[1]; ++y)
        for (int z = 0; z < cnt[2]; ++z) {
          const int J = dense_lookup(c.map, lo[0] + x, lo[1] + y, lo[2] + z);
          const double ww = w[0][x] * w[1][y] * w[2][z];
          a0 += ww * uc[3 * J];
          a1 += ww * uc[3 * J + 1];
          a2 += ww * uc[3 * J + 2];
        }
    uf[3 * i] += a0;
    uf[3 * i + 1] += a1;
    uf[3 * i + 2] += a2;
  }
}

constexpr int kMaxSgsWaves = 4096;
constexpr int kSgsSmem = 4 * (kMaxSgsWaves + 1);

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

/// Everything a row update needs except the neighbour values of u: it does not depend on the
/// wave, so it is loaded before the grid barrier that precedes the row's wave.
struct SgsRow {
  int i, c;
  double h[9];
  double D[9], b[3], uo[3];  // thread 0 only
};

__device__ __forceinline__ void sgs_load_row(const LevelView& L, const double* __restrict__ b, const double* u,
                                             int i, int s, SgsRow& R) {
  R.i = i;
  R.c = -1;
#pragma unroll
  for (int q = 0; q < 9; ++q) R.h[q] = 0.0;
  if (s >= kSlots) return;  // pad threads issue no loads (the barrier thread is one of them)
  R.c = __ldg(L.cols + (long long)i * kSlotPitch + s);
  const double* h = L.H + (long long)i * 9 * kSlotPitch + s;
#pragma unroll
  for (int q = 0; q < 9; ++q) R.h[q] = __ldcs(h + q * kSlotPitch);  // inactive slots hold zeros
  if (s == 0) {
#pragma unroll
    for (int q = 0; q < 9; ++q) R.D[q] = __ldg(L.dinv + 9 * (long long)i + q);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      R.b[a] = __ldg(b + 3 * (long long)i + a);
      R.uo[a] = __ldcg(u + 3 * (long long)i + a);  // only row i itself ever writes u_i
    }
  }
}

/// Grid barrier for the cooperative SGS kernel.  The arriving thread is the CTA's last (a pad
/// slot that never issues loads), so the release fence does not wait on the row prefetches of
/// the other threads.  Arrival counts grow monotonically: round t completes at t * gridDim.x.
__device__ __forceinline__ void sgs_grid_barrier(unsigned int* bar, unsigned int round) {
  __syncthreads();
  if (threadIdx.x == blockDim.x - 1) {
    const unsigned int target = round * gridDim.x;
    unsigned int prev;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
    if (prev == target - 1) {
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(bar + 1), "r"(round) : "memory");
    } else {
      unsigned int g;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      } while (g < round);
    }
  }
  __syncthreads();
}

/// One symmetric Gauss-Seidel sweep (multigrid.hpp:298-316) over the wave schedule, barrier
/// variant (HOT_SGS_COARSE=barrier; the dataflow k_sgs_flow is the default): a row of wave w
/// reads only neighbours of earlier waves (already updated) or later waves (still old),
/// exactly as the serial colour-ordered sweep does, with a grid barrier after every wave.
__global__ void __launch_bounds__(kSgsThreads) k_sgs(LevelView L, const int* __restrict__ wave_start,
                                                    const int* __restrict__ wave_rows, int nwaves, double* u,
                                                    const double* __restrict__ b, long long* trace,
                                                    unsigned int* bar) {
  // One CTA (128 threads = one per diagonal-storage slot) per row; after the barrier only the
  // gather of the neighbours' u (one L2 round trip), the FMA and the CTA reduction remain.
  extern __shared__ __align__(16) char sgs_smem[];
  __shared__ double red[kSgsThreads][3];
  cg::grid_group grid = cg::this_grid();
  const bool tr = trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  const int s = threadIdx.x, lane = s & 31, wid = s >> 5;
  int* ws = reinterpret_cast<int*>(sgs_smem);
  for (int k2 = threadIdx.x; k2 <= nwaves; k2 += blockDim.x) ws[k2] = wave_start[k2];
  __syncthreads();
  SgsRow R;
  bool have = false;
  {
    const int r0 = ws[0] + blockIdx.x;
    if (r0 < ws[1]) {
      sgs_load_row(L, b, u, __ldg(wave_rows + r0), s, R);
      have = true;
    }
  }
  int wave_counter = 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int k = 0; k < nwaves; ++k) {
      const int w = pass == 0 ? k : nwaves - 1 - k;
      const int e = ws[w + 1];
      if (tr && wave_counter < 1024) {
        trace[4 * wave_counter + 1] = gtimer();
        trace[4 * wave_counter + 2] = clock64();
      }
      for (int r = ws[w] + blockIdx.x; r < e; r += gridDim.x) {
        if (!have) sgs_load_row(L, b, u, __ldg(wave_rows + r), s, R);
        have = false;
        double x0 = 0.0, x1 = 0.0, x2 = 0.0;
        if (s < kSlots) {
          const double* xp = u + 3 * (R.c >= 0 ? R.c : 0);
          x0 = __ldcg(xp);
          x1 = __ldcg(xp + 1);
          x2 = __ldcg(xp + 2);
        }
        // row sum in the streaming kernels' order (k_sgs_flow<2>): lane l adds slots l, l+32,
        // l+64, l+96, then the warp sum
        red[s][0] = R.h[0] * x0 + R.h[1] * x1 + R.h[2] * x2;
        red[s][1] = R.h[3] * x0 + R.h[4] * x1 + R.h[5] * x2;
        red[s][2] = R.h[6] * x0 + R.h[7] * x1 + R.h[8] * x2;
        __syncthreads();
        double y0 = 0.0, y1 = 0.0, y2 = 0.0;
        if (wid == 0) {
          double b0 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int k2 = 0; k2 < kSgsThreads / 32; ++k2) {
            b0 += red[lane + 32 * k2][0];
            b1 += red[lane + 32 * k2][1];
            b2 += red[lane + 32 * k2][2];
          }
          y0 = wsum(b0);
          y1 = wsum(b1);
          y2 = wsum(b2);
        }
        if (s == 0) {
          const double r0 = R.b[0] - y0, r1 = R.b[1] - y1, r2 = R.b[2] - y2;
          const int i = R.i;
          u[3 * i] = R.uo[0] + (R.D[0] * r0 + R.D[1] * r1 + R.D[2] * r2);
          u[3 * i + 1] = R.uo[1] + (R.D[3] * r0 + R.D[4] * r1 + R.D[5] * r2);
          u[3 * i + 2] = R.uo[2] + (R.D[6] * r0 + R.D[7] * r1 + R.D[8] * r2);
        }
        __syncthreads();
      }
      if (tr && wave_counter < 1024) trace[4 * wave_counter + 3] = gtimer();
      {  // prepare this CTA's first row of the next wave
        const int np_ = k + 1 < nwaves ? pass : pass + 1;
        const int nk = k + 1 < nwaves ? k + 1 : 0;
        if (np_ < 2) {
          const int wn = np_ == 0 ? nk : nwaves - 1 - nk;
          const int rn = ws[wn] + blockIdx.x;
          if (rn < ws[wn + 1]) {
            sgs_load_row(L, b, u, __ldg(wave_rows + rn), s, R);
            have = true;
          }
        }
      }
      sgs_grid_barrier(bar, (unsigned int)(wave_counter + 1));
      if (tr && wave_counter < 1024) trace[4 * (wave_counter + 1)] = gtimer();
      ++wave_counter;
    }
  }
}

/// One wave of the Gauss-Seidel sweep as a plain streaming launch (large levels): rows of a
/// wave never couple, so u is read through the read-only path and the kernel boundary
/// orders the waves.
/// One Gauss-Seidel wave (rows of one colour class; no two couple), one warp per row.
/// Launched with programmatic dependent launch: the row's 9 KB of blocks and its column ids do
/// not depend on the previous wave, so they are loaded into registers BEFORE
/// griddepcontrol.wait and stream in while the previous wave drains; only the u gathers (L2,
/// ld.cg: written by the previous wave) and b, dinv wait.
constexpr int kWaveThreads = 128;
__global__ void __launch_bounds__(kWaveThreads) k_sgs_wave(LevelView L, const int* __restrict__ rows, int count,
                                                           double* __restrict__ u, const double* __restrict__ b,
                                                           int pdl) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool live = r < count;
  const int i = live ? __ldg(rows + r) : 0;
  int c[4];
  double hv[4][9];
  if (live) {
    const int* cols = L.cols + (long long)i * kSlotPitch;
    const double* h = L.H + (long long)i * 9 * kSlotPitch;
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = __ldg(cols + lane + 32 * k);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int e = 0; e < 9; ++e) hv[k][e] = __ldcs(h + e * kSlotPitch + lane + 32 * k);
  }
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (!live) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double* xp = u + 3 * (c[k] >= 0 ? c[k] : 0);  // inactive slots: zero block
    const double x0 = __ldcg(xp), x1 = __ldcg(xp + 1), x2 = __ldcg(xp + 2);
    a0 += hv[k][0] * x0 + hv[k][1] * x1 + hv[k][2] * x2;
    a1 += hv[k][3] * x0 + hv[k][4] * x1 + hv[k][5] * x2;
    a2 += hv[k][6] * x0 + hv[k][7] * x1 + hv[k][8] * x2;
  }
  const double y0 = wsum(a0), y1 = wsum(a1), y2 = wsum(a2);
  if (lane == 0) {
    const double* D = L.dinv + 9 * i;
    const double ub0 = __ldcg(u + 3 * i), ub1 = __ldcg(u + 3 * i + 1), ub2 = __ldcg(u + 3 * i + 2);
    const double r0 = __ldcg(b + 3 * i) - y0, r1 = __ldcg(b + 3 * i + 1) - y1, r2 = __ldcg(b + 3 * i + 2) - y2;
    u[3 * i] = ub0 + (D[0] * r0 + D[1] * r1 + D[2] * r2);
    u[3 * i + 1] = ub1 + (D[3] * r0 + D[4] * r1 + D[5] * r2);
    u[3 * i + 2] = ub2 + (D[6] * r0 + D[7] * r1 + D[8] * r2);
  }
}

/// Coarse-level symmetric Gauss-Seidel as a dataflow kernel (exact reference order,
/// multigrid.hpp:296-320).  Rows are dealt round-robin, in wave order (a topological order of
/// the sweep's dependency graph), to co-resident CTAs (one thread per slot).  A row starts as
/// soon as its own predecessors are done -- the coupled rows earlier in the pass order (lower
/// wave forward, higher wave backward; plus, backward, the row's own forward update) -- instead
/// of a grid barrier after every wave.  The rows later in the pass order wait for this row, so
/// they still hold their old values when it reads them: exactly the sequential sweep.
/// Progress: the lowest unfinished row in pass order always has all predecessors done and its
/// CTA has reached it (each CTA walks its rows in order).
///
/// The values are their own flags: the forward pass writes uf, the backward pass ub (and u),
/// both filled with an all-ones NaN sentinel before the sweep, each row written exactly once
/// per pass.  A waiting thread polls its column's three entries until none is the sentinel and
/// uses the values it polled, so a dependency costs one L2 round trip for the poll plus the
/// writer's store, instead of a flag poll, then a gather, then a release store (cfg2 level-1:
/// 2.3 us per dependency level with separate epoch flags).
__device__ __forceinline__ bool sgs_sentinel(double v) { return __double_as_longlong(v) == -1LL; }
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
/// Spin until the three entries at p are written (not the sentinel); returns them.
__device__ __forceinline__ void sgs_poll3(const double* p, double& x0, double& x1, double& x2) {
  do {
    x0 = ld_relaxed(p);
    x1 = ld_relaxed(p + 1);
    x2 = ld_relaxed(p + 2);
  } while (sgs_sentinel(x0) || sgs_sentinel(x1) || sgs_sentinel(x2));
}

template <int R>
__global__ void __launch_bounds__(level_pitch(R)) k_sgs_flow(LevelView L, const int* __restrict__ order, int n,
                                                         const int* __restrict__ wave_of, double* u,
                                                         const double* __restrict__ b, double* uf, double* ub) {
  constexpr int T = level_pitch(R), S = level_slots(R);  // one thread per diagonal-storage slot
  __shared__ double red[T / 32][3];
  __shared__ double uold[3];  // u_i, from the diagonal slot's gather (no second L2 round trip)
  // radius 2: the row sum in the streaming / per-wave kernels' order (lane l accumulates slots
  // l, l+32, l+64, l+96, then the warp sum), so the level-0 update is bitwise the same whichever
  // schedule runs it (one GPU small or large, or a slab)
  __shared__ double term[R == 2 ? T : 1][3];
  const int s = threadIdx.x, lane = s & 31, wid = s >> 5;
  // The next row of this CTA (its blocks, column id and wave ids) is requested before the current
  // row's polls, so a row whose predecessors finish finds its own data already in registers:
  // only the poll and the reduction stay on the dependency chain.
  struct Pre {
    int i, c, wi, wc;
    double h[9];
  };
  auto fetch = [&](int pass, int k, Pre& P) {
    P.i = __ldg(order + (pass == 0 ? k : n - 1 - k));
    P.c = -1;
    P.wi = P.wc = 0;
#pragma unroll
    for (int q = 0; q < 9; ++q) P.h[q] = 0.0;
    if (s < S) {
      P.c = __ldg(L.cols + (long long)P.i * T + s);
      const double* hp = L.H + (long long)P.i * 9 * T + s;
#pragma unroll
      for (int q = 0; q < 9; ++q) P.h[q] = __ldcs(hp + q * T);
      P.wi = __ldg(wave_of + P.i);
      P.wc = __ldg(wave_of + max(P.c, 0));
    }
  };
  Pre nx;
  if (blockIdx.x < n) fetch(0, blockIdx.x, nx);
  for (int pass = 0; pass < 2; ++pass) {
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
      const Pre cur = nx;
      if (k + (int)gridDim.x < n) fetch(pass, k + gridDim.x, nx);
      else if (pass == 0) fetch(1, blockIdx.x, nx);
      const int i = cur.i, c = cur.c;
      const double* h = cur.h;
      double D[9], rb[3];
      if (s == 0) {
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] = __ldg(L.dinv + 9 * (long long)i + q);
#pragma unroll
        for (int a = 0; a < 3; ++a) rb[a] = __ldg(b + 3 * (long long)i + a);
      }
      // each thread gathers its own column: predecessors in the pass order (and, backward, every
      // forward value) are polled until written; the others still hold the pass's input
      double x0 = 0.0, x1 = 0.0, x2 = 0.0;
      if (c >= 0) {
        const int wi = cur.wi, wc = cur.wc;
        if (pass == 0) {
          if (wc < wi) sgs_poll3(uf + 3 * c, x0, x1, x2);
          else {  // a successor or the row itself: the input
            x0 = __ldcg(u + 3 * c);
            x1 = __ldcg(u + 3 * c + 1);
            x2 = __ldcg(u + 3 * c + 2);
          }
        } else {
          if (wc > wi) sgs_poll3(ub + 3 * c, x0, x1, x2);
          else sgs_poll3(uf + 3 * c, x0, x1, x2);  // forward values (the row's own included)
        }
        if (s == S / 2) {
          uold[0] = x0;
          uold[1] = x1;
          uold[2] = x2;
        }
      }
      double a0 = h[0] * x0 + h[1] * x1 + h[2] * x2;
      double a1 = h[3] * x0 + h[4] * x1 + h[5] * x2;
      double a2 = h[6] * x0 + h[7] * x1 + h[8] * x2;
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      if constexpr (R == 2) {
        term[s][0] = a0;
        term[s][1] = a1;
        term[s][2] = a2;
        __syncthreads();
        if (wid == 0) {
          double b0 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int k = 0; k < T / 32; ++k) {
            b0 += term[lane + 32 * k][0];
            b1 += term[lane + 32 * k][1];
            b2 += term[lane + 32 * k][2];
          }
          y0 = wsum(b0);
          y1 = wsum(b1);
          y2 = wsum(b2);
        }
      } else {
        a0 = wsum(a0);
        a1 = wsum(a1);
        a2 = wsum(a2);
        if (lane == 0) {
          red[wid][0] = a0;
          red[wid][1] = a1;
          red[wid][2] = a2;
        }
        __syncthreads();
        if (s == 0) {
#pragma unroll
          for (int q = 0; q < T / 32; ++q) {
            y0 += red[q][0];
            y1 += red[q][1];
            y2 += red[q][2];
          }
        }
      }
      if (s == 0) {
        const double uo0 = uold[0], uo1 = uold[1], uo2 = uold[2];
        const double r0 = rb[0] - y0, r1 = rb[1] - y1, r2 = rb[2] - y2;
        const double n0 = uo0 + (D[0] * r0 + D[1] * r1 + D[2] * r2);
        const double n1 = uo1 + (D[3] * r0 + D[4] * r1 + D[5] * r2);
        const double n2 = uo2 + (D[6] * r0 + D[7] * r1 + D[8] * r2);
        double* out = (pass == 0 ? uf : ub) + 3 * i;
        st_relaxed(out, n0);
        st_relaxed(out + 1, n1);
        st_relaxed(out + 2, n2);
        if (pass == 1) {  // the sweep's result (every forward reader of u[i] is done: they
          u[3 * i] = n0;  // are coupled to i, and i's backward update waited for them)
          u[3 * i + 1] = n1;
          u[3 * i + 2] = n2;
        }
      }
      __syncthreads();
    }
  }
}

/// Level-0 symmetric Gauss-Seidel, all waves of both passes in ONE persistent cooperative
/// kernel (one CTA per SM).  Each warp owns a ring of kStreamStages row buffers in shared memory
/// filled by the bulk-copy engine (cp.async.bulk, completion on an mbarrier): a row's blocks
/// (9 KB) and column ids (512 B) are contiguous in the diagonal storage, so one row = two bulk
/// copies, issued by lane 0 and bypassing the L1 miss path.  The producer walks the warp's
/// flat (wave, row) sequence kStreamStages rows ahead of the consumer, ACROSS wave boundaries:
/// blocks and columns do not depend on u, so HBM streaming never drains at the grid barrier
/// between waves; only the u gathers (ld.cg, L2) wait for it.  Row arithmetic is identical to
/// k_sgs_wave (same summation order).
constexpr int kStreamRowBytes = 9 * kSlotPitch * 8 + kSlotPitch * 4;  // 9728
/// W warps per CTA, S ring stages per warp (8 x 2, launch_sgs_stream)
template <int W, int S>
constexpr int stream_smem() { return W * S * kStreamRowBytes + W * S * 8; }

struct StreamCursor {  // position in a warp's flat (wave, row) sequence
  int q, m;           // q: 0..2*nwaves-1 (forward then backward), m: this warp's m-th row of wave w(q)
};

template <int W, int S>
__global__ void __launch_bounds__(W * 32, 1)
    k_sgs_stream(LevelView L, const int* __restrict__ wave_start, const int* __restrict__ wave_rows, int nwaves,
                 double* u, const double* __restrict__ b, unsigned int* bar, int q_lo, int q_hi) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * W + wib, nw = gridDim.x * W;
  unsigned char* ring = sm_raw + (size_t)wib * S * kStreamRowBytes;
  unsigned long long* mb =
      reinterpret_cast<unsigned long long*>(sm_raw + (size_t)W * S * kStreamRowBytes) +
      wib * S;
  // the flat sequence q = 0 .. 2 nwaves - 1 (forward, then backward); this launch runs [q_lo, q_hi)
  const int nq = q_hi;
  auto wave_of = [&](int q) { return q < nwaves ? q : 2 * nwaves - 1 - q; };
  auto count_of = [&](int q) {
    const int w = wave_of(q);
    return __ldg(wave_start + w + 1) - __ldg(wave_start + w);
  };
  // advance a cursor to the next existing row of this warp (or q == nq)
  auto settle = [&](StreamCursor& c) {
    while (c.q < nq && gw + c.m * nw >= count_of(c.q)) {
      ++c.q;
      c.m = 0;
    }
  };
  unsigned long long policy = 0;
  if (lane == 0) {
    policy = l2_evict_first_policy();
    for (int s = 0; s < S; ++s) mbar_init(mb + s, 1);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](const StreamCursor& c, int stage) {
    const int w = wave_of(c.q);
    const int i = __ldg(wave_rows + __ldg(wave_start + w) + gw + c.m * nw);
    unsigned char* dst = ring + (size_t)stage * kStreamRowBytes;
    const unsigned mbar = smem_u32(mb + stage);
    mbar_expect_tx(mbar, kStreamRowBytes);
    bulk_g2s_hint(dst, L.H + (long long)i * 9 * kSlotPitch, 9 * kSlotPitch * 8, mbar, policy);
    bulk_g2s_hint(dst + 9 * kSlotPitch * 8, L.cols + (long long)i * kSlotPitch, kSlotPitch * 4, mbar, policy);
    return i;
  };
  // prologue: fill the ring
  StreamCursor prod{q_lo, 0};
  settle(prod);
  int rowid[S];
  for (int s = 0; s < S; ++s) {
    rowid[s] = -1;
    if (prod.q < nq) {
      int i = 0;
      if (lane == 0) i = issue(prod, s);
      rowid[s] = __shfl_sync(0xffffffffu, i, 0);
      ++prod.m;
      settle(prod);
    }
  }
  int stage = 0;
  unsigned phase_bits = 0;  // bit s: parity to wait for on stage s
  for (int q = q_lo; q < nq; ++q) {
    if (q > q_lo) sgs_grid_barrier(bar, (unsigned int)(q - q_lo));
    const int cnt = count_of(q);
    for (int r = gw; r < cnt; r += nw) {
      const int i = rowid[stage];
      mbar_wait(smem_u32(mb + stage), (phase_bits >> stage) & 1u);
      phase_bits ^= 1u << stage;
      const double* H = reinterpret_cast<const double*>(ring + (size_t)stage * kStreamRowBytes);
      const int* cols = reinterpret_cast<const int*>(ring + (size_t)stage * kStreamRowBytes + 9 * kSlotPitch * 8);
      int c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = cols[lane + 32 * k];
      double xv[4][3];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double* xp = u + 3 * (c[k] >= 0 ? c[k] : 0);
#pragma unroll
        for (int a = 0; a < 3; ++a) xv[k][a] = __ldcg(xp + a);
      }
      double D[9], rb[3], ub[3];
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) D[k] = __ldg(L.dinv + 9 * i + k);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          rb[a] = __ldg(b + 3 * i + a);
          ub[a] = __ldcg(u + 3 * i + a);
        }
      }
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int s = lane + 32 * k;
        double hv[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) hv[e] = H[e * kSlotPitch + s];
        a0 += hv[0] * xv[k][0] + hv[1] * xv[k][1] + hv[2] * xv[k][2];
        a1 += hv[3] * xv[k][0] + hv[4] * xv[k][1] + hv[5] * xv[k][2];
        a2 += hv[6] * xv[k][0] + hv[7] * xv[k][1] + hv[8] * xv[k][2];
      }
      __syncwarp();  // all lanes are done with this stage's shared memory
      if (prod.q < nq) {
        int ni = 0;
        if (lane == 0) ni = issue(prod, stage);
        rowid[stage] = __shfl_sync(0xffffffffu, ni, 0);
        ++prod.m;
        settle(prod);
      }
      const double y0 = wsum(a0), y1 = wsum(a1), y2 = wsum(a2);
      if (lane == 0) {
        const double r0 = rb[0] - y0, r1 = rb[1] - y1, r2 = rb[2] - y2;
        u[3 * i] = ub[0] + (D[0] * r0 + D[1] * r1 + D[2] * r2);
        u[3 * i + 1] = ub[1] + (D[3] * r0 + D[4] * r1 + D[5] * r2);
        u[3 * i + 2] = ub[2] + (D[6] * r0 + D[7] * r1 + D[8] * r2);
      }
      stage = stage + 1 == S ? 0 : stage + 1;
    }
  }
}

/// Deterministic grid reduction: every block sums all block partials in the same fixed tree.
__device__ __forceinline__ double grid_total(const double* partials, int nparts) {
  __shared__ double ws[kMgWarps];
  __shared__ double res;
  double v = 0.0;
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) v += __ldcg(partials + k);
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kMgWarps; ++w) t += ws[w];
    res = t;
  }
  __syncthreads();
  const double r = res;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void block_partial(double v, double* partials) {
  __shared__ double ws[kMgWarps];
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kMgWarps; ++w) t += ws[w];
    partials[blockIdx.x] = t;
  }
  __syncthreads();
}

template <int R>
__global__ void __launch_bounds__(kMgThreads) k_pcg(LevelView L, const double* __restrict__ b, double* x, double* r,
                                                    double* z, double* p, double* Ap, double rel, int cap,
                                                    double* partials, int* stat, int* iter_acc) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  const int nb = gridDim.x;
  // x = 0, r = b, z = D^-1 r, p = z, rho = r.z
  double loc = 0.0;
  for (int i = tid; i < L.n; i += nt) {
    const double* D = L.dinv + 9 * i;
    const double r0 = b[3 * i], r1 = b[3 * i + 1], r2 = b[3 * i + 2];
    const double z0 = D[0] * r0 + D[1] * r1 + D[2] * r2;
    const double z1 = D[3] * r0 + D[4] * r1 + D[5] * r2;
    const double z2 = D[6] * r0 + D[7] * r1 + D[8] * r2;
    x[3 * i] = x[3 * i + 1] = x[3 * i + 2] = 0.0;
    r[3 * i] = r0;
    r[3 * i + 1] = r1;
    r[3 * i + 2] = r2;
    z[3 * i] = p[3 * i] = z0;
    z[3 * i + 1] = p[3 * i + 1] = z1;
    z[3 * i + 2] = p[3 * i + 2] = z2;
    loc += r0 * z0 + r1 * z1 + r2 * z2;
  }
  block_partial(loc, partials);
  grid.sync();
  double rho = grid_total(partials, nb);
  int its = 0;
  int status = 0;
  if (!(rho > 0.0)) {
    if (rho < 0.0) status = 1;
  } else {
    const double threshold = rel * rel * rho;
    for (int it = 0; it < cap; ++it) {
      grid.sync();  // p complete; partials free
      loc = 0.0;
      for (int i = gw; i < L.n; i += nw) {
        double y0, y1, y2;
        row_product<R>(L, i, p, lane, y0, y1, y2, true);
        if (lane == 0) {
          Ap[3 * i] = y0;
          Ap[3 * i + 1] = y1;
          Ap[3 * i + 2] = y2;
          loc += __ldcg(p + 3 * i) * y0 + __ldcg(p + 3 * i + 1) * y1 + __ldcg(p + 3 * i + 2) * y2;
        }
      }
      block_partial(loc, partials);
      grid.sync();
      const double pAp = grid_total(partials, nb);
      if (!(pAp > 0.0)) {
        status = 2;
        break;
      }
      const double alpha = rho / pAp;
      grid.sync();  // everyone has read partials
      loc = 0.0;
      for (int i = tid; i < L.n; i += nt) {
        const double* D = L.dinv + 9 * i;
        double rr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          x[3 * i + a] = __dadd_rn(x[3 * i + a], __dmul_rn(alpha, __ldcg(p + 3 * i + a)));
          rr[a] = __dsub_rn(r[3 * i + a], __dmul_rn(alpha, __ldcg(Ap + 3 * i + a)));
          r[3 * i + a] = rr[a];
        }
        const double z0 = D[0] * rr[0] + D[1] * rr[1] + D[2] * rr[2];
        const double z1 = D[3] * rr[0] + D[4] * rr[1] + D[5] * rr[2];
        const double z2 = D[6] * rr[0] + D[7] * rr[1] + D[8] * rr[2];
        z[3 * i] = z0;
        z[3 * i + 1] = z1;
        z[3 * i + 2] = z2;
        loc += rr[0] * z0 + rr[1] * z1 + rr[2] * z2;
      }
      block_partial(loc, partials);
      grid.sync();
      const double rho_new = grid_total(partials, nb);
      its = it + 1;
      if (rho_new <= threshold) break;
      const double beta = rho_new / rho;
      for (int i = tid; i < L.n; i += nt)
#pragma unroll
        for (int a = 0; a < 3; ++a) p[3 * i + a] = __dadd_rn(z[3 * i + a], __dmul_rn(beta, p[3 * i + a]));
      rho = rho_new;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    stat[0] = status;
    stat[1] = its;
    if (iter_acc) *iter_acc += its;
  }
}

int mgrid(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

int coop_blocks(const void* fn, int threads, int smem = 0) { return resident_blocks(fn, threads, smem); }

}  // namespace


template <int R>
int sgs_flow_blocks() {
  // every co-resident CTA: capped at 4 per SM the cfg2 level-1 smoother drops 1.03 -> 1.00 ms per
  // step but the level-0 streaming smoother that follows it rises 1.70 -> 1.91 (bench.py).  The
  // grid size changes no value (the dataflow enforces the serial order).
  return coop_blocks((const void*)k_sgs_flow<R>, level_pitch(R), 0);
}

void launch_sgs_flow(LevelView L, const int* order, const int* wave_of, double* u, const double* b, double* uf,
                     double* ub, cudaStream_t s) {
  if (L.n == 0) return;
  int n = L.n;
  // the all-ones NaN sentinel: "not written yet" for every row of both passes
  cudaMemsetAsync(uf, 0xff, sizeof(double) * 3 * (size_t)n, s);
  cudaMemsetAsync(ub, 0xff, sizeof(double) * 3 * (size_t)n, s);
  void* args[] = {&L, (void*)&order, &n, (void*)&wave_of, &u, (void*)&b, &uf, &ub};
  if (L.radius == 2) {
    const int grid = std::min(sgs_flow_blocks<2>(), n);
    cudaLaunchCooperativeKernel((const void*)k_sgs_flow<2>, grid, level_pitch(2), args, 0, s);
  } else {
    const int grid = std::min(sgs_flow_blocks<3>(), n);
    cudaLaunchCooperativeKernel((const void*)k_sgs_flow<3>, grid, level_pitch(3), args, 0, s);
  }
  count_launches(1);
}

int sgs_max_blocks() { return coop_blocks((const void*)k_sgs, kSgsThreads, kSgsSmem); }
int pcg_max_blocks() {
  return std::min(coop_blocks((const void*)k_pcg<2>, kMgThreads), coop_blocks((const void*)k_pcg<3>, kMgThreads));
}

void launch_mark_parents(LevelView fine, DenseMap cmap, int quad, uint8_t* flags, cudaStream_t s) {
  if (fine.n) { k_mark_parents<<<mgrid(fine.n, 256), 256, 0, s>>>(fine, cmap, quad, flags); count_launches(1); }
}
void launch_coarse_dirichlet(LevelView fine, DenseMap cmap, int quad, uint8_t* cdir, cudaStream_t s) {
  if (fine.n) { k_coarse_dirichlet<<<mgrid(fine.n, 256), 256, 0, s>>>(fine, cmap, quad, cdir); count_launches(1); }
}
template <int W, int S>
void launch_galerkin_x_t(LevelView fine, double* X, cudaStream_t s) {
  const int gx_blocks = coop_blocks((const void*)k_galerkin_x<W, S>, W * 32, galx_smem<W, S>());
  const int blocks = (int)std::min<long long>(gx_blocks, ((long long)(fine.hi - fine.lo) + W - 1) / W);
  k_galerkin_x<W, S><<<std::max(1, blocks), W * 32, galx_smem<W, S>(), s>>>(fine, X);
  count_launches(1);
}

void launch_galerkin(LevelView fine, LevelView coarse, double* X, cudaStream_t s) {
  if (coarse.n == 0) return;
  if (coarse.radius == 3) {  // quadratic embedding
    const int fr = fine.radius;
    const int smem = kGqWarps * 9 * level_pitch(fr) * 8;
    const void* fx = fr == 2 ? (const void*)k_galerkin_qx<2> : (const void*)k_galerkin_qx<3>;
    set_max_dynamic_smem(fx, smem);
    const int bx = mgrid((long long)fine.n * 32, kGqWarps * 32);
    const int bc = mgrid((long long)coarse.n * 32, kMgThreads);
    if (fr == 2) {
      k_galerkin_qx<2><<<bx, kGqWarps * 32, smem, s>>>(fine, X);
      k_galerkin_qc<2><<<bc, kMgThreads, 0, s>>>(fine, coarse, X);
    } else {
      k_galerkin_qx<3><<<bx, kGqWarps * 32, smem, s>>>(fine, X);
      k_galerkin_qc<3><<<bc, kMgThreads, 0, s>>>(fine, coarse, X);
    }
    count_launches(2);
    return;
  }
  // 8 warps x 1 row buffer.  cfg2 hierarchy phase per step: 8x1 0.973 ms, 4x1 / 6x1 0.982, 4x2
  // 1.044, 16x1 1.048, 4x3 1.188, 8x2 1.208: more warps in flight beat a deeper ring
  launch_galerkin_x_t<8, 1>(fine, X, s);
  if (coarse.hi > coarse.lo) {
    k_galerkin_c<<<mgrid((long long)(coarse.hi - coarse.lo) * 32, kMgThreads), kMgThreads, 0, s>>>(fine, coarse, X);
    count_launches(1);
  }
}
void launch_level_dinv(LevelView L, int* singular_flag, cudaStream_t s) {
  if (L.hi > L.lo) { k_level_dinv<<<mgrid(L.hi - L.lo, 256), 256, 0, s>>>(L, singular_flag); count_launches(1); }
}
void launch_level_waves(LevelView L, int coarse, int modulus, const int* off, int* wave_of, cudaStream_t s) {
  if (L.n) { k_level_waves<<<mgrid(L.n, 256), 256, 0, s>>>(L, coarse, modulus, off[0], off[1], off[2], wave_of); count_launches(1); }
}
int bucket_scratch_ints(int n, int nwaves) {
  const long long nb = std::max(1, (n + kBucketRows - 1) / kBucketRows);
  return (int)(2 * (nb * nwaves + 1) + 2);
}
void launch_bucket_rows(const int* wave_of, int n, int wmin, int* counts, int* start, int* cursor, int* rows,
                        int nwaves, int* scan_tmp, cudaStream_t s, int row_base) {
  wave_of += row_base;
  const int nb = std::max(1, (n + kBucketRows - 1) / kBucketRows);
  const long long len = (long long)nb * nwaves + 1;
  int* bc = cursor;         // (wave, block) counts, wave-major, + the total slot
  int* off = cursor + len;  // their exclusive scan
  const size_t sm = sizeof(int) * (size_t)std::max(nwaves, 1);
  set_max_dynamic_smem((const void*)k_wave_block_count, (int)sm);
  set_max_dynamic_smem((const void*)k_wave_block_scatter, (int)sm);
  if (n) {
    k_wave_block_count<<<nb, 256, sm, s>>>(wave_of, n, wmin, nwaves, bc);
  } else {
    cudaMemsetAsync(bc, 0, sizeof(int) * len, s);
  }
  launch_exclusive_scan(bc, off, (int)len, scan_tmp, nullptr, s);
  k_wave_totals<<<std::max(1, (nwaves + 256) / 256), 256, 0, s>>>(off, nb, nwaves, counts, start);
  if (n) k_wave_block_scatter<<<nb, 32, sm, s>>>(wave_of, n, wmin, nwaves, off, rows, row_base);
  count_launches(n ? 3 : 1);
}
void launch_plane_starts(const int* coords, int n, int lo0, int nplanes, int* out, cudaStream_t s) {
  k_plane_starts<<<mgrid(nplanes + 1, 128), 128, 0, s>>>(coords, n, lo0, nplanes, out);
  count_launches(1);
}
void launch_sgs_wave1(LevelView L, const int* rows, int cnt, double* u, const double* b, cudaStream_t s) {
  if (cnt <= 0) return;
  k_sgs_wave<<<(cnt + kWaveThreads / 32 - 1) / (kWaveThreads / 32), kWaveThreads, 0, s>>>(L, rows, cnt, u, b, 0);
  count_launches(1);
}
void launch_spmv(LevelView L, const double* x, double* y, cudaStream_t s) {
  if (L.hi <= L.lo) return;
  if (L.radius == 2)
    k_spmv<2><<<mgrid((long long)(L.hi - L.lo) * 32, kMgThreads), kMgThreads, 0, s>>>(L, x, y, nullptr);
  else
    k_spmv<3><<<mgrid((long long)(L.hi - L.lo) * 32, kMgThreads), kMgThreads, 0, s>>>(L, x, y, nullptr);
  count_launches(1);
}
void launch_residual(LevelView L, const double* b, const double* u, double* r, cudaStream_t s) {
  if (L.hi <= L.lo) return;
  if (L.radius == 2)
    k_spmv<2><<<mgrid((long long)(L.hi - L.lo) * 32, kMgThreads), kMgThreads, 0, s>>>(L, u, r, b);
  else
    k_spmv<3><<<mgrid((long long)(L.hi - L.lo) * 32, kMgThreads), kMgThreads, 0, s>>>(L, u, r, b);
  count_launches(1);
}
void launch_restrict(LevelView fine, LevelView coarse, const double* rf, double* bc, cudaStream_t s) {
  const int quad = coarse.radius == 3;  // quadratic-embedding coarse levels carry radius 3
  if (coarse.n) { k_restrict<<<mgrid(coarse.n, 128), 128, 0, s>>>(fine, coarse, quad, rf, bc); count_launches(1); }
}
void launch_prolong_add(LevelView fine, LevelView coarse, const double* uc, double* uf, cudaStream_t s) {
  const int quad = coarse.radius == 3;
  if (fine.n) { k_prolong_add<<<mgrid(fine.n, 128), 128, 0, s>>>(fine, coarse, quad, uc, uf); count_launches(1); }
}
void launch_sgs(LevelView L, const int* wave_start, const int* wave_rows, int nwaves, double* u, const double* b,
                int grid_blocks, unsigned int* bar, cudaStream_t s, long long* trace) {
  if (L.n == 0 || nwaves == 0) return;
  cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned int), s);
  void* args[] = {&L, (void*)&wave_start, (void*)&wave_rows, &nwaves, &u, (void*)&b, &trace, &bar};
  { cudaLaunchCooperativeKernel((const void*)k_sgs, grid_blocks, kSgsThreads, args, kSgsSmem, s); count_launches(1); }
}

template <int W, int S>
int sgs_stream_blocks_t() {
  return coop_blocks((const void*)k_sgs_stream<W, S>, W * 32, stream_smem<W, S>());
}

template <int W, int S>
void launch_sgs_stream_t(LevelView L, const int* wave_start, const int* wave_rows, int nwaves, double* u,
                         const double* b, unsigned int* bar, cudaStream_t s, int q_lo, int q_hi, int max_rows) {
  // fewer CTAs when no wave has rows for all warps: the grid barrier costs grow with the CTA count
  int grid = sgs_stream_blocks_t<W, S>();
  if (max_rows > 0) grid = std::max(1, std::min(grid, (max_rows + W - 1) / W));
  void* args[] = {&L, (void*)&wave_start, (void*)&wave_rows, &nwaves, &u, (void*)&b, &bar, &q_lo, &q_hi};
  cudaLaunchCooperativeKernel((const void*)k_sgs_stream<W, S>, grid, W * 32, args, stream_smem<W, S>(), s);
  count_launches(1);
}

int sgs_stream_blocks() { return sgs_stream_blocks_t<8, 2>(); }


void launch_sgs_stream(LevelView L, const int* wave_start, const int* wave_rows, int nwaves, double* u,
                       const double* b, unsigned int* bar, cudaStream_t s, int q_lo, int q_hi, int max_rows) {
  if (L.n == 0 || nwaves == 0) return;
  if (q_hi < 0) q_hi = 2 * nwaves;
  if (q_hi <= q_lo) return;
  cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned int), s);
  // 8 warps x 2 ring stages per CTA.  cfg2 level-0 smoother per step: 8x2 1.52 ms, 16x1 1.52,
  // 6x3 1.57, 4x4 1.78, 4x5 1.85: the limit is rows in flight, not bytes in flight
  launch_sgs_stream_t<8, 2>(L, wave_start, wave_rows, nwaves, u, b, bar, s, q_lo, q_hi, max_rows);
}

void launch_sgs_waves(LevelView L, const int* wave_start_host, const int* wave_rows, int nwaves, double* u,
                      const double* b, cudaStream_t s) {
  constexpr int pdl = 1;  // programmatic dependent launch between consecutive waves
  for (int pass = 0; pass < 2; ++pass)
    for (int k = 0; k < nwaves; ++k) {
      const int w = pass == 0 ? k : nwaves - 1 - k;
      const int cnt = wave_start_host[w + 1] - wave_start_host[w];
      if (cnt == 0) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)((cnt + kWaveThreads / 32 - 1) / (kWaveThreads / 32)));
      cfg.blockDim = dim3(kWaveThreads);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl ? 1 : 0;
      const int* rw = wave_rows + wave_start_host[w];
      cudaLaunchKernelEx(&cfg, k_sgs_wave, L, rw, cnt, u, b, pdl);
      count_launches(1);
    }
}

void launch_pcg(LevelView L, const double* b, double* x, double* r, double* z, double* p, double* Ap, double rel,
                int cap, double* partials, int* stat, int* iter_acc, int grid_blocks, cudaStream_t s) {
  void* args[] = {&L, (void*)&b, &x, &r, &z, &p, &Ap, &rel, &cap, &partials, &stat, &iter_acc};
  const void* fn = L.radius == 2 ? (const void*)k_pcg<2> : (const void*)k_pcg<3>;
  { cudaLaunchCooperativeKernel(fn, grid_blocks, kMgThreads, args, 0, s); count_launches(1); }
}

}  // namespace hotb200
