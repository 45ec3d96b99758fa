// Stage 2 (One-to-many attention, attention.hpp:207-252) fused on the
// sm_100a tensor core, C = 32, h <= 4 heads, M views:
//
//   n      = rms_norm(V) * g                     (SIMT, thread = texel)
//   S      = n [Wq_0 | ... | Wq_{h-1}]           tcgen05.mma kind::f16, 3-term
//                                                fp16 split, M=128, TMEM
//   l_im   = <S_i, Δ_m> / sqrt(C); w = softmax_m; head_i = sum_m w_im Δ_m
//   O      = sum_i head_i Wo_i                   tcgen05.mma kind::f16, split
//   V     += O
//
// The projections use the conv's fp16 split (tc::split_f16, same ~2^-22
// relative error per product as 3xTF32): per 16-channel K step
//   MMA1 N=64h: D[:, 0:64h] (+)= Xh * [Wh ; Wl']^T,   MMA2 N=32h: D[:, 32h:64h] += Xl' * Wh^T
// and S = D[:, c] + 2^-11 D[:, 32h + c] (likewise O with h = 1).
//
// Persistent warp-specialised CTA, one per SM, 128-texel tiles:
//   w0     TMA producer: V tiles (128B-swizzled, 4 buffers, one tile ahead of
//          the Δ slices) and, per view, the tile's Δ slice [128 texels][32]
//          (one 2-D TMA box over Δ[m][p][32], 128B-swizzled) into an NS-deep
//          ring -- twice per tile (scores, then mix; the second read hits L2)
//   w1     MMA issuer (one elected lane; warp-uniform descriptors)
//   w2-5   consumers (and w6-9 for h >= 2: the heads split over two groups),
//          thread <-> texel row <-> TMEM lane, software-pipelined
//          across tiles so neither MMA round trip is on the critical path:
//            scores(i) [S(i) requested an iteration earlier] -> finish(i-1)
//            [O(i-1) + V, TMA store] -> stage n(i+1) -> mix(i) -> stage heads(i)
// Weights are split once per CTA and stay resident (K-major interleave).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstring>

#include "host.h"
#include "kernels.h"
#include "tc.cuh"

namespace lvsg {
namespace {

constexpr int C = 32;
constexpr int TILE = 128;
constexpr int NCONS = 128;                 // threads of one consumer group
constexpr int NJ = C / 8;                  // 8-channel fp16 K chunks
constexpr int NG = C / 4;                  // 4-channel Δ groups
constexpr int A_LBO = TILE * 16;           // 2 KB: one 8-channel plane of 128 rows
constexpr int A_HALF = NJ * A_LBO;         // 8 KB: hi (or lo') planes
constexpr int A_BYTES = 2 * A_HALF;        // 16 KB per staging buffer
constexpr int V_BYTES = TILE * C * 4;      // 16 KB
constexpr int D_BYTES = TILE * C * 4;      // one view slice [128][32] fp32, 16 KB
constexpr int NV = 4;                      // V tile buffers

// h >= 2: two consumer groups (warps 2-5, 6-9) split the heads over the same
// texels, so two consumer warps share each SM sub-partition
template <int H>
constexpr int groups() {
  return H >= 2 ? 2 : 1;
}
template <int H>
constexpr int nthreads() {
  return 64 + NCONS * groups<H>();
}

template <int H>
constexpr uint32_t tmem_cols() {  // S (64h columns) + O (64 columns), power of two
  return H == 1 ? 128u : H == 2 ? 256u : 512u;
}

template <int H>
struct Smem {
  static constexpr int BQ_ROWS = 64 * H;            // [Wq hi ; Wq lo'] rows
  static constexpr int BQ_LBO = BQ_ROWS * 16;
  static constexpr int BQ_BYTES = NJ * BQ_LBO;
  static constexpr int BO_LBO = 64 * 16;            // per head [Wo hi ; Wo lo']
  static constexpr int BO_BYTES = NJ * BO_LBO;
  static constexpr int OFF_V = 0;                   // NV buffers, 1 KB aligned (swizzle)
  static constexpr int OFF_A = OFF_V + NV * V_BYTES;
  static constexpr int OFF_BQ = OFF_A + 2 * A_BYTES;
  static constexpr int OFF_BO = OFF_BQ + BQ_BYTES;
  static constexpr int OFF_D = OFF_BO + H * BO_BYTES;
  static constexpr int BUDGET = 227 * 1024 - 512;
  static constexpr int NS = (BUDGET - OFF_D) / D_BYTES > 8 ? 8 : (BUDGET - OFF_D) / D_BYTES;
  static constexpr int OFF_BAR = OFF_D + NS * D_BYTES;
  // bars: v_full[NV] v_empty[NV] d_full[NS] d_empty[NS] a_full[2] a_free[2] s_done o_done
  // s_free w_full o_free
  static constexpr int NBAR = 2 * NV + 2 * NS + 4 + 5;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16;
  static_assert(NS >= 3, "shared memory budget");
  static_assert(OFF_D % 1024 == 0 && OFF_V % 1024 == 0, "128B-swizzled TMA destinations");
};

// A[j][row][8 halves] (hi) and A[4 + j][row] (lo') <- x[32] of this row;
// returns whether a value overflows the split (tc::split_overflows).
__device__ __forceinline__ bool stage_row(uint8_t* a, int row, const float* x) {
  bool ovf = false;
#pragma unroll
  for (int c = 0; c < C; ++c) ovf |= tc::split_overflows(x[c]);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    __align__(16) __half2 h[4], l[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) tc::split_f16x2(x[8 * j + 2 * k], x[8 * j + 2 * k + 1], h[k], l[k]);
    *reinterpret_cast<uint4*>(a + j * A_LBO + row * 16) = *reinterpret_cast<uint4*>(h);
    *reinterpret_cast<uint4*>(a + A_HALF + j * A_LBO + row * 16) = *reinterpret_cast<uint4*>(l);
  }
  return ovf;
}

// B rows (K-major interleave): w(n, k) for n < N, hi in rows [0, N), lo' in [N, 2N).
template <typename F>
__device__ __forceinline__ bool stage_weights(uint8_t* b, int N, int tid, int nt, F w) {
  __half* bh = reinterpret_cast<__half*>(b);
  bool ovf = false;
  for (int e = tid; e < NJ * N * 8; e += nt) {
    const int k8 = e & 7, n = (e >> 3) % N, j = (e >> 3) / N;
    __half hi, lo;
    const float x = w(n, 8 * j + k8);
    tc::split_f16(x, hi, lo);
    ovf |= tc::split_overflows(x);
    bh[(j * 2 * N + n) * 8 + k8] = hi;
    bh[(j * 2 * N + N + n) * 8 + k8] = lo;
  }
  return ovf;
}

// D (+)= A * B over K = 32: MMA1 N = 2n into d, MMA2 N = n (lo' x hi) into d + n.
__device__ __forceinline__ void mma_split(uint32_t d, uint32_t a, uint32_t b, int n, bool acc0) {
  const uint32_t id1 = tc::idesc_f16(128, 2 * n), id2 = tc::idesc_f16(128, n);
  const uint64_t ah = tc::smem_desc(a, A_LBO, 128), al = tc::smem_desc(a + A_HALF, A_LBO, 128);
  const uint64_t bd = tc::smem_desc(b, 2 * n * 16, 128);
#pragma unroll
  for (int s = 0; s < NJ / 2; ++s) {
    const uint64_t ao = uint64_t((2 * s * A_LBO) >> 4), bo = uint64_t((2 * s * 2 * n * 16) >> 4);
    tc::mma_f16(d, ah + ao, bd + bo, id1, (acc0 || s > 0) ? 1u : 0u);
    tc::mma_f16(d + uint32_t(n), al + ao, bd + bo, id2, 1u);
  }
}

__device__ __forceinline__ uint32_t swz(int r, int c4) {  // 128B-swizzled [rows][128 B]
  return uint32_t(r * 128 + ((c4 ^ (r & 7)) << 4));
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const void* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
#ifndef LVSG_ATT_PF
#define LVSG_ATT_PF 1
#endif
#ifndef LVSG_ATT_INTERLEAVE
#define LVSG_ATT_INTERLEAVE 0
#endif
#ifndef LVSG_ATT_PFPOS
#define LVSG_ATT_PFPOS 1
#endif
#ifndef LVSG_ATT_PFMIN
#define LVSG_ATT_PFMIN 4
#endif
__device__ __forceinline__ void tma_store_2d(const void* map, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// MM: the view count (EXACT) or, for other counts, an upper bound on the
// runtime view count Mr (views m >= Mr are skipped; MM in {8, 16, 32}).
template <int H, int MM, bool EXACT>
__global__ void __launch_bounds__(nthreads<H>(), 1)
    attend_tc_kernel(const __grid_constant__ CUtensorMap vmap,
                     const __grid_constant__ CUtensorMap dmap, int64_t P,
                     const float* __restrict__ wq, const float* __restrict__ wo,
                     const float* __restrict__ gain, int zero_scores, int num_tiles, int Mr,
                     const uint8_t* __restrict__ wimg, int wimg_early, int* ovf_flag) {
  const int M = EXACT ? MM : Mr;
  auto has = [&](int m) { return EXACT || m < Mr; };
  using S = Smem<H>;
  constexpr int NS = S::NS;
  constexpr int NTH = nthreads<H>(), NGRP = groups<H>(), HG = H / NGRP;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint64_t* v_full = bars;            // [NV] V tile landed
  uint64_t* v_empty = bars + NV;      // [NV] V tile stored back (buffer free)
  uint64_t* d_full = bars + 2 * NV;   // [NS] Δ slice landed
  uint64_t* d_empty = d_full + NS;    // [NS] consumers done with the slice
  uint64_t* a_full = d_empty + NS;    // [2] A operand staged
  uint64_t* a_free = a_full + 2;      // [2] MMAs done reading A
  uint64_t* s_done = a_free + 2;      // S ready
  uint64_t* o_done = s_done + 1;      // O ready
  uint64_t* s_free = o_done + 1;      // every consumer has read S (TMEM S may be rewritten)
  uint64_t* w_full = s_free + 1;      // pre-split weight image landed (wimg != nullptr)
  uint64_t* o_free = w_full + 1;      // the finishing group has read O (TMEM O may be rewritten)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::NBAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  tc::pdl_launch_dependents();
  if (blockIdx.x >= num_tiles) return;
  const uint32_t sb = tc::smem_u32(smem);
  if (tid == 0 && (sb & 1023u)) __trap();  // swizzle atoms need 1 KB alignment
  const int passes = zero_scores ? 1 : 2;
  const int ntl = (num_tiles - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);  // my tiles
  auto tile_of = [&](int i) { return int(blockIdx.x) + i * int(gridDim.x); };

  // resident weights: Bq rows n = 32*i + c -> Wq_i[k][c]; Bo_i rows n -> Wo[32i + k][n]
  // (split here unless the context's pre-split image is given: one bulk copy)
  bool ovf = false;  // an fp16-split operand overflowed (reported once per thread)
  if (!wimg) {
    ovf |= stage_weights(smem + S::OFF_BQ, 32 * H, tid, NTH,
                         [&](int n, int k) { return __ldg(wq + ((n >> 5) * C + k) * C + (n & 31)); });
    for (int h = 0; h < H; ++h)
      ovf |= stage_weights(smem + S::OFF_BO + h * S::BO_BYTES, 32, tid, NTH,
                           [&](int n, int k) { return __ldg(wo + (h * C + k) * C + n); });
  }
  if (tid == 0) {
    for (int k = 0; k < NV; ++k) {
      tc::mbar_init(&v_full[k], 1);
      tc::mbar_init(&v_empty[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(&a_full[k], NCONS);
      tc::mbar_init(&a_free[k], 1);
    }
    for (int k = 0; k < NS; ++k) {
      tc::mbar_init(&d_full[k], 1);
      tc::mbar_init(&d_empty[k], NCONS * NGRP);
    }
    tc::mbar_init(s_done, 1);
    tc::mbar_init(o_done, 1);
    tc::mbar_init(s_free, NCONS * NGRP);
    tc::mbar_init(w_full, 1);
    tc::mbar_init(o_free, NCONS);
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, tmem_cols<H>());
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const uint32_t tmem_s = tmem, tmem_o = tmem + 64 * H;
  // a settled weight image loads under the previous kernel's tail, a fresh
  // one after the wait
  if (wimg && wimg_early && tid == 0) {
    tc::mbar_expect_tx(w_full, S::BQ_BYTES + H * S::BO_BYTES);
    tc::bulk_load(sb + S::OFF_BQ, wimg, S::BQ_BYTES + H * S::BO_BYTES, w_full);
  }
  tc::pdl_wait();  // the prologue above overlaps the previous kernel (weights are static)
  if (wimg && !wimg_early && tid == 0) {
    tc::mbar_expect_tx(w_full, S::BQ_BYTES + H * S::BO_BYTES);
    tc::bulk_load(sb + S::OFF_BQ, wimg, S::BQ_BYTES + H * S::BO_BYTES, w_full);
  }

  if (warp == 0) {
    // ---- producer: V(i+1) is issued before tile i's slices ----
    if (lane == 0) {
      int k = 0;
      auto load_v = [&](int j) {
        const int vb = j % NV;
        if (j >= NV) tc::mbar_wait(&v_empty[vb], uint32_t((j / NV - 1) & 1));
        tc::mbar_expect_tx(&v_full[vb], V_BYTES);
        tma_load_2d(sb + S::OFF_V + vb * V_BYTES, &vmap, 0, tile_of(j) * TILE, &v_full[vb]);
      };
      load_v(0);
      for (int i = 0; i < ntl; ++i) {
        if (i + 1 < ntl) load_v(i + 1);
        // one 2-D box per view slice: rows m P + [128 i, 128 i + 128) of Δ[M P][32]
        // (rows past P of a view are the next view's, never used; past M P: zero)
        for (int pass = 0; pass < passes; ++pass) {
          // the next tile's Δ slices into L2 (CTAs with a few tiles
          // excepted): its first (scores) pass then waits on L2, not HBM
          if (LVSG_ATT_PF > 0 && pass == LVSG_ATT_PFPOS && ntl > LVSG_ATT_PFMIN && i + 1 < ntl)
            for (int m = 0; m < M; ++m)
              tma_prefetch_2d(&dmap, 0, int(m * P) + tile_of(i + 1) * TILE);
          for (int m = 0; m < M; ++m, ++k) {
            const int sl = k % NS;
            if (k >= NS) tc::mbar_wait(&d_empty[sl], uint32_t((k / NS - 1) & 1));
            tc::mbar_expect_tx(&d_full[sl], D_BYTES);
            tma_load_2d(sb + S::OFF_D + sl * D_BYTES, &dmap, 0, int(m * P) + tile_of(i) * TILE,
                        &d_full[sl]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: S(first); per tile i: S(i+1), then O over the heads ----
    // A operand stagings in issue order: n(0); per tile i: n(i+1) (group 0),
    // then heads 0 .. H-1 (head h by group h / HG). One consumer group: two
    // buffers used alternately; two groups: buffer g belongs to group g, so
    // every a_free phase a group waits on follows one it waited on itself
    // (a parity wait is exact only when the waiter is at most one phase
    // behind -- with shared buffers one group could pass a stale parity of a
    // buffer whose previous use belonged to the other group)
    int ca[2] = {0, 0}, ns = 0;
    if (wimg) tc::mbar_wait(w_full, 0);
    auto next_a = [&](int owner) {
      const int b = NGRP == 1 ? (ca[0] & 1) : owner;
      const uint32_t ph = NGRP == 1 ? uint32_t((ca[0] >> 1) & 1) : uint32_t(ca[owner] & 1);
      tc::mbar_wait(&a_full[b], ph);
      ++ca[NGRP == 1 ? 0 : owner];
      __syncwarp();
      tc::fence_after();
      return b;
    };
    auto issue_s = [&]() {
      const int b = next_a(0);
      // S lives in one TMEM accumulator: S(j) is written only once every
      // consumer of both groups has read S(j-1) (with two groups the ring lets
      // one group run up to NS slices ahead of the other)
      if (ns > 0) tc::mbar_wait(s_free, uint32_t((ns - 1) & 1));
      ++ns;
      __syncwarp();
      tc::fence_after();
      if (tc::elect_one()) {
        mma_split(tmem_s, sb + S::OFF_A + b * A_BYTES, sb + S::OFF_BQ, 32 * H, false);
        tc::commit(s_done);
        tc::commit(&a_free[b]);
      }
      __syncwarp();
    };
    issue_s();
    for (int i = 0; i < ntl; ++i) {
      if (i + 1 < ntl) issue_s();
      // heads in order (O sums the heads in the reference's K order); with
      // LVSG_ATT_INTERLEAVE the two groups' heads alternate (0, HG, 1, ...),
      // so neither group's first staging waits behind the other's last
      // (~3% faster at H = 4, but a different rounding of O)
      for (int k = 0; k < H; ++k) {
        const int h = (NGRP == 2 && LVSG_ATT_INTERLEAVE) ? (k & 1) * HG + (k >> 1) : k;
        const int b = next_a(h / HG);
        if (NGRP == 2 && k == 0 && i > 0) {
          // two groups: group 1 reads O(i-1) (finish_tile) while group 0
          // already stages head 0 of tile i; O(i) overwrites it only after
          tc::mbar_wait(o_free, uint32_t((i - 1) & 1));
          tc::fence_after();
        }
        if (tc::elect_one()) {
          mma_split(tmem_o, sb + S::OFF_A + b * A_BYTES, sb + S::OFF_BO + h * S::BO_BYTES, 32,
                    k > 0);
          if (k == H - 1) tc::commit(o_done);
          tc::commit(&a_free[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- consumers: group grp owns heads [grp*HG, (grp+1)*HG); group 0 also
    //      stages n and writes V back ----
    const int grp = (warp - 2) >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;  // texel row of the tile == TMEM lane
    const uint32_t lane_base = uint32_t(q * 32) << 16;
    const float inv_temp = __double2float_rn(1.0 / sqrt(double(C)));
    // two groups: group 0 starts tiles (rms-norm, n staging) and group 1
    // finishes them (O + V, TMA store), so neither group runs behind the
    // other on the Δ ring the two share
    const int fin_grp = NGRP - 1;
    const bool storer = warp == 2 + 4 * fin_grp && lane == 0;
    int k = 0;
    // A stagings (the MMA issuer consumes them in the same order): group 0
    // stages n(0), then per tile n(i+1) and its heads; group 1 its heads.
    // cs counts this group's stagings (see next_a for the buffers).
    int cs = 0;
    auto stage = [&](const float* x) {
      const int b = NGRP == 1 ? (cs & 1) : grp;
      if (NGRP == 1 ? cs >= 2 : cs >= 1)
        tc::mbar_wait(&a_free[b], NGRP == 1 ? uint32_t(((cs >> 1) - 1) & 1) : uint32_t((cs - 1) & 1));
      ovf |= stage_row(smem + S::OFF_A + b * A_BYTES, row, x);
      tc::fence_proxy_async();
      tc::mbar_arrive(&a_full[b]);
      ++cs;
    };
    auto slice_row = [&](float* dm) {  // this texel's row of the next Δ slice
      const int sl = k % NS;
      tc::mbar_wait(&d_full[sl], uint32_t((k / NS) & 1));
      const uint8_t* d = smem + S::OFF_D + sl * D_BYTES;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const float4 t = *reinterpret_cast<const float4*>(d + swz(row, g));
        dm[4 * g] = t.x, dm[4 * g + 1] = t.y, dm[4 * g + 2] = t.z, dm[4 * g + 3] = t.w;
      }
      // these generic-proxy reads must be ordered before the TMA (async
      // proxy) that refills the slot once the last consumer arrives: without
      // the proxy fence the last arriver's loads can return the next slice
      tc::fence_proxy_async();
      tc::mbar_arrive(&d_empty[sl]);
      ++k;
    };
    auto tmem_split = [&](uint32_t col, int n, float* out) {  // D[:, col] + 2^-11 D[:, col + n]
      float lo[32];
      tc::tmem_ld32(lane_base + col, out);
      tc::tmem_ld32(lane_base + col + uint32_t(n), lo);
#pragma unroll
      for (int c = 0; c < 32; ++c) out[c] = fmaf(lo[c], 1.0f / tc::kF16LoScale, out[c]);
    };
    auto start_tile = [&](int j) {  // n = rms_norm(V) * g -> A (requests S(j)); group 0
      const int vb = j % NV;
      const uint8_t* vt = smem + S::OFF_V + vb * V_BYTES;
      tc::mbar_wait(&v_full[vb], uint32_t((j / NV) & 1));
      float x[C];
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 t = *reinterpret_cast<const float4*>(vt + swz(row, c4));
        x[4 * c4] = t.x, x[4 * c4 + 1] = t.y, x[4 * c4 + 2] = t.z, x[4 * c4 + 3] = t.w;
      }
      float ms = 0.f;
#pragma unroll
      for (int c = 0; c < C; ++c) ms = fmaf(x[c], x[c], ms);
      const float r = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(ms, float(C)), 1e-6f)));
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = fm(fm(x[c], r), __ldg(gain + c));
      stage(x);
    };
    auto finish_tile = [&](int j) {  // V(j) += O(j), TMA store; group fin_grp
      const int vb = j % NV;
      uint8_t* vt = smem + S::OFF_V + vb * V_BYTES;
      // the finishing group's own acquire of the V tile (group 0 waited for
      // it in start_tile; the buffer is refilled only after this store)
      if (NGRP == 2) tc::mbar_wait(&v_full[vb], uint32_t((j / NV) & 1));
      tc::mbar_wait(o_done, uint32_t(j & 1));
      tc::fence_after();
      float o[C];
      tmem_split(tmem_o, 32, o);
      tc::fence_before();
      if (NGRP == 2) tc::mbar_arrive(o_free);
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        float4* pv = reinterpret_cast<float4*>(vt + swz(row, c4));
        float4 t = *pv;
        t.x = fa(t.x, o[4 * c4]);
        t.y = fa(t.y, o[4 * c4 + 1]);
        t.z = fa(t.z, o[4 * c4 + 2]);
        t.w = fa(t.w, o[4 * c4 + 3]);
        *pv = t;
      }
      tc::fence_proxy_async();
      named_sync(1, NCONS);
      if (storer) {
        if (j > 0) {  // the previous store has left its buffer: hand it back
          tc::bulk_wait_read<0>();
          tc::mbar_arrive(&v_empty[(j - 1) % NV]);
        }
        tma_store_2d(&vmap, sb + S::OFF_V + vb * V_BYTES, 0, tile_of(j) * TILE);
        tc::bulk_commit();
      }
    };

    if (grp == 0) start_tile(0);
    for (int i = 0; i < ntl; ++i) {
      // ---- scores(i) for this group's heads: S in registers, one pass over Δ ----
      float w[HG][MM];
      if (zero_scores) {
#pragma unroll
        for (int h = 0; h < HG; ++h)
#pragma unroll
          for (int m = 0; m < MM; ++m) w[h][m] = has(m) ? __fdiv_rn(1.0f, float(M)) : 0.f;
        tc::mbar_arrive(s_free);
      } else {
        float sv[HG][C];
        tc::mbar_wait(s_done, uint32_t(i & 1));
        tc::fence_after();
#pragma unroll
        for (int h = 0; h < HG; ++h)
          tmem_split(tmem_s + uint32_t(32 * (grp * HG + h)), 32 * H, sv[h]);
        tc::fence_before();
        tc::mbar_arrive(s_free);
        // views in pairs, each dot as 4 interleaved partial sums: 8 independent
        // 8-deep FMA chains instead of one 32-deep chain per (view, head)
#pragma unroll
        for (int m = 0; m < MM; m += 2) {
          if (!has(m)) break;
          float d0[C], d1[C];
          slice_row(d0);
          if (has(m + 1))
            slice_row(d1);
          else
#pragma unroll
            for (int c = 0; c < C; ++c) d1[c] = 0.f;
#pragma unroll
          for (int h = 0; h < HG; ++h) {
            // 4 interleaved partial sums per dot as two packed f32x2 pairs
            // (FFMA2: the same per-lane roundings and order)
            float2 a0[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float2 a1[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int c = 0; c < C; c += 4) {
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                const float2 s2 = make_float2(sv[h][c + 2 * r], sv[h][c + 2 * r + 1]);
                a0[r] = __ffma2_rn(s2, make_float2(d0[c + 2 * r], d0[c + 2 * r + 1]), a0[r]);
                a1[r] = __ffma2_rn(s2, make_float2(d1[c + 2 * r], d1[c + 2 * r + 1]), a1[r]);
              }
            }
            w[h][m] = fm(fa(fa(a0[0].x, a0[0].y), fa(a0[1].x, a0[1].y)), inv_temp);
            w[h][m + 1] = fm(fa(fa(a1[0].x, a1[0].y), fa(a1[1].x, a1[1].y)), inv_temp);
          }
        }
        // softmax over views (tape.hpp:390-404: max, exp(x - max), sum, * 1/sum)
#pragma unroll
        for (int h = 0; h < HG; ++h) {
          float mx = w[h][0];
#pragma unroll
          for (int m = 1; m < MM; ++m)
            if (has(m)) mx = fmaxf(mx, w[h][m]);
          float sum = 0.f;
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            w[h][m] = has(m) ? expf(fsb(w[h][m], mx)) : 0.f;
            if (has(m)) sum = fa(sum, w[h][m]);
          }
          const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
          for (int m = 0; m < MM; ++m) w[h][m] = fm(w[h][m], inv);
        }
      }
      if (grp == fin_grp && i > 0) finish_tile(i - 1);
      if (grp == 0 && i + 1 < ntl) start_tile(i + 1);
      // ---- mix(i): this group's heads in one pass over Δ ----
      float hd[HG][C];
#pragma unroll
      for (int h = 0; h < HG; ++h)
#pragma unroll
        for (int c = 0; c < C; ++c) hd[h][c] = 0.f;
#pragma unroll
      for (int m = 0; m < MM; m += 2) {
        if (!has(m)) break;
        float d0[C], d1[C];
        slice_row(d0);
        if (has(m + 1))
          slice_row(d1);
        else
#pragma unroll
          for (int c = 0; c < C; ++c) d1[c] = 0.f;
#pragma unroll
        for (int h = 0; h < HG; ++h) {
          const float2 wa = make_float2(w[h][m], w[h][m]), wb = make_float2(w[h][m + 1], w[h][m + 1]);
#pragma unroll
          for (int c = 0; c < C; c += 2) {
            float2 t = __ffma2_rn(wa, make_float2(d0[c], d0[c + 1]), make_float2(hd[h][c], hd[h][c + 1]));
            t = __ffma2_rn(wb, make_float2(d1[c], d1[c + 1]), t);
            hd[h][c] = t.x, hd[h][c + 1] = t.y;
          }
        }
      }
#pragma unroll
      for (int h = 0; h < HG; ++h) stage(hd[h]);
    }
    if (grp == fin_grp) {
      finish_tile(ntl - 1);
      if (storer) tc::bulk_wait<0>();
    }
  }
  if (ovf && ovf_flag) atomicOr(ovf_flag, 2);
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, tmem_cols<H>());
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

template <int H, int MM, bool EXACT>
void launch(float* V, const float* D, int64_t P, int M, const float* wq, const float* wo,
            const float* gain, int zero, const void* wimg, bool wimg_early, int* ovf,
            cudaStream_t st) {
  smem_optin(reinterpret_cast<const void*>(attend_tc_kernel<H, MM, EXACT>), Smem<H>::BYTES);
  const int sms = sm_count();
  // V [P][32] fp32 as a 2-D map, 128-texel boxes (128B swizzle)
  CUtensorMap vmap, dmap;
  std::memset(&vmap, 0, sizeof(vmap));
  std::memset(&dmap, 0, sizeof(dmap));
  {
    cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(P)};
    cuuint64_t strides[1] = {cuuint64_t(C) * 4};
    cuuint32_t box[2] = {cuuint32_t(C), cuuint32_t(TILE)};
    cuuint32_t estr[2] = {1, 1};
    if (encode_fn()(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, V, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      throw CudaError("attention: V tensor map");
  }
  {
    // Δ[m][p][32] as one 2-D map [M P rows][32 floats], 128-texel boxes (128B swizzle)
    cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(P) * cuuint64_t(M)};
    cuuint64_t strides[1] = {cuuint64_t(C) * 4};
    cuuint32_t box[2] = {cuuint32_t(C), cuuint32_t(TILE)};
    cuuint32_t estr[2] = {1, 1};
    if (encode_fn()(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(D), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      throw CudaError("attention: delta tensor map");
  }
  const int tiles = int((P + TILE - 1) / TILE);
  const int grid = tiles < sms ? tiles : sms;
  launch_pdl(true, attend_tc_kernel<H, MM, EXACT>, grid, nthreads<H>(), Smem<H>::BYTES, st, vmap,
             dmap, P, wq, wo, gain, zero, tiles, M, static_cast<const uint8_t*>(wimg),
             wimg_early ? 1 : 0, ovf);
}

// The weight image of attend_tc_kernel<H>'s resident B operands, in its
// shared-memory layout: [Wq hi ; Wq lo'] for all heads, then per head
// [Wo hi ; Wo lo'] (stage_weights), made once per weight binding.
template <int H>
__global__ void attend_tc_weights_kernel(const float* __restrict__ wq, const float* __restrict__ wo,
                                         uint8_t* out, int* ovf_flag) {
  pdl_grid_sync();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  bool ovf = stage_weights(out, 32 * H, tid, nt, [&](int n, int k) {
    return __ldg(wq + ((n >> 5) * C + k) * C + (n & 31));
  });
  for (int h = 0; h < H; ++h)
    ovf |= stage_weights(out + Smem<H>::BQ_BYTES + h * Smem<H>::BO_BYTES, 32, tid, nt,
                         [&](int n, int k) { return __ldg(wo + (h * C + k) * C + n); });
  if (ovf && ovf_flag) atomicOr(ovf_flag, 2);
}

}  // namespace

size_t attend_tc_weight_bytes(int heads) {
  switch (heads) {
    case 1: return Smem<1>::BQ_BYTES + Smem<1>::BO_BYTES;
    case 2: return Smem<2>::BQ_BYTES + 2 * Smem<2>::BO_BYTES;
    case 4: return Smem<4>::BQ_BYTES + 4 * Smem<4>::BO_BYTES;
    default: return 0;
  }
}

void attend_tc_prepare(const float* wq, const float* wo, int heads, void* dst, int* ovf,
                       cudaStream_t st) {
  uint8_t* o = static_cast<uint8_t*>(dst);
  switch (heads) {
    case 1: launch_k(attend_tc_weights_kernel<1>, 8, 256, 0, st, wq, wo, o, ovf); break;
    case 2: launch_k(attend_tc_weights_kernel<2>, 8, 256, 0, st, wq, wo, o, ovf); break;
    case 4: launch_k(attend_tc_weights_kernel<4>, 8, 256, 0, st, wq, wo, o, ovf); break;
    default: break;
  }
}

bool attend_tc_supported(int C_, int M, int heads) {
  return C_ == C && (heads == 1 || heads == 2 || heads == 4) && M >= 1 && M <= 32;
}

bool attend_tc(float* V, const float* deltas, int64_t P, int C_, int M, int heads, const float* wq,
               const float* wo, const float* gain, int zero_scores, const void* wimg,
               bool wimg_early, int* ovf, cudaStream_t st) {
  if (wimg && (reinterpret_cast<uintptr_t>(wimg) & 15)) return false;
  if (C_ != C || !encode_fn() || (reinterpret_cast<uintptr_t>(V) & 15) ||
      (reinterpret_cast<uintptr_t>(deltas) & 15) || P * M >= (int64_t(1) << 31))
    return false;
#define LVSG_ATT(HH)                                                                  \
  if (heads == HH) {                                                                  \
    switch (M) {                                                                      \
      case 2: launch<HH, 2, true>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st); break;   \
      case 4: launch<HH, 4, true>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st); break;   \
      case 8: launch<HH, 8, true>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st); break;   \
      case 16: launch<HH, 16, true>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st); break; \
      default:                                                                        \
        if (M < 8)                                                                    \
          launch<HH, 8, false>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st);       \
        else if (M < 16)                                                              \
          launch<HH, 16, false>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st);      \
        else                                                                          \
          launch<HH, 32, false>(V, deltas, P, M, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st);      \
    }                                                                                 \
    return true;                                                                      \
  }
  if (M < 1 || M > 32) return false;
  LVSG_ATT(1) LVSG_ATT(2) LVSG_ATT(4)
#undef LVSG_ATT
  return false;
}

}  // namespace lvsg
