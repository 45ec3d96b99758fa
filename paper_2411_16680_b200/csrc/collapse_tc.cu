// layer_collapse (network.hpp:440-455) on the sm_100a tensor core, C = 32:
//
//   cat = [a | b]                  (the two layers of a pair, K = 64)
//   h   = gelu(cat W1 + b1)        tcgen05.mma kind::f16, N = 64
//   out = (a + b) / 2 + (h W2 + b2)  tcgen05.mma kind::f16, N = 32
//
// with the conv's / attention's 3-term fp16 split (tc::split_f16: ~2^-22
// relative error per product, fp32 accumulation in TMEM). Per 64-channel K
// step pair: MMA1 N = 2n over [Wh ; Wl'] and MMA2 N = n with the lo' rows of
// the activations; the epilogue forms D[:, c] + 2^-11 D[:, n + c].
//
// One 128-texel tile per loop iteration (thread = texel row = TMEM lane):
// load a, b -> stage [a|b] -> MMA1 -> GELU epilogue -> stage h -> MMA2 ->
// output epilogue. No warp specialisation: two CTAs per SM (56 KB of shared
// memory and 256 TMEM columns each) overlap each other's phases. The split
// weight image is made once per weight binding (collapse_tc_prepare) and
// arrives by one bulk copy per CTA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include <algorithm>

#include "host.h"
#include "kernels.h"
#include "tc.cuh"

namespace lvsg {
namespace {

constexpr int C = 32;
constexpr int K1 = 2 * C;                     // [a | b]
constexpr int N1 = 2 * C;                     // hidden width
constexpr int N2 = C;                         // output width
constexpr int TILE = 128;
constexpr int NJ = K1 / 8;                    // 8-channel fp16 K chunks (both MMAs: K = 64)
constexpr int A_LBO = TILE * 16;              // one 8-channel plane of 128 rows
constexpr int A_HALF = NJ * A_LBO;            // hi (or lo') planes: 16 KB
constexpr int A_BYTES = 2 * A_HALF;           // 32 KB
constexpr int W1_BYTES = NJ * 2 * N1 * 16;    // [W1h ; W1l'] per chunk: 16 KB
constexpr int W2_BYTES = NJ * 2 * N2 * 16;    // 8 KB
constexpr int ROW_TILE = TILE * C * 4;         // one 128B-swizzled [128][32] fp32 tile, 16 KB
constexpr int OFF_A = 0;
constexpr int OFF_W1 = OFF_A + A_BYTES;
constexpr int OFF_W2 = OFF_W1 + W1_BYTES;
constexpr int OFF_IN = OFF_W2 + W2_BYTES;     // TMA path: the a and b row tiles (1 KB aligned)
constexpr int OFF_OUT = OFF_IN + 2 * ROW_TILE;  // TMA path: the output staging tile
constexpr int OFF_BAR = OFF_OUT + ROW_TILE;
constexpr int SMEM_USED = OFF_BAR + 4 * 8 + 16;
static_assert(OFF_IN % 1024 == 0 && OFF_OUT % 1024 == 0, "swizzled staging alignment");
// requested dynamic shared memory: caps residency at two CTAs per SM, so the
// 256-column TMEM allocations of co-resident CTAs always fit (512 columns)
constexpr int SMEM_BYTES = 110 * 1024;
constexpr uint32_t TMEM_COLS = 256;           // D1: 128 columns, D2: 64 columns
static_assert(SMEM_USED <= SMEM_BYTES, "shared memory layout");

// row `row` of a K = 8 NJK A operand (planes of A_LBO bytes; lo' planes at
// `half` bytes) <- x[8 NJK]; returns whether a value overflows the split
template <int NJK>
__device__ __forceinline__ bool stage_row_k(uint8_t* a, int half, int row, const float* x) {
  bool ovf = false;
#pragma unroll
  for (int j = 0; j < NJK; ++j) {
    __align__(16) __half2 h[4], l[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      tc::split_f16x2(x[8 * j + 2 * k], x[8 * j + 2 * k + 1], h[k], l[k]);
      ovf |= tc::split_overflows(x[8 * j + 2 * k]) | tc::split_overflows(x[8 * j + 2 * k + 1]);
    }
    *reinterpret_cast<uint4*>(a + j * A_LBO + row * 16) = *reinterpret_cast<uint4*>(h);
    *reinterpret_cast<uint4*>(a + half + j * A_LBO + row * 16) = *reinterpret_cast<uint4*>(l);
  }
  return ovf;
}
__device__ __forceinline__ bool stage_row64(uint8_t* a, int row, const float* x) {
  return stage_row_k<NJ>(a, A_HALF, row, x);
}

// D (=) A * B over K = 8 NJK: MMA1 N = 2n into d, MMA2 N = n (lo' x hi) into d + n.
template <int NJK>
__device__ __forceinline__ void mma_split_k(uint32_t d, uint32_t a, int half, uint32_t b, int n) {
  const uint32_t id1 = tc::idesc_f16(128, 2 * n), id2 = tc::idesc_f16(128, n);
  const uint64_t ah = tc::smem_desc(a, A_LBO, 128), al = tc::smem_desc(a + half, A_LBO, 128);
  const uint64_t bd = tc::smem_desc(b, 2 * n * 16, 128);
#pragma unroll
  for (int s = 0; s < NJK / 2; ++s) {
    const uint64_t ao = uint64_t((2 * s * A_LBO) >> 4), bo = uint64_t((2 * s * 2 * n * 16) >> 4);
    tc::mma_f16(d, ah + ao, bd + bo, id1, s > 0 ? 1u : 0u);
    tc::mma_f16(d + uint32_t(n), al + ao, bd + bo, id2, 1u);
  }
}
__device__ __forceinline__ void mma_split64(uint32_t d, uint32_t a, uint32_t b, int n) {
  mma_split_k<NJ>(d, a, A_HALF, b, n);
}

__device__ __forceinline__ void load_row32(const float* p, float* v) {
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int k = 0; k < C / 4; ++k) {
    const float4 t = __ldg(q + k);
    v[4 * k] = t.x, v[4 * k + 1] = t.y, v[4 * k + 2] = t.z, v[4 * k + 3] = t.w;
  }
}

__device__ __forceinline__ uint32_t swz128(int r, int c4) {  // 128B-swizzled [rows][128 B]
  return uint32_t(r * 128 + ((c4 ^ (r & 7)) << 4));
}
__device__ __forceinline__ void tma_load_rows(uint32_t dst, const CUtensorMap* map, int row,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_rows(const CUtensorMap* map, uint32_t src, int row) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(0), "r"(row)
               : "memory");
}

// kTma (PL a multiple of 128: a tile's texels are 128 consecutive rows of
// one layer pair): the a and b rows of the next tile arrive by two TMA boxes
// while this tile computes, and the output leaves through a 128B-swizzled
// staging tile and one TMA store; otherwise per-thread row loads / stores.
template <bool kTma>
__global__ void __launch_bounds__(TILE, 2)
    collapse_tc_kernel(const __grid_constant__ CUtensorMap vmap,
                       const __grid_constant__ CUtensorMap omap, const float* __restrict__ V,
                       int L2, int PL, const uint8_t* __restrict__ wimg,
                       const float* __restrict__ b1, const float* __restrict__ b2,
                       float* __restrict__ out, int num_tiles, int* ovf_flag) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* w_full = bars;       // weight image landed
  uint64_t* m1_done = bars + 1;  // h pre-activations in TMEM
  uint64_t* m2_done = bars + 2;  // outputs in TMEM
  uint64_t* in_full = bars + 3;  // kTma: the tile's a / b rows landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int tid = threadIdx.x, warp = tid >> 5;
  tc::pdl_launch_dependents();
  if (blockIdx.x >= num_tiles) return;
  const uint32_t sb = tc::smem_u32(smem);
  if (tid == 0) {
    tc::mbar_init(w_full, 1);
    tc::mbar_init(m1_done, 1);
    tc::mbar_init(m2_done, 1);
    tc::mbar_init(in_full, 1);
    tc::mbar_init_fence();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t d1 = tmem, d2 = tmem + 2 * N1;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;  // warp w reads TMEM lanes 32w..32w+31
  tc::pdl_wait();
  if (tid == 0) {
    tc::mbar_expect_tx(w_full, W1_BYTES + W2_BYTES);
    tc::bulk_load(sb + OFF_W1, wimg, W1_BYTES + W2_BYTES, w_full);
  }
  float bias2[C];
#pragma unroll
  for (int c = 0; c < C; ++c) bias2[c] = __ldg(b2 + c);
  // kTma: rows of layer 2l (a) and 2l + 1 (b) for output tile t
  auto load_in = [&](int t) {
    const int row0 = t * TILE;  // output texel row; PL % TILE == 0
    const int l = row0 / PL, q0 = row0 - l * PL;
    tc::mbar_expect_tx(in_full, 2 * ROW_TILE);
    tma_load_rows(sb + OFF_IN, &vmap, (2 * l) * PL + q0, in_full);
    tma_load_rows(sb + OFF_IN + ROW_TILE, &vmap, (2 * l + 1) * PL + q0, in_full);
  };
  if (kTma && tid == 0) load_in(blockIdx.x);
  tc::mbar_wait(w_full, 0);
  bool ovf = false;
  const int64_t total = (int64_t)L2 * PL;
  int it = 0;
  for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
    const int64_t p = (int64_t)tile * TILE + tid;  // output texel (l, q) = (p / PL, p % PL)
    const bool valid = p < total;
    float a[C], b[C];
    if (kTma) {
      tc::mbar_wait(in_full, uint32_t(it & 1));
#pragma unroll
      for (int c4 = 0; c4 < C / 4; ++c4) {
        const float4 ta = *reinterpret_cast<const float4*>(smem + OFF_IN + swz128(tid, c4));
        const float4 tb = *reinterpret_cast<const float4*>(smem + OFF_IN + ROW_TILE + swz128(tid, c4));
        a[4 * c4] = ta.x, a[4 * c4 + 1] = ta.y, a[4 * c4 + 2] = ta.z, a[4 * c4 + 3] = ta.w;
        b[4 * c4] = tb.x, b[4 * c4 + 1] = tb.y, b[4 * c4 + 2] = tb.z, b[4 * c4 + 3] = tb.w;
      }
    } else if (valid) {
      const int64_t l = p / PL, q = p - l * PL;
      load_row32(V + ((2 * l) * PL + q) * C, a);
      load_row32(V + ((2 * l + 1) * PL + q) * C, b);
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) a[c] = b[c] = 0.f;
    }
    {
      float x[K1];
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = a[c], x[C + c] = b[c];
      ovf |= stage_row64(smem + OFF_A, tid, x);
    }
    tc::fence_proxy_async();  // also orders the row-tile reads before their TMA refill
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      if (kTma && tile + int(gridDim.x) < num_tiles) load_in(tile + gridDim.x);
      mma_split64(d1, sb + OFF_A, sb + OFF_W1, N1);
      tc::commit(m1_done);
    }
    tc::mbar_wait(m1_done, uint32_t(it & 1));
    tc::fence_after();
    float h[N1];
    {
      float lo[32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        tc::tmem_ld32(lane_base + d1 + uint32_t(32 * half), h + 32 * half);
        tc::tmem_ld32(lane_base + d1 + uint32_t(N1 + 32 * half), lo);
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const float v0 = fmaf(lo[c], 1.0f / tc::kF16LoScale, h[32 * half + c]);
          const float v1 = fmaf(lo[c + 1], 1.0f / tc::kF16LoScale, h[32 * half + c + 1]);
          const float2 g = gelu2_ref(make_float2(fa(v0, __ldg(b1 + 32 * half + c)),
                                                 fa(v1, __ldg(b1 + 32 * half + c + 1))));
          h[32 * half + c] = g.x, h[32 * half + c + 1] = g.y;
        }
      }
    }
    // MMA1 has read A (m1_done): restage it with h
    ovf |= stage_row64(smem + OFF_A, tid, h);
    tc::fence_proxy_async();
    tc::fence_before();
    if (kTma && tid == 0) tc::bulk_wait_read<0>();  // the previous tile's store left the staging tile
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      mma_split64(d2, sb + OFF_A, sb + OFF_W2, N2);
      tc::commit(m2_done);
    }
    tc::mbar_wait(m2_done, uint32_t(it & 1));
    tc::fence_after();
    float y[C], lo[C];
    tc::tmem_ld32(lane_base + d2, y);
    tc::tmem_ld32(lane_base + d2 + uint32_t(N2), lo);
    if (kTma || valid) {
      float4* o = reinterpret_cast<float4*>(out + p * C);
#pragma unroll
      for (int c4 = 0; c4 < C / 4; ++c4) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = 4 * c4 + k;
          const float r = fmaf(lo[c], 1.0f / tc::kF16LoScale, y[c]);
          v[k] = fa(fm(fa(a[c], b[c]), 0.5f), fa(r, bias2[c]));
        }
        if (kTma)
          *reinterpret_cast<float4*>(smem + OFF_OUT + swz128(tid, c4)) = make_float4(v[0], v[1], v[2], v[3]);
        else
          o[c4] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    if (kTma) tc::fence_proxy_async();  // staging writes before the TMA store reads them
    // every thread has read D1 / D2 and MMA2 has read A before the next tile
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (kTma && tid == 0) {
      tma_store_rows(&omap, sb + OFF_OUT, tile * TILE);
      tc::bulk_commit();
    }
  }
  if (kTma && tid == 0) tc::bulk_wait<0>();
  if (ovf && ovf_flag) atomicOr(ovf_flag, 2);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// The image: [W1h ; W1l'] (rows n = hidden unit, K-major chunks) then
// [W2h ; W2l'], the layout stage_weights gives the attention (attn_tc.cu).
__global__ void collapse_tc_weights_kernel(const float* __restrict__ w1,
                                           const float* __restrict__ w2, uint8_t* out,
                                           int* ovf_flag) {
  pdl_grid_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  __half* bh = reinterpret_cast<__half*>(out);
  bool ovf = false;
  if (e < NJ * N1 * 8) {  // W1: w(n, k) = w1[k][n], [2C][2C]
    const int k8 = e & 7, n = (e >> 3) % N1, j = (e >> 3) / N1;
    const float x = __ldg(w1 + (8 * j + k8) * N1 + n);
    __half hi, lo;
    tc::split_f16(x, hi, lo);
    ovf = tc::split_overflows(x);
    bh[(j * 2 * N1 + n) * 8 + k8] = hi;
    bh[(j * 2 * N1 + N1 + n) * 8 + k8] = lo;
  } else if (e < NJ * N1 * 8 + NJ * N2 * 8) {  // W2: w(n, k) = w2[k][n], [2C][C]
    const int f = e - NJ * N1 * 8;
    const int k8 = f & 7, n = (f >> 3) % N2, j = (f >> 3) / N2;
    const float x = __ldg(w2 + (8 * j + k8) * N2 + n);
    __half hi, lo;
    tc::split_f16(x, hi, lo);
    ovf = tc::split_overflows(x);
    __half* b2h = bh + W1_BYTES / 2;
    b2h[(j * 2 * N2 + n) * 8 + k8] = hi;
    b2h[(j * 2 * N2 + N2 + n) * 8 + k8] = lo;
  }
  if (ovf && ovf_flag) atomicOr(ovf_flag, 2);
}

// ---- ray encodings: rays_k = resize_bilinear(base -> Hk x Wk) @ ray_proj ----
// (network.hpp:397-413). The A operand is each pixel's resized 32-channel
// base row (the resize's exact taps, its f32 lerps); one split GEMM, N = 32.
constexpr int RNJ = C / 8;                       // K = 32
constexpr int R_AHALF = RNJ * A_LBO;             // 8 KB
constexpr int R_ABYTES = 2 * R_AHALF;            // 16 KB
constexpr int R_WBYTES = RNJ * 2 * C * 16;       // 4 KB
constexpr int R_OUT_BYTES = TILE * C * 4;        // one 128B-swizzled output tile, 16 KB
constexpr int R_OFF_OUT = 0;                     // two staging tiles (1 KB aligned)
constexpr int R_OFF_A = 2 * R_OUT_BYTES;
constexpr int R_OFF_W = R_OFF_A + R_ABYTES;
constexpr int R_OFF_BAR = R_OFF_W + R_WBYTES;
constexpr int R_SMEM = R_OFF_BAR + 2 * 8 + 16;


// One 128-pixel tile per iteration: resize taps -> split A -> MMA -> the
// rows through a 128B-swizzled staging tile (two, alternating) and one TMA
// store (the per-thread 128-byte row stores were a third of the kernel).
__global__ void __launch_bounds__(TILE, 4)
    ray_project_tc_kernel(const __grid_constant__ CUtensorMap omap, const float* __restrict__ base,
                          int M, int hK, int wK, int Hk, int Wk, const uint8_t* __restrict__ wimg,
                          int num_tiles, int* ovf_flag) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + R_OFF_BAR);
  uint64_t* w_full = bars;
  uint64_t* m_done = bars + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  tc::pdl_launch_dependents();
  if (blockIdx.x >= num_tiles) return;
  const uint32_t sb = tc::smem_u32(smem);
  if (tid == 0 && (sb & 1023u)) __trap();  // swizzle atoms need 1 KB alignment
  if (tid == 0) {
    tc::mbar_init(w_full, 1);
    tc::mbar_init(m_done, 1);
    tc::mbar_init_fence();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  tc::pdl_wait();
  if (tid == 0) {
    tc::mbar_expect_tx(w_full, R_WBYTES);
    tc::bulk_load(sb + R_OFF_W, wimg, R_WBYTES, w_full);
  }
  const double sy = dd(double(hK), double(Hk)), sx = dd(double(wK), double(Wk));
  tc::mbar_wait(w_full, 0);
  bool ovf = false;
  const int n = M * Hk * Wk;
  int it = 0;
  for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
    const int i = tile * TILE + tid;
    // this thread's pixel: taps and fractions once; the loads cooperatively,
    // 8 lanes per pixel with one 16-byte channel group each (a tap's
    // 128-byte base row is one coalesced request)
    int r00 = 0, r01 = 0, r10 = 0, r11 = 0;
    float fy = 0.f, fx = 0.f;
    const bool live = i < n;
    if (live) {
      const int q = i / Wk, x = i - q * Wk;
      const int m = q / Hk, y = q - m * Hk;
      int y0, y1, x0, x1;
      resize_tap_s(y, sy, hK, y0, y1, fy);
      resize_tap_s(x, sx, wK, x0, x1, fx);
      const int mb = m * hK * wK;
      r00 = mb + y0 * wK + x0;
      r01 = mb + y0 * wK + x1;
      r10 = mb + y1 * wK + x0;
      r11 = mb + y1 * wK + x1;
    }
    const int lane = tid & 31, wbase = tid & ~31, g = lane & 7;
    const float4* b4 = reinterpret_cast<const float4*>(base);
#pragma unroll 8
    for (int k = 0; k < 8; ++k) {
      const int src = 4 * k + (lane >> 3);
      const int s00 = __shfl_sync(0xffffffffu, r00, src), s01 = __shfl_sync(0xffffffffu, r01, src);
      const int s10 = __shfl_sync(0xffffffffu, r10, src), s11 = __shfl_sync(0xffffffffu, r11, src);
      const float sfy = __shfl_sync(0xffffffffu, fy, src), sfx = __shfl_sync(0xffffffffu, fx, src);
      const float4 A = __ldg(b4 + s00 * 8 + g), B = __ldg(b4 + s01 * 8 + g);
      const float4 Cc = __ldg(b4 + s10 * 8 + g), D = __ldg(b4 + s11 * 8 + g);
      const float4 v = make_float4(lerp2(A.x, B.x, Cc.x, D.x, sfx, sfy), lerp2(A.y, B.y, Cc.y, D.y, sfx, sfy),
                                   lerp2(A.z, B.z, Cc.z, D.z, sfx, sfy), lerp2(A.w, B.w, Cc.w, D.w, sfx, sfy));
      __align__(8) __half2 h[2], l[2];
      tc::split_f16x2(v.x, v.y, h[0], l[0]);
      tc::split_f16x2(v.z, v.w, h[1], l[1]);
      ovf |= tc::split_overflows(v.x) | tc::split_overflows(v.y) | tc::split_overflows(v.z) |
             tc::split_overflows(v.w);
      const int o = R_OFF_A + (g >> 1) * A_LBO + (wbase + src) * 16 + (g & 1) * 8;
      *reinterpret_cast<uint2*>(smem + o) = *reinterpret_cast<uint2*>(h);
      *reinterpret_cast<uint2*>(smem + R_AHALF + o) = *reinterpret_cast<uint2*>(l);
    }
    tc::fence_proxy_async();
    tc::fence_before();
    if (tid == 0) tc::bulk_wait_read<1>();  // staging tile (it & 1) read out by its store
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      mma_split_k<RNJ>(tmem, sb + R_OFF_A, R_AHALF, sb + R_OFF_W, C);
      tc::commit(m_done);
    }
    tc::mbar_wait(m_done, uint32_t(it & 1));
    tc::fence_after();
    float y[C], lo[C];
    tc::tmem_ld32(lane_base + tmem, y);
    tc::tmem_ld32(lane_base + tmem + uint32_t(C), lo);
    uint8_t* ot = smem + R_OFF_OUT + (it & 1) * R_OUT_BYTES;
#pragma unroll
    for (int c4 = 0; c4 < C / 4; ++c4)
      *reinterpret_cast<float4*>(ot + swz128(tid, c4)) =
          make_float4(fmaf(lo[4 * c4], 1.0f / tc::kF16LoScale, y[4 * c4]),
                      fmaf(lo[4 * c4 + 1], 1.0f / tc::kF16LoScale, y[4 * c4 + 1]),
                      fmaf(lo[4 * c4 + 2], 1.0f / tc::kF16LoScale, y[4 * c4 + 2]),
                      fmaf(lo[4 * c4 + 3], 1.0f / tc::kF16LoScale, y[4 * c4 + 3]));
    tc::fence_proxy_async();  // generic staging writes before the TMA store reads them
    tc::fence_before();
    __syncthreads();          // also: TMEM read and A consumed before the next tile's MMA
    tc::fence_after();
    if (tid == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
              reinterpret_cast<uint64_t>(&omap)),
          "r"(sb + R_OFF_OUT + (it & 1) * R_OUT_BYTES), "r"(0), "r"(tile * TILE)
          : "memory");
      tc::bulk_commit();
    }
  }
  if (tid == 0) tc::bulk_wait<0>();
  if (ovf && ovf_flag) atomicOr(ovf_flag, 2);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

// ray_proj [32 in][32 out] -> [Wh ; Wl'] image (rows n = output channel).
__global__ void ray_tc_weights_kernel(const float* __restrict__ proj, uint8_t* out, int* ovf_flag) {
  pdl_grid_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= RNJ * C * 8) return;
  const int k8 = e & 7, n = (e >> 3) % C, j = (e >> 3) / C;
  const float x = __ldg(proj + (8 * j + k8) * C + n);
  __half hi, lo;
  tc::split_f16(x, hi, lo);
  __half* bh = reinterpret_cast<__half*>(out);
  bh[(j * 2 * C + n) * 8 + k8] = hi;
  bh[(j * 2 * C + C + n) * 8 + k8] = lo;
  if (tc::split_overflows(x) && ovf_flag) atomicOr(ovf_flag, 2);
}

}  // namespace

size_t ray_tc_weight_bytes() { return R_WBYTES; }

void ray_tc_prepare(const float* proj, void* dst, int* ovf, cudaStream_t st) {
  launch_k(ray_tc_weights_kernel, (RNJ * C * 8 + 255) / 256, 256, 0, st, proj,
           static_cast<uint8_t*>(dst), ovf);
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

bool ray_project_tc(const float* base, int M, int hK, int wK, int Hk, int Wk, const float* wimg,
                    float* out, int* ovf, cudaStream_t st) {
  const int64_t n = (int64_t)M * Hk * Wk;
  if (!wimg || (reinterpret_cast<uintptr_t>(wimg) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
      (reinterpret_cast<uintptr_t>(base) & 15) || n >= (int64_t(1) << 31) ||
      (int64_t)M * hK * wK * C >= (int64_t(1) << 31) || !encode_fn())
    return false;
  // out [n][32] fp32 as a 2-D map, 128-pixel boxes, 128B swizzle
  CUtensorMap omap;
  std::memset(&omap, 0, sizeof(omap));
  cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(n)};
  cuuint64_t strides[1] = {cuuint64_t(C) * 4};
  cuuint32_t box[2] = {cuuint32_t(C), cuuint32_t(TILE)};
  cuuint32_t estr[2] = {1, 1};
  if (encode_fn()(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const int tiles = int((n + TILE - 1) / TILE);
  smem_optin(reinterpret_cast<const void*>(ray_project_tc_kernel), R_SMEM);
  const int grid = std::min(tiles, sm_count() * 4);
  launch_pdl(false, ray_project_tc_kernel, grid, TILE, R_SMEM, st, omap, base, M, hK, wK, Hk, Wk,
             reinterpret_cast<const uint8_t*>(wimg), tiles, ovf);
  return true;
}

size_t collapse_tc_weight_bytes() { return W1_BYTES + W2_BYTES; }

void collapse_tc_prepare(const float* w1, const float* w2, void* dst, int* ovf, cudaStream_t st) {
  const int n = NJ * N1 * 8 + NJ * N2 * 8;
  launch_k(collapse_tc_weights_kernel, (n + 255) / 256, 256, 0, st, w1, w2,
           static_cast<uint8_t*>(dst), ovf);
}

bool layer_collapse_tc(const float* V, int L, int64_t PL, int C_, const float* wimg,
                       const float* b1, const float* b2, float* out, int* ovf, cudaStream_t st) {
  if (C_ != C || !wimg || (reinterpret_cast<uintptr_t>(wimg) & 15) || (L & 1) ||
      (reinterpret_cast<uintptr_t>(V) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return false;
  const int64_t total = (int64_t)(L / 2) * PL;
  const int64_t tiles = (total + TILE - 1) / TILE;
  if (tiles >= (int64_t(1) << 31) || PL >= (int64_t(1) << 31)) return false;
  const int grid = int(std::min<int64_t>(tiles, int64_t(sm_count()) * 2));
  // the TMA path: every tile inside one layer pair, rows addressable by
  // 32-bit box coordinates
  CUtensorMap vmap, omap;
  std::memset(&vmap, 0, sizeof(vmap));
  std::memset(&omap, 0, sizeof(omap));
  bool tma = PL % TILE == 0 && (int64_t)L * PL < (int64_t(1) << 31) && encode_fn() != nullptr;
  auto rows_map = [&](CUtensorMap* m, const float* ptr, int64_t rows) {
    cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(C) * 4};
    cuuint32_t box[2] = {cuuint32_t(C), cuuint32_t(TILE)};
    cuuint32_t estr[2] = {1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (tma) tma = rows_map(&vmap, V, (int64_t)L * PL) && rows_map(&omap, out, total);
  if (tma) {
    smem_optin(reinterpret_cast<const void*>(collapse_tc_kernel<true>), SMEM_BYTES);
    launch_pdl(true, collapse_tc_kernel<true>, grid, TILE, SMEM_BYTES, st, vmap, omap, V, L / 2,
               int(PL), reinterpret_cast<const uint8_t*>(wimg), b1, b2, out, int(tiles), ovf);
  } else {
    smem_optin(reinterpret_cast<const void*>(collapse_tc_kernel<false>), SMEM_BYTES);
    launch_pdl(true, collapse_tc_kernel<false>, grid, TILE, SMEM_BYTES, st, vmap, omap, V, L / 2,
               int(PL), reinterpret_cast<const uint8_t*>(wimg), b1, b2, out, int(tiles), ovf);
  }
  return true;
}

}  // namespace lvsg
