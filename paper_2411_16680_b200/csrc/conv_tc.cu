// conv3x3 (Cin = Cout = 32, channel-last) as an implicit GEMM on the sm_100a
// tensor core: tcgen05.mma kind::f16 with a 3-term fp16 split so the solve
// stays fp32-accurate (SURVEY.md §7 hard part 2):
//     x = xh + 2^-11 xl',  w = wh + 2^-11 wl'   (tc::split_f16)
//     y = b + sum_tap,ci x*w  ~=  xh*wh + 2^-11 (xh*wl' + xl'*wh)
// -- the same ~2^-22 relative error per product as 3xTF32, at half the
// shared-memory operand bytes per MAC (K = 16 per instruction), which is what
// bounds this N = 32-output-channel GEMM.
//
// Tile = 16 rows x 8 columns of output pixels (M = 128 GEMM rows, row
// m = 8g + i <-> pixel (y0+g, x0+i)), N = 32 output channels, K = 9 taps x 32
// input channels. The 18 x 10 x 32 input halo arrives as one TMA box;
// converter warps rewrite it as four 8-channel fp16 planes of hi and lo'
// ([18][10][8] halves each) -- the K-major "interleave" operand layout with
// core-matrix groups SBO = 160 B apart (one halo row), so each tap (dy, dx) is
// the same descriptor with its start address moved by (10*dy + dx) * 16
// bytes: im2col costs nothing. The optional conv-MLP rms-norm is applied in
// the converter from the 32 channels already in shared memory. Weights
// [Wh ; Wl'] (N = 64) stay resident. Per K step (16 channels of one tap):
//     MMA1  N=64: D[:, 0:64]  += Xh  * [Wh ; Wl']^T
//     MMA2  N=32: D[:, 32:64] += Xl' * Wh^T
// and the epilogue forms D[:, c] + 2^-11 D[:, 32+c].
//
// Warp roles of the persistent CTA (1 per SM): w0 TMA producer, w1 MMA issuer
// (+ TMEM owner), w2-5 converters, w6-9 epilogue; two raw TMA stages, two
// hi/lo plane buffers and two TMEM accumulators, hand-offs through mbarriers.
// Semantics of kernels_ref.hpp:72-96 (zero padding) with the bias / GELU /
// residual / rms-norm-input options of ConvArgs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "kernels.h"
#include "tc.cuh"

namespace lvsg {
namespace {

constexpr int TW = 8, TH = 16;
constexpr int HWD = TW + 2, HHT = TH + 2;       // 10 x 18 halo
constexpr int HALO_PX = HWD * HHT;              // 180
constexpr int NCH = 4;                          // 8-channel fp16 planes (Cin = 32)
constexpr int RAW_BYTES = HALO_PX * 32 * 4;     // one TMA box [18][10][32] (23040)
constexpr int LBO_A = HALO_PX * 16 + 16;        // plane stride (padded: conflict-free stores)
constexpr int HALF_BYTES = NCH * LBO_A;         // hi (or lo) planes of one buffer
constexpr int PLANES_BYTES = 2 * HALF_BYTES;
constexpr int W_ROWS = 64;                      // 32 hi + 32 lo
constexpr int W_BYTES = 9 * NCH * W_ROWS * 16;  // 36864
constexpr int OFF_RAW = W_BYTES;                // 2 raw TMA stages
constexpr int OFF_PLANES = OFF_RAW + 2 * RAW_BYTES;
constexpr int OFF_RMS = OFF_PLANES + 2 * PLANES_BYTES;
constexpr int OFF_BAR = OFF_RMS + 192 * 4;
constexpr int NBAR = 12;
constexpr int SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
constexpr int NT = 320;  // 10 warps
constexpr uint32_t TMEM_COLS = 128;
constexpr int NCONV = 128, NEPI = 128;

struct TileCoord {
  int b, y0, x0;
};

__device__ __forceinline__ TileCoord tile_coord(int t, int H, int W) {
  const int tx_n = (W + TW - 1) / TW, ty_n = (H + TH - 1) / TH;
  const int per = tx_n * ty_n;
  TileCoord c;
  c.b = t / per;
  const int r = t - c.b * per;
  c.y0 = (r / tx_n) * TH;
  c.x0 = (r % tx_n) * TW;
  return c;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c, int x,
                                            int y, int b, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(x), "r"(y), "r"(b), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void issue_tile(uint64_t ah0, uint64_t al0, uint64_t b0,
                                           uint32_t tmem_acc) {
  constexpr uint32_t id64 = tc::idesc_f16(128, 64);
  constexpr uint32_t id32 = tc::idesc_f16(128, 32);
#pragma unroll
  for (int tap = 0; tap < 9; ++tap) {
    const int dy = tap / 3, dx = tap % 3;
#pragma unroll
    for (int s = 0; s < NCH / 2; ++s) {
      const uint64_t aoff = uint64_t((2 * s * LBO_A + (dy * HWD + dx) * 16) >> 4);
      const uint64_t boff = uint64_t(((tap * NCH + 2 * s) * W_ROWS * 16) >> 4);
      tc::mma_f16(tmem_acc, ah0 + aoff, b0 + boff, id64, (tap | s) != 0);
      tc::mma_f16(tmem_acc + 32, al0 + aoff, b0 + boff, id32, 1u);
    }
  }
}

__global__ void __launch_bounds__(NT, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap xmap, const ConvArgs a, int num_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __half* w_s = reinterpret_cast<__half*>(smem);
  float* rms_s = reinterpret_cast<float*>(smem + OFF_RMS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* raw_full = bars;          // [2] TMA bytes landed
  uint64_t* raw_empty = bars + 2;      // [2] converters done reading raw
  uint64_t* conv_full = bars + 4;      // [2] hi/lo planes ready
  uint64_t* planes_empty = bars + 6;   // [2] MMAs done reading the planes
  uint64_t* mma_done = bars + 8;       // [2] accumulator ready
  uint64_t* acc_empty = bars + 10;     // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  if (blockIdx.x >= num_tiles) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // weights: [tap][plane j][row n][8 halves], rows 0..31 = fp16 hi, 32..63 = lo'
  for (int e = tid; e < 9 * NCH * W_ROWS * 8; e += NT) {
    const int k8 = e & 7, n = (e >> 3) & 63, rest = e >> 9;
    const int j = rest % NCH, tap = rest / NCH;
    const int co = n & 31, ci = 8 * j + k8;
    __half h, l;
    tc::split_f16(__ldg(a.w + (co * w_cin_of(a) + a.w_ci0 + ci) * 9 + tap), h, l);
    w_s[e] = n < 32 ? h : l;
  }
  tc::fence_proxy_async();
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&raw_full[b], 1);
      tc::mbar_init(&raw_empty[b], NCONV);
      tc::mbar_init(&conv_full[b], NCONV);
      tc::mbar_init(&planes_empty[b], 1);
      tc::mbar_init(&mma_done[b], 1);
      tc::mbar_init(&acc_empty[b], NEPI);
    }
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);

  if (warp == 0) {
    // ---- TMA producer: one [18][10][32] box per tile into the raw ring ----
    if (lane == 0) {
      int i = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
        const int r = i & 1;
        if (i >= 2) tc::mbar_wait(&raw_empty[r], uint32_t(((i >> 1) - 1) & 1));
        const TileCoord tc_ = tile_coord(t, a.H, a.W);
        mbar_expect_tx(&raw_full[r], RAW_BYTES);
        tma_load_4d(sbase + OFF_RAW + r * RAW_BYTES, &xmap, 0, tc_.x0 - 1, tc_.y0 - 1, tc_.b,
                    &raw_full[r]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (lane == 0) {
      const uint64_t b0 = tc::smem_desc(sbase, W_ROWS * 16, 128);
      int i = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
        const int b = i & 1;
        tc::mbar_wait(&conv_full[b], uint32_t((i >> 1) & 1));
        if (i >= 2) tc::mbar_wait(&acc_empty[b], uint32_t(((i >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t hi = sbase + OFF_PLANES + b * PLANES_BYTES;
        issue_tile(tc::smem_desc(hi, LBO_A, HWD * 16),
                   tc::smem_desc(hi + HALF_BYTES, LBO_A, HWD * 16), b0, tmem + uint32_t(b * 64));
        tc::commit(&planes_empty[b]);
        tc::commit(&mma_done[b]);
      }
    }
  } else if (warp < 6) {
    // ---- converters: raw pixel-major box -> fp16 hi / lo' K-major planes ----
    const int ct = tid - 64;
    int i = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      const float* raw = reinterpret_cast<const float*>(smem + OFF_RAW + b * RAW_BYTES);
      float* hi = reinterpret_cast<float*>(smem + OFF_PLANES + b * PLANES_BYTES);
      float* lo = reinterpret_cast<float*>(smem + OFF_PLANES + b * PLANES_BYTES + HALF_BYTES);
      tc::mbar_wait(&raw_full[b], uint32_t((i >> 1) & 1));
      if (a.rinv) {
        // conv_mlp_residual's rms_norm over the pixel's 32 channels
        named_sync(1, NCONV);  // previous tile's scale reads are done
        for (int px = ct; px < HALO_PX; px += NCONV) {
          float ms = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // all 32 channels
            const float4 v = *reinterpret_cast<const float4*>(raw + px * 32 + 4 * j);
            ms = fmaf(v.x, v.x, ms);
            ms = fmaf(v.y, v.y, ms);
            ms = fmaf(v.z, v.z, ms);
            ms = fmaf(v.w, v.w, ms);
          }
          rms_s[px] = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(ms, 32.0f), 1e-6f)));
        }
        named_sync(1, NCONV);
      }
      if (i >= 2) tc::mbar_wait(&planes_empty[b], uint32_t(((i >> 1) - 1) & 1));
      for (int e = ct; e < HALO_PX * NCH; e += NCONV) {
        const int px = e >> 2, j = e & 3;
        float v[8];
        {
          const float4 v0 = *reinterpret_cast<const float4*>(raw + px * 32 + 8 * j);
          const float4 v1 = *reinterpret_cast<const float4*>(raw + px * 32 + 8 * j + 4);
          v[0] = v0.x, v[1] = v0.y, v[2] = v0.z, v[3] = v0.w;
          v[4] = v1.x, v[5] = v1.y, v[6] = v1.z, v[7] = v1.w;
        }
        if (a.rinv) {
          const float r = rms_s[px];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fm(fm(v[k], r), __ldg(a.gain + 8 * j + k));
        }
        __align__(16) __half h[8], l[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) tc::split_f16(v[k], h[k], l[k]);
        const int off = j * LBO_A + px * 16;  // bytes
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(hi) + off) = *reinterpret_cast<uint4*>(h);
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(lo) + off) = *reinterpret_cast<uint4*>(l);
      }
      tc::mbar_arrive(&raw_empty[b]);
      tc::fence_proxy_async();
      tc::mbar_arrive(&conv_full[b]);
    }
  } else {
    // ---- epilogue: TMEM -> bias / GELU / residual -> global ----
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;
    int i = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      tc::mbar_wait(&mma_done[b], uint32_t((i >> 1) & 1));
      tc::fence_after();
      const uint32_t taddr = tmem + uint32_t(b * 64) + (uint32_t(q * 32) << 16);
      float d0[32], d1[32];
      tc::tmem_ld32(taddr, d0);
      tc::tmem_ld32(taddr + 32, d1);
      tc::fence_before();
      tc::mbar_arrive(&acc_empty[b]);
      const TileCoord tt = tile_coord(t, a.H, a.W);
      const int y = tt.y0 + (row >> 3), x = tt.x0 + (row & 7);
      if (y >= a.H || x >= a.W) continue;
      const long long pix = (long long)y * a.W + x;
      float* o = a.out + (long long)tt.b * a.out_bstride + pix * a.out_pstride;
      const float* rs =
          a.resid ? a.resid + (long long)tt.b * a.res_bstride + pix * a.res_pstride : nullptr;
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = 4 * c4 + k;
          float y_ = fmaf(d1[c], 1.0f / tc::kF16LoScale, d0[c]);
          if (a.bias) y_ = fa(y_, __ldg(a.bias + c));
          if (a.gelu) y_ = gelu_ref(y_);
          v[k] = y_;
        }
        if (rs) {
          const float4 r = *reinterpret_cast<const float4*>(rs + 4 * c4);
          v[0] = fa(r.x, v[0]);
          v[1] = fa(r.y, v[1]);
          v[2] = fa(r.z, v[2]);
          v[3] = fa(r.w, v[3]);
        }
        *reinterpret_cast<float4*>(o + 4 * c4) = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
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

}  // namespace

bool conv3x3_tc_supported(const ConvArgs& a) {
  if (a.Cin != 32 || a.Cout != 32 || a.nsrc != 1 || a.src[0].C != 32) return false;
  if (a.src[0].pstride % 4 || a.out_pstride % 4 || (a.resid && a.res_pstride % 4)) return false;
  if (a.src[0].bstride % 4) return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return encode_fn() && al(a.src[0].ptr) && al(a.out) && (!a.resid || al(a.resid)) &&
         (!a.gain || al(a.gain));
}

void conv3x3_tc(const ConvArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3x3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  // input [B, H, W, 32] (pixel stride pstride, batch stride bstride floats)
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const ConvSrc& S = a.src[0];
  cuuint64_t dims[4] = {32, cuuint64_t(a.W), cuuint64_t(a.H), cuuint64_t(a.B)};
  cuuint64_t strides[3] = {cuuint64_t(S.pstride) * 4, cuuint64_t(S.pstride) * 4 * a.W,
                           cuuint64_t(S.bstride) * 4};
  cuuint32_t box[4] = {32, HWD, HHT, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(S.ptr), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int tiles = a.B * ((a.H + TH - 1) / TH) * ((a.W + TW - 1) / TW);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = tiles < sms ? tiles : sms;
  conv3x3_tc_kernel<<<grid, NT, SMEM_BYTES, st>>>(map, a, tiles);
}

}  // namespace lvsg
