// conv3x3 (Cin = Cout = 32, channel-last) as an implicit GEMM on the sm_100a
// tensor core: tcgen05.mma kind::tf32 with a 3xTF32 split so the solve stays
// fp32-accurate (SURVEY.md §7 hard part 2):
//     y = b + sum_tap,ci x*w  ~=  xh*wh + (xh*wl + xl*wh)
//
// Tile = 16 rows x 8 columns of output pixels (M = 128 GEMM rows, row
// m = 8g + i <-> pixel (y0+g, x0+i)), N = 32 output channels, K = 9 taps x 32
// input channels. The input halo (18 x 10 pixels x 32 channels) is staged
// once per tile as hi and lo tf32 planes in the K-major "interleave" layout
// (16-byte rows, core-matrix groups SBO = 160 B apart = one halo row); every
// tap (dy, dx) is then just the descriptor start address shifted by
// (10*dy + dx) * 16 bytes -- im2col costs nothing. Weights (hi rows 0..31, lo
// rows 32..63) stay resident in shared memory for the whole persistent CTA.
// Per K step (8 channels of one tap):
//     MMA1  N=64: D[:, 0:64]  += Xh * [Wh ; Wl]^T
//     MMA2  N=32: D[:, 32:64] += Xl * Wh^T
// and the epilogue sums D[:, c] + D[:, 32+c]. Two TMEM accumulators and two
// halo buffers pipeline tile t+1's staging and MMAs against tile t's
// epilogue. Semantics of kernels_ref.hpp:72-96 (zero padding), fused with the
// bias / GELU / residual / rms-norm-input options of ConvArgs.
#include "kernels.h"
#include "tc.cuh"

namespace lvsg {
namespace {

constexpr int TW = 8, TH = 16;
constexpr int HWD = TW + 2, HHT = TH + 2;       // 10 x 18 halo
constexpr int HALO_PX = HWD * HHT;              // 180
constexpr int NCH = 8;                          // 4-channel chunks of Cin = 32
constexpr int LBO_A = HALO_PX * 16 + 16;        // chunk stride (padded: bank-conflict free)
constexpr int HALO_BYTES = NCH * LBO_A;         // one plane (hi or lo)
constexpr int W_ROWS = 64;                      // 32 hi + 32 lo
constexpr int W_BYTES = 9 * NCH * W_ROWS * 16;  // 73728
constexpr int SMEM_BYTES = W_BYTES + 4 * HALO_BYTES + 64;
constexpr int NWORK = 256;        // staging / epilogue threads (8 warps)
constexpr int NT = NWORK + 32;     // + one MMA-issuer warp
constexpr uint32_t TMEM_COLS = 128;  // two 64-column accumulators

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

__device__ __forceinline__ void stage_halo(const ConvArgs& a, const TileCoord& tc_, float* hi,
                                           float* lo) {
  const ConvSrc& S = a.src[0];
  const float* src = S.ptr + (long long)tc_.b * S.bstride;
  const long long HW = (long long)a.H * a.W;
  // all global loads of this thread first (memory-level parallelism), then
  // the tf32 split and the shared-memory stores
  constexpr int PER = (HALO_PX * NCH + NWORK - 1) / NWORK;
  float4 vals[PER];
  float rs[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x + k * NWORK;
    vals[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    rs[k] = 1.f;
    if (e < HALO_PX * NCH) {
      const int px = e >> 3, j = e & 7;
      const int hy = px / HWD, hx = px - hy * HWD;
      const int gy = tc_.y0 - 1 + hy, gx = tc_.x0 - 1 + hx;
      if (gy >= 0 && gy < a.H && gx >= 0 && gx < a.W) {
        const long long p = (long long)gy * a.W + gx;
        vals[k] = __ldg(reinterpret_cast<const float4*>(src + p * S.pstride) + j);
        if (a.rinv) rs[k] = __ldg(a.rinv + tc_.b * HW + p);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x + k * NWORK;
    if (e >= HALO_PX * NCH) break;
    const int px = e >> 3, j = e & 7;
    float4 v = vals[k];
    if (a.rinv) {
      const float r = rs[k];
      const float4 g = __ldg(reinterpret_cast<const float4*>(a.gain) + j);
      v.x = fm(fm(v.x, r), g.x);
      v.y = fm(fm(v.y, r), g.y);
      v.z = fm(fm(v.z, r), g.z);
      v.w = fm(fm(v.w, r), g.w);
    }
    float4 h, l;
    tc::split_tf32(v.x, h.x, l.x);
    tc::split_tf32(v.y, h.y, l.y);
    tc::split_tf32(v.z, h.z, l.z);
    tc::split_tf32(v.w, h.w, l.w);
    const int off = (j * LBO_A) / 4 + px * 4;
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

// MMA issue for one tile: 9 taps x 4 K-steps x {N=64 hi, N=32 lo}. Every
// descriptor is a base descriptor plus a compile-time start-address offset.
__device__ __forceinline__ void issue_tile(uint64_t ah0, uint64_t al0, uint64_t b0,
                                           uint32_t tmem_acc) {
  constexpr uint32_t id64 = tc::idesc_tf32(128, 64);
  constexpr uint32_t id32 = tc::idesc_tf32(128, 32);
#pragma unroll
  for (int tap = 0; tap < 9; ++tap) {
    const int dy = tap / 3, dx = tap % 3;
#pragma unroll
    for (int s = 0; s < NCH / 2; ++s) {
      const uint64_t aoff = uint64_t((2 * s * LBO_A + (dy * HWD + dx) * 16) >> 4);
      const uint64_t boff = uint64_t(((tap * NCH + 2 * s) * W_ROWS * 16) >> 4);
      tc::mma_tf32(tmem_acc, ah0 + aoff, b0 + boff, id64, (tap | s) != 0);
      tc::mma_tf32(tmem_acc + 32, al0 + aoff, b0 + boff, id32, 1u);
    }
  }
}

// Worker warp w: TMEM lanes 32*(w%4).. (tile rows), accumulator columns
// 16*(w/4).. of both halves.
__device__ __forceinline__ void epilogue(const ConvArgs& a, const TileCoord& t, uint32_t tmem_acc,
                                         int warp, int lane) {
  const int q = warp & 3, h = warp >> 2;
  const int row = q * 32 + lane;
  const int y = t.y0 + (row >> 3), x = t.x0 + (row & 7);
  const uint32_t taddr = tmem_acc + (uint32_t(q * 32) << 16) + uint32_t(h * 16);
  float d0[16], d1[16];
  tc::tmem_ld16(taddr, d0);
  tc::tmem_ld16(taddr + 32, d1);
  if (y >= a.H || x >= a.W) return;
  const long long pix = (long long)y * a.W + x;
  float* o = a.out + (long long)t.b * a.out_bstride + pix * a.out_pstride + h * 16;
  const float* rs =
      a.resid ? a.resid + (long long)t.b * a.res_bstride + pix * a.res_pstride + h * 16 : nullptr;
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * c4 + k;
      float y_ = fa(d0[c], d1[c]);
      if (a.bias) y_ = fa(y_, __ldg(a.bias + h * 16 + c));
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

// Warp-specialised persistent CTA: warps 0..7 stage halos and run
// epilogues, warp 8 issues the MMAs. mbarriers: halo_full[b] (256 worker
// arrivals), mma_done[b] (tcgen05.commit), acc_empty[b] (256 arrivals).
__global__ void __launch_bounds__(NT, 1) conv3x3_tc_kernel(const ConvArgs a, int num_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* w_s = reinterpret_cast<float*>(smem);
  float* halo[2][2];
  halo[0][0] = reinterpret_cast<float*>(smem + W_BYTES);
  halo[0][1] = reinterpret_cast<float*>(smem + W_BYTES + HALO_BYTES);
  halo[1][0] = reinterpret_cast<float*>(smem + W_BYTES + 2 * HALO_BYTES);
  halo[1][1] = reinterpret_cast<float*>(smem + W_BYTES + 3 * HALO_BYTES);
  uint64_t* halo_full = reinterpret_cast<uint64_t*>(smem + W_BYTES + 4 * HALO_BYTES);
  uint64_t* mma_done = halo_full + 2;
  uint64_t* acc_empty = halo_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(halo_full + 6);

  if (blockIdx.x >= num_tiles) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // weights: [tap][chunk j][row n][4], rows 0..31 = tf32 hi, 32..63 = lo
  for (int e = tid; e < 9 * NCH * W_ROWS * 4; e += NT) {
    const int c4 = e & 3, n = (e >> 2) & 63, rest = e >> 8;
    const int j = rest % NCH, tap = rest / NCH;
    const int co = n & 31, ci = 4 * j + c4;
    float h, l;
    tc::split_tf32(__ldg(a.w + (co * 32 + ci) * 9 + tap), h, l);
    w_s[e] = n < 32 ? h : l;
  }
  tc::fence_proxy_async();
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&halo_full[b], NWORK);
      tc::mbar_init(&mma_done[b], 1);
      tc::mbar_init(&acc_empty[b], NWORK);
    }
    tc::mbar_init_fence();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == NWORK / 32) {
    // ---- MMA issuer (one thread) ----
    if (lane == 0) {
      const uint64_t b0 = tc::smem_desc(tc::smem_u32(w_s), W_ROWS * 16, 128);
      const uint64_t ah0 = tc::smem_desc(tc::smem_u32(halo[0][0]), LBO_A, HWD * 16);
      const uint64_t al0 = tc::smem_desc(tc::smem_u32(halo[0][1]), LBO_A, HWD * 16);
      const uint64_t ah1 = tc::smem_desc(tc::smem_u32(halo[1][0]), LBO_A, HWD * 16);
      const uint64_t al1 = tc::smem_desc(tc::smem_u32(halo[1][1]), LBO_A, HWD * 16);
      int i = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
        const int b = i & 1;
        tc::mbar_wait(&halo_full[b], uint32_t((i >> 1) & 1));
        if (i >= 2) tc::mbar_wait(&acc_empty[b], uint32_t(((i - 2) >> 1) & 1));
        tc::fence_after();
        issue_tile(b ? ah1 : ah0, b ? al1 : al0, b0, tmem + uint32_t(b * 64));
        tc::commit(&mma_done[b]);
      }
    }
  } else {
    // ---- workers: stage tile i, then drain tile i-1 ----
    int i = 0;
    int tprev = -1;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      stage_halo(a, tile_coord(t, a.H, a.W), halo[b][0], halo[b][1]);
      tc::fence_proxy_async();
      tc::mbar_arrive(&halo_full[b]);
      if (tprev >= 0) {
        const int pb = (i - 1) & 1;
        tc::mbar_wait(&mma_done[pb], uint32_t(((i - 1) >> 1) & 1));
        tc::fence_after();
        epilogue(a, tile_coord(tprev, a.H, a.W), tmem + uint32_t(pb * 64), warp, lane);
        tc::fence_before();
        tc::mbar_arrive(&acc_empty[pb]);
      }
      tprev = t;
    }
    if (tprev >= 0) {
      const int pb = (i - 1) & 1;
      tc::mbar_wait(&mma_done[pb], uint32_t(((i - 1) >> 1) & 1));
      tc::fence_after();
      epilogue(a, tile_coord(tprev, a.H, a.W), tmem + uint32_t(pb * 64), warp, lane);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace

bool conv3x3_tc_supported(const ConvArgs& a) {
  if (a.Cin != 32 || a.Cout != 32 || a.nsrc != 1 || a.src[0].C != 32) return false;
  if (a.src[0].pstride % 4 || a.out_pstride % 4 || (a.resid && a.res_pstride % 4)) return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return al(a.src[0].ptr) && al(a.out) && (!a.resid || al(a.resid)) && (!a.gain || al(a.gain));
}

void conv3x3_tc(const ConvArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3x3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  const int tiles = a.B * ((a.H + TH - 1) / TH) * ((a.W + TW - 1) / TW);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = tiles < sms ? tiles : sms;
  conv3x3_tc_kernel<<<grid, NT, SMEM_BYTES, st>>>(a, tiles);
}

}  // namespace lvsg
