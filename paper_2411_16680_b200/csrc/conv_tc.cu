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
// (+ TMEM owner), w2-5 converters, w6-13 epilogue (two warpgroups taking
// alternate tiles); NR raw TMA stages, NP hi/lo plane buffers and NA TMEM
// accumulators, hand-offs through mbarriers. Each epilogue warp owns one
// 4-row x 8-column sub-box of the tile: its residual arrives by TMA one tile
// ahead, and its output is staged in 128B-swizzled shared memory and leaves as
// one TMA tile store (full-line writes; image edges clipped by the TMA unit).
// Semantics of kernels_ref.hpp:72-96 (zero padding) with the bias / GELU /
// residual / rms-norm-input options of ConvArgs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "host.h"
#include "kernels.h"
#include "tc.cuh"

// Development probe bitmask (0 in every shipped build): skip the MMAs (1), the
// epilogue's TMEM reads / math / stores (2), the converters' work (4), the
// TMA loads (8); timing-only: 128B-aligned A plane starts (16), SBO = 128 (32).
#ifndef LVSG_CONV_PROBE
#define LVSG_CONV_PROBE 0
#endif

#ifndef LVSG_GELU2
#define LVSG_GELU2 1
#endif
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
constexpr int NR = 3;   // raw TMA stages
constexpr int NP = 2;   // converted hi/lo plane buffers
constexpr int NA = 4;   // TMEM accumulators (64 columns each)
constexpr int EPW = 2;  // epilogue warpgroups
constexpr int NEW = 4 * EPW;                    // epilogue warps
constexpr int SUB_ROWS = 4;                     // image rows per epilogue sub-box
constexpr int SUB_BYTES = SUB_ROWS * TW * 128;  // [4][8][32] fp32 = 4096
constexpr int OFF_OUT = 0;                      // 1024-aligned (128B swizzle)
constexpr int OFF_RES = OFF_OUT + NEW * SUB_BYTES;
constexpr int OFF_W = OFF_RES + NEW * SUB_BYTES;
constexpr int OFF_RAW = OFF_W + W_BYTES;
constexpr int OFF_PLANES = OFF_RAW + NR * RAW_BYTES;
constexpr int OFF_SMALL = OFF_PLANES + NP * PLANES_BYTES;  // rms[192], bias[32], gain[32], walpha[288]
constexpr int OFF_BAR = OFF_SMALL + (256 + 288) * 4;
constexpr int NAL = 8;  // kAlpha: ring of per-tile alpha halos [180] (in the unused residual area)
constexpr int NBAR = 2 * NR + 2 * NP + 2 * NA + NEW + 1 + NAL;
static_assert(NAL * HALO_PX * 4 <= NEW * SUB_BYTES, "alpha halos fit the residual staging");
constexpr int SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
constexpr int NT = 64 + 128 + 128 * EPW;
constexpr uint32_t TMEM_COLS = 64 * NA;
constexpr int NCONV = 128, NEPI = 128;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
static_assert((OFF_RES | OFF_W) % 1024 == 0, "swizzled staging alignment");

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

__device__ __forceinline__ void issue_tile(uint64_t ah0, uint64_t al0, uint64_t b0,
                                           uint32_t tmem_acc) {
  constexpr uint32_t id64 = tc::idesc_f16(128, 64);
  constexpr uint32_t id32 = tc::idesc_f16(128, 32);
#pragma unroll
  for (int tap = 0; tap < 9; ++tap) {
    const int dy = tap / 3, dx = tap % 3;
#pragma unroll
    for (int s = 0; s < NCH / 2; ++s) {
      const uint64_t aoff = (LVSG_CONV_PROBE & 16) ? uint64_t(s * 2048 >> 4)
                                                   : uint64_t((2 * s * LBO_A + (dy * HWD + dx) * 16) >> 4);
      const uint64_t boff = uint64_t(((tap * NCH + 2 * s) * W_ROWS * 16) >> 4);
      tc::mma_f16(tmem_acc, ah0 + aoff, b0 + boff, id64, (tap | s) != 0);
      tc::mma_f16(tmem_acc + 32, al0 + aoff, b0 + boff, id32, 1u);
    }
  }
}

// 16-byte chunk c4 of row r in a 128B-swizzled [rows][128 B] staging buffer.
__device__ __forceinline__ uint32_t swz(int r, int c4) {
  return uint32_t(r * 128 + ((c4 ^ (r & 7)) << 4));
}

// kPool: 0 none, 1 the fused mean pool, 2 the pool also stored into peer
// GPUs' pyramids (the fused exchange; its own instantiation so the common
// pool path carries no peer code)
#ifdef LVSG_TIMELINE
constexpr int kTlSlots = 1024;
__device__ unsigned long long g_conv_tl[kTlSlots][4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CONV_TL(k, op)                                                          \
  if (a.tl_slot > 0 && a.tl_slot <= kTlSlots && threadIdx.x == 0)               \
    op(&g_conv_tl[a.tl_slot - 1][k], gtime());
#else
#define CONV_TL(k, op)
#endif

template <bool kAlpha, int kPool>
__global__ void __launch_bounds__(NT, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap xmap,
                      const __grid_constant__ CUtensorMap omap,
                      const __grid_constant__ CUtensorMap rmap, const ConvArgs a, int num_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* rms_s = reinterpret_cast<float*>(smem + OFF_SMALL);
  float* bias_s = rms_s + 192;
  float* gain_s = bias_s + 32;
  float* walpha_s = gain_s + 32;  // [tap][co] weights of the folded alpha channel
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* raw_full = bars;                 // [NR] TMA bytes landed
  uint64_t* raw_empty = raw_full + NR;       // [NR] converters done reading raw
  uint64_t* conv_full = raw_empty + NR;      // [NP] hi/lo planes ready
  uint64_t* planes_empty = conv_full + NP;   // [NP] MMAs done reading the planes
  uint64_t* mma_done = planes_empty + NP;    // [NA] accumulator ready
  uint64_t* acc_empty = mma_done + NA;       // [NA] accumulator drained
  uint64_t* res_full = acc_empty + NA;       // [NEW] residual sub-box landed
  uint64_t* w_full = res_full + NEW;         // weight image landed
  uint64_t* alpha_full = w_full + 1;         // [NAL] kAlpha: a tile's alpha halo in smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  tc::pdl_launch_dependents();
  if (blockIdx.x >= num_tiles) return;
  CONV_TL(0, atomicMin)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = tc::smem_u32(smem);
  if (tid == 0 && (sbase & 1023u)) __trap();  // swizzle atoms need 1 KB alignment

  if (tid < 32) bias_s[tid] = a.bias ? __ldg(a.bias + tid) : 0.f;
  else if (tid < 64) gain_s[tid - 32] = a.gain ? __ldg(a.gain + tid - 32) : 1.f;
  if constexpr (kAlpha)
    for (int e = tid; e < 288; e += NT) {
      const int co = e & 31, tap = e >> 5;
      walpha_s[e] = __ldg(a.w + ((long long)co * w_cin_of(a) + a.alpha_ci) * 9 + tap);
    }
  tc::fence_proxy_async();
  if (tid == 0) {
    for (int k = 0; k < NR; ++k) {
      tc::mbar_init(&raw_full[k], 1);
      tc::mbar_init(&raw_empty[k], NCONV);
    }
    for (int k = 0; k < NP; ++k) {
      tc::mbar_init(&conv_full[k], NCONV);
      tc::mbar_init(&planes_empty[k], 1);
    }
    for (int k = 0; k < NA; ++k) {
      tc::mbar_init(&mma_done[k], 1);
      tc::mbar_init(&acc_empty[k], NEPI);
    }
    for (int k = 0; k < NEW; ++k) tc::mbar_init(&res_full[k], 1);
    tc::mbar_init(w_full, 1);
    for (int k = 0; k < NAL; ++k) tc::mbar_init(&alpha_full[k], NCONV);
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  // a settled weight image (made and synchronised by an earlier call) loads
  // under the previous kernel's tail; a freshly prepared one after the wait
  if (a.w_early && tid == 0) {
    tc::mbar_expect_tx(w_full, W_BYTES);
    tc::bulk_load(sbase + OFF_W, a.wsplit, W_BYTES, w_full);
  }
  // everything above overlaps the previous kernel under PDL; global data
  // (inputs, residual, outputs, a freshly prepared weight image) only below
  tc::pdl_wait();
  CONV_TL(1, atomicMin)
  if (!a.w_early && tid == 0) {
    tc::mbar_expect_tx(w_full, W_BYTES);
    tc::bulk_load(sbase + OFF_W, a.wsplit, W_BYTES, w_full);
  }

  if (warp == 0) {
    // ---- TMA producer: one [18][10][32] box per tile into the raw ring ----
    if (lane == 0) {
      int i = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
        const int r = i % NR;
        if (i >= NR) tc::mbar_wait(&raw_empty[r], uint32_t((i / NR - 1) & 1));
        if ((LVSG_CONV_PROBE & 8)) {
          tc::mbar_arrive(&raw_full[r]);
          continue;
        }
        const TileCoord tc_ = tile_coord(t, a.H, a.W);
        tc::mbar_expect_tx(&raw_full[r], RAW_BYTES);
        tc::tma_load_4d(sbase + OFF_RAW + r * RAW_BYTES, &xmap, 0, tc_.x0 - 1, tc_.y0 - 1, tc_.b,
                        &raw_full[r]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: the whole warp walks the ring, one elected lane issues ----
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // provably warp-uniform
    const uint64_t b0 = tc::smem_desc(sbase + OFF_W, W_ROWS * 16, 128);
    tc::mbar_wait(w_full, 0);
    int i = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
      const int b = i % NP, ac = i % NA;
      tc::mbar_wait(&conv_full[b], uint32_t((i / NP) & 1));
      if (i >= NA) tc::mbar_wait(&acc_empty[ac], uint32_t((i / NA - 1) & 1));
      tc::fence_after();
      const uint32_t hi = sbase + OFF_PLANES + b * PLANES_BYTES;
      constexpr uint32_t sbo = (LVSG_CONV_PROBE & 32) ? 128 : HWD * 16;
      constexpr uint32_t lbo = (LVSG_CONV_PROBE & 16) ? 2944 : LBO_A;
      if (tc::elect_one()) {
        if (!(LVSG_CONV_PROBE & 1))
          issue_tile(tc::smem_desc(hi, lbo, sbo), tc::smem_desc(hi + HALF_BYTES, lbo, sbo), b0,
                     tm + uint32_t(ac * 64));
        tc::commit(&planes_empty[b]);
        tc::commit(&mma_done[ac]);
      }
      __syncwarp();
    }
  } else if (warp < 6) {
    // ---- converters: raw pixel-major box -> fp16 hi / lo' K-major planes ----
    const int ct = tid - 64;
    const int j = ct & 3;  // this thread's 8-channel plane (NCONV % 4 == 0)
    float g8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) g8[k] = gain_s[8 * j + k];
    int i = 0;
    bool ovf = false;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++i) {
      const int r = i % NR, b = i % NP;
      const float* raw = reinterpret_cast<const float*>(smem + OFF_RAW + r * RAW_BYTES);
      uint8_t* hi = smem + OFF_PLANES + b * PLANES_BYTES;
      uint8_t* lo = hi + HALF_BYTES;
      // kAlpha: this tile's halo of the folded alpha channel, loaded before the
      // conversion (its latency overlaps it) and kept in smem for the epilogue
      float alv[2] = {0.f, 0.f};
      if constexpr (kAlpha) {
        const TileCoord c = tile_coord(t, a.H, a.W);
        const float* ab = a.alpha + (long long)c.b * a.alpha_bstride;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int e = ct + q * NCONV;
          const int yy = c.y0 - 1 + e / HWD, xx = c.x0 - 1 + e % HWD;
          if (e < HALO_PX && yy >= 0 && yy < a.H && xx >= 0 && xx < a.W)
            alv[q] = __ldg(ab + ((long long)yy * a.W + xx) * a.alpha_pstride);
        }
      }
      tc::mbar_wait(&raw_full[r], uint32_t((i / NR) & 1));
      if (i >= NP) tc::mbar_wait(&planes_empty[b], uint32_t((i / NP - 1) & 1));
      for (int e = ct; e < ((LVSG_CONV_PROBE & 4) ? 0 : HALO_PX * NCH); e += NCONV) {
        const int px = e >> 2;
        float v[8];
        {
          const float4 v0 = *reinterpret_cast<const float4*>(raw + px * 32 + 8 * j);
          const float4 v1 = *reinterpret_cast<const float4*>(raw + px * 32 + 8 * j + 4);
          v[0] = v0.x, v[1] = v0.y, v[2] = v0.z, v[3] = v0.w;
          v[4] = v1.x, v[5] = v1.y, v[6] = v1.z, v[7] = v1.w;
        }
        if (a.rinv) {
          // conv_mlp_residual's rms_norm over the pixel's 32 channels: the
          // pixel's 4 plane threads are adjacent lanes (quad reduction)
          float ms = 0.f;
#pragma unroll
          for (int k = 0; k < 8; ++k) ms = fmaf(v[k], v[k], ms);
          const unsigned qm = __activemask();  // the loop tail cuts at a quad boundary
          ms += __shfl_xor_sync(qm, ms, 1);
          ms += __shfl_xor_sync(qm, ms, 2);
          const float rr = __fdiv_rn(1.0f, __fsqrt_rn(fa(fm(ms, 0.03125f), 1e-6f)));  // ms / 32, exactly
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fm(fm(v[k], rr), g8[k]);
        }
        __align__(16) __half2 h[4], l[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::split_f16x2(v[2 * k], v[2 * k + 1], h[k], l[k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) ovf |= tc::split_overflows(v[k]);
        const int off = j * LBO_A + px * 16;  // bytes
        *reinterpret_cast<uint4*>(hi + off) = *reinterpret_cast<uint4*>(h);
        *reinterpret_cast<uint4*>(lo + off) = *reinterpret_cast<uint4*>(l);
      }
      // one proxy fence orders this thread's generic reads of the raw box
      // before the TMA that refills it (WAR across proxies) and its plane
      // writes before the MMAs that read them
      tc::fence_proxy_async();
      tc::mbar_arrive(&raw_empty[r]);
      tc::mbar_arrive(&conv_full[b]);
      if constexpr (kAlpha) {
        // slot i % NAL: its previous tile (i - NAL) left the epilogue before
        // this converter could reach tile i (planes_empty of i - 2 needs the
        // accumulator of i - 6, drained after i - 8 by the same warpgroup)
        float* sa = reinterpret_cast<float*>(smem + OFF_RES) + (i % NAL) * HALO_PX;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (ct + q * NCONV < HALO_PX) sa[ct + q * NCONV] = alv[q];
        tc::mbar_arrive(&alpha_full[i % NAL]);
      }
    }
    if (ovf && a.ovf) atomicOr(a.ovf, 2);
  } else {
    // ---- epilogue: TMEM -> bias / GELU / residual -> swizzled smem -> TMA store ----
    const int ew = warp - 6;   // 0..NEW-1
    const int g = ew >> 2;     // warpgroup: tiles i with i % EPW == g
    const int q = warp & 3;    // TMEM lane quadrant this warp may access
    const int sy = q * SUB_ROWS;  // sub-box row offset inside the tile
    const uint32_t out_s = sbase + OFF_OUT + ew * SUB_BYTES;
    const uint32_t res_s = sbase + OFF_RES + ew * SUB_BYTES;
    uint8_t* out_p = smem + OFF_OUT + ew * SUB_BYTES;
    const uint8_t* res_p = smem + OFF_RES + ew * SUB_BYTES;
    const bool has_res = a.resid != nullptr;
    const int step = EPW * gridDim.x;
    uint32_t rph = 0;
    auto sub_valid = [&](const TileCoord& c) { return c.y0 + sy < a.H; };
    auto res_issue = [&](int t) {
      const TileCoord c = tile_coord(t, a.H, a.W);
      if (lane == 0 && sub_valid(c)) {
        tc::mbar_expect_tx(&res_full[ew], SUB_BYTES);
        tc::tma_load_4d(res_s, &rmap, 0, c.x0, c.y0 + sy, c.b, &res_full[ew]);
      }
    };
    int t = blockIdx.x + g * gridDim.x;
    if (has_res && t < num_tiles) res_issue(t);
    for (int i = g; t < num_tiles; t += step, i += EPW) {
      const int ac = i % NA;
      tc::mbar_wait(&mma_done[ac], uint32_t((i / NA) & 1));
      tc::fence_after();
      if ((LVSG_CONV_PROBE & 2)) {
        tc::mbar_arrive(&acc_empty[ac]);
        continue;
      }
      const uint32_t taddr = tmem + uint32_t(ac * 64) + (uint32_t(q * 32) << 16);
      float d0[32], d1[32];
      tc::tmem_ld32(taddr, d0);
      tc::tmem_ld32(taddr + 32, d1);
      tc::fence_before();
      tc::mbar_arrive(&acc_empty[ac]);
      const TileCoord tt = tile_coord(t, a.H, a.W);
      const bool valid = sub_valid(tt);
      float al[9];
      if constexpr (kAlpha) {  // the folded single-channel input: its 9 taps, from the halo
        const int row = q * 32 + lane;  // tile row m <-> pixel (y0 + m/8, x0 + m%8)
        tc::mbar_wait(&alpha_full[i % NAL], uint32_t((i / NAL) & 1));
        const float* sa = reinterpret_cast<const float*>(smem + OFF_RES) + (i % NAL) * HALO_PX;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
          al[tap] = sa[((row >> 3) + tap / 3) * HWD + (row & 7) + tap % 3];  // zero outside
      }
#pragma unroll
      for (int c = 0; c < 32; c += 2) {  // D[:, c] + 2^-11 D[:, 32 + c], packed (FFMA2)
        const float2 s = __ffma2_rn(make_float2(d1[c], d1[c + 1]),
                                    make_float2(1.0f / tc::kF16LoScale, 1.0f / tc::kF16LoScale),
                                    make_float2(d0[c], d0[c + 1]));
        d0[c] = s.x, d0[c + 1] = s.y;
      }
      if constexpr (kAlpha) {
        // the folded channel's 9 taps for 4 output channels per step, the
        // weights as 16-byte broadcasts (taps ascending per channel)
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          // packed f32x2 FMAs (FFMA2: the same per-lane roundings as fmaf)
          float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const float4 w = reinterpret_cast<const float4*>(walpha_s + tap * 32)[c4];
            const float2 a2 = make_float2(al[tap], al[tap]);
            s01 = __ffma2_rn(a2, make_float2(w.x, w.y), s01);
            s23 = __ffma2_rn(a2, make_float2(w.z, w.w), s23);
          }
          const float s4[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
          for (int k = 0; k < 4; ++k) d0[4 * c4 + k] = fa(d0[4 * c4 + k], s4[k]);
        }
      }
      if (a.bias) {
#pragma unroll
        for (int c = 0; c < 32; c += 2) {  // packed adds (FADD2); nothing multiplies into them
          const float2 s = __fadd2_rn(make_float2(d0[c], d0[c + 1]), make_float2(bias_s[c], bias_s[c + 1]));
          d0[c] = s.x, d0[c + 1] = s.y;
        }
      }
      if (a.gelu) {
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
#if LVSG_GELU2
          const float2 g2 = gelu2_ref(make_float2(d0[c], d0[c + 1]));
          d0[c] = g2.x, d0[c + 1] = g2.y;
#else
          d0[c] = gelu_ref(d0[c]);
          d0[c + 1] = gelu_ref(d0[c + 1]);
#endif
        }
      }
      if (has_res && valid) {
        tc::mbar_wait(&res_full[ew], rph);
        rph ^= 1u;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 r = *reinterpret_cast<const float4*>(res_p + swz(lane, c4));
          d0[4 * c4 + 0] = fa(r.x, d0[4 * c4 + 0]);
          d0[4 * c4 + 1] = fa(r.y, d0[4 * c4 + 1]);
          d0[4 * c4 + 2] = fa(r.z, d0[4 * c4 + 2]);
          d0[4 * c4 + 3] = fa(r.w, d0[4 * c4 + 3]);
        }
        tc::fence_proxy_async();  // the reads above before the TMA refilling the sub-box
        __syncwarp();
      }
      if (has_res && t + step < num_tiles) res_issue(t + step);
      if constexpr (kPool) {
        // the encoder's mean_pool2 of this warp's 4 x 8 sub-box: 2 x 2 groups
        // are lanes (l, l+1, l+8, l+9); same summation order as mean_pool2
        if (valid) {
          const int py = tt.y0 + sy + (lane >> 3), px = tt.x0 + (lane & 7);
          const bool writer = !(lane & 1) && !((lane >> 3) & 1) && (py >> 1) < (a.H >> 1) &&
                              (px >> 1) < (a.W >> 1);
          float* po = a.pool_out + (long long)tt.b * a.pool_bstride +
                      ((long long)(py >> 1) * (a.W >> 1) + (px >> 1)) * 32;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            float r[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float v00 = d0[4 * c4 + k];
              const float v01 = __shfl_down_sync(0xffffffffu, v00, 1);
              const float v10 = __shfl_down_sync(0xffffffffu, v00, 8);
              const float v11 = __shfl_down_sync(0xffffffffu, v00, 9);
              r[k] = fm(fa(fa(fa(v00, v01), v10), v11), 0.25f);
            }
            if (writer) {
              const float4 pv = make_float4(r[0], r[1], r[2], r[3]);
              *reinterpret_cast<float4*>(po + 4 * c4) = pv;
              // fused pyramid exchange: the same float4 into every peer's copy
              if constexpr (kPool == 2)
                for (int q = 0; q < a.npool_peer; ++q)
                  *reinterpret_cast<float4*>(a.pool_peer[q] + (po - a.pool_out) + 4 * c4) = pv;
            }
          }
          if constexpr (kPool == 2) __threadfence_system();  // peer stores before the barrier
        }
      }
      if (!valid) continue;
      if (lane == 0) tc::bulk_wait_read<0>();  // previous store left the staging buffer
      __syncwarp();
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4)
        *reinterpret_cast<float4*>(out_p + swz(lane, c4)) =
            make_float4(d0[4 * c4], d0[4 * c4 + 1], d0[4 * c4 + 2], d0[4 * c4 + 3]);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tc::tma_store_4d(&omap, out_s, 0, tt.x0, tt.y0 + sy, tt.b);
        tc::bulk_commit();
      }
    }
    if (lane == 0) tc::bulk_wait<0>();
  }
  tc::fence_before();
  __syncthreads();
  CONV_TL(2, atomicMax)
#ifdef LVSG_TIMELINE
  if (a.tl_slot > 0 && a.tl_slot <= kTlSlots && tid == 0) atomicAdd(&g_conv_tl[a.tl_slot - 1][3], 1ull);
#endif
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// Weight image: [tap][plane j][row n][8 halves], rows 0..31 = fp16 hi of
// w[co = n][w_ci0 + 8j + k8][tap], rows 32..63 = lo' (tc::split_f16).
__global__ void conv3x3_tc_weights_kernel(const ConvArgs a, __half* out) {
  pdl_grid_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 9 * NCH * W_ROWS * 8) return;
  const int k8 = e & 7, n = (e >> 3) & 63, rest = e >> 9;
  const int j = rest % NCH, tap = rest / NCH;
  const int co = n & 31, ci = 8 * j + k8;
  __half h, l;
  const float wv = __ldg(a.w + (co * w_cin_of(a) + a.w_ci0 + ci) * 9 + tap);
  tc::split_f16(wv, h, l);
  out[e] = n < 32 ? h : l;
  if (tc::split_overflows(wv) && a.ovf) atomicOr(a.ovf, 2);
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
  if (a.src[0].bstride % 4 || a.out_bstride % 4 || (a.resid && a.res_bstride % 4)) return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return encode_fn() && al(a.src[0].ptr) && al(a.out) && (!a.resid || al(a.resid)) &&
         (!a.gain || al(a.gain));
}

namespace {

// [B][H][W][pstride] fp32 (first 32 channels) as a 4-D tensor map.
CUtensorMap make_map(const float* p, long long pstride, long long bstride, int W, int H, int B,
                     cuuint32_t bw, cuuint32_t bh, CUtensorMapSwizzle swz) {
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  cuuint64_t dims[4] = {32, cuuint64_t(W), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(pstride) * 4, cuuint64_t(pstride) * 4 * W,
                           cuuint64_t(bstride) * 4};
  cuuint32_t box[4] = {32, bw, bh, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(p),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed");
  return map;
}

}  // namespace

void conv3x3_tc_prepare(const ConvArgs& a, void* dst, cudaStream_t st) {
  static_assert(kConvTcWeightBytes == W_BYTES, "weight image size");
  launch_k(conv3x3_tc_weights_kernel, (W_BYTES / 2 + 255) / 256, 256, 0, st, a,
           static_cast<__half*>(dst));
}

void conv3x3_tc(const ConvArgs& a, cudaStream_t st) {
  if (!a.wsplit || (reinterpret_cast<uintptr_t>(a.wsplit) & 15))
    throw CudaError("conv3x3_tc: missing or misaligned weight image (conv3x3_tc_prepare)");
  const ConvSrc& S = a.src[0];
  const CUtensorMap xmap =
      make_map(S.ptr, S.pstride, S.bstride, a.W, a.H, a.B, HWD, HHT, CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap omap = make_map(a.out, a.out_pstride, a.out_bstride, a.W, a.H, a.B, TW,
                                    SUB_ROWS, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap rmap = a.resid ? make_map(a.resid, a.res_pstride, a.res_bstride, a.W, a.H, a.B,
                                              TW, SUB_ROWS, CU_TENSOR_MAP_SWIZZLE_128B)
                                   : omap;
  const int tiles = a.B * ((a.H + TH - 1) / TH) * ((a.W + TW - 1) / TW);
  const int sms = sm_count();
  const int grid = tiles < sms ? tiles : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute lattr[1];
  lattr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  lattr[0].val.programmaticStreamSerializationAllowed = (a.pdl && pdl_enabled()) ? 1 : 0;
  cfg.attrs = lattr;
  cfg.numAttrs = 1;
  auto kern = a.alpha                         ? conv3x3_tc_kernel<true, 0>
              : a.pool_out && a.npool_peer > 0 ? conv3x3_tc_kernel<false, 2>
              : a.pool_out                    ? conv3x3_tc_kernel<false, 1>
                                              : conv3x3_tc_kernel<false, 0>;
  smem_optin(reinterpret_cast<const void*>(kern), SMEM_BYTES);
  if (a.alpha && a.pool_out) throw CudaError("conv3x3_tc: alpha and pool together are not built");
  // the alpha halos live in the residual staging area
  if (a.alpha && a.resid) throw CudaError("conv3x3_tc: alpha and a residual together are not built");
  if (cudaLaunchKernelEx(&cfg, kern, xmap, omap, rmap, a, tiles) != cudaSuccess)
    throw CudaError("conv3x3_tc: launch failed");
}

void conv_timeline_reset() {
#ifdef LVSG_TIMELINE
  static unsigned long long init[kTlSlots][4];
  for (int i = 0; i < kTlSlots; ++i) {
    init[i][0] = init[i][1] = ~0ull;
    init[i][2] = init[i][3] = 0;
  }
  cudaMemcpyToSymbol(g_conv_tl, init, sizeof(init));
#endif
}
int conv_timeline_read(unsigned long long* out, int slots) {
#ifdef LVSG_TIMELINE
  const int n = slots < kTlSlots ? slots : kTlSlots;
  cudaMemcpyFromSymbol(out, g_conv_tl, size_t(n) * 4 * sizeof(unsigned long long));
  return n;
#else
  (void)out;
  (void)slots;
  return -1;
#endif
}

}  // namespace lvsg
