// conv3x3 (Cin = Cout = 32, channel-last) with a 1-D Winograd F(2,3) along x
// and the direct tap shift along y, on the sm_100a tensor core (tcgen05.mma
// kind::f16, the same 3-term fp16 split as conv_tc.cu).
//
// Why: at M = 128 every SS-mode MMA pays ~50 cycles of exposed A-operand read
// on top of its math (50 + N/2 cycles measured), so the direct
// conv is bound by its MMA count (72 per 256 output pixels). F(2,3) along x
// computes two adjacent outputs from four transformed inputs:
//     v0 = d0 - d2, v1 = d1 + d2, v2 = d2 - d1, v3 = d1 - d3        (B^T d)
//     u0 = g0, u1 = (g0 + g1 + g2)/2, u2 = (g0 - g1 + g2)/2, u3 = g2  (G g)
//     y(2t) = m0 + m1 + m2,  y(2t+1) = m1 - m2 - m3                    (A^T m)
// with m_xi = sum_dy sum_ci v_xi(y+dy) u_xi(dy): 4 GEMMs per pixel pair, each
// K = 3 dy x 32 ci -- 48 MMAs per 256 output pixels. The dy taps stay free:
// the transformed planes hold all 18 halo rows and a dy shift is a
// descriptor start offset of 8 rows (one core-matrix group).
//
// Work item = 16 output rows x 16 output columns: M = 128 GEMM rows
// r = 8y + t <-> output pixels (y0+y, x0+2t) and (y0+y, x0+2t+1). The 18 x 18
// x 32 halo arrives by one TMA box (128B-swizzled); converter warps build the
// four transformed planes V_xi [18 rows x 8 pairs][32 ch] as fp16 hi / lo'
// (K-major interleave) through a 3-deep ring; the MMA warp accumulates
// D_xi [128 x 64] (hi | lo columns) in TMEM, two work items deep (512 cols);
// the epilogue warpgroup inverts the transform, applies bias / GELU /
// residual and leaves through a 128B-swizzled staging box and TMA stores.
// Semantics of kernels_ref.hpp:72-96 (zero padding), options as conv_tc.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "host.h"
#include "kernels.h"
#include "tc.cuh"

// Development probe bitmask (0 in shipped builds): skip the MMAs (1), the
// epilogue (2), the converters' transforms (4), the TMA loads (8).
#ifndef LVSG_CONV_PROBE
#define LVSG_CONV_PROBE 0
#endif

namespace lvsg {
namespace {

constexpr int OW = 16, OH = 16;              // output block
constexpr int NTX = OW / 2;                  // pixel pairs per row
constexpr int HW_ = OW + 2, HH_ = OH + 2;    // 18 x 18 halo
constexpr int HALO_PX = HW_ * HH_;           // 324
constexpr int RAW_BYTES = HALO_PX * 128;     // 41472
constexpr int RAW_STRIDE = 41 * 1024;        // 1 KB aligned stages (128B swizzle)
constexpr int VROWS = HH_ * NTX;             // 144 plane rows (hy, t)
constexpr int LBO_V = VROWS * 16;            // one 8-channel group: 2304 B
constexpr int V_HALF = 4 * LBO_V;            // hi (or lo') planes: 9216 B
constexpr int V_SLOT = 2 * V_HALF;           // 18432 B
constexpr int W_BYTES = 4 * 3 * 4 * 64 * 16; // [xi][dy][j][64 rows][8 halves] = 49152
constexpr int NR = 2, NV = 3;
constexpr int STG_BYTES = 4 * 16 * 128;      // per epilogue warp: [4 rows][16 px][128 B]
constexpr int OFF_STG = 0;
constexpr int OFF_W = OFF_STG + 4 * STG_BYTES;   // 32768
constexpr int OFF_RAW = OFF_W + W_BYTES;         // 81920
constexpr int OFF_V = OFF_RAW + NR * RAW_STRIDE;
constexpr int OFF_SMALL = OFF_V + NV * V_SLOT;   // rms[324 -> 328], bias[32], gain[32]
constexpr int OFF_BAR = OFF_SMALL + (328 + 64) * 4;
constexpr int NBAR = 2 * NR + 2 * NV + 2 + 2 + 4 + 1;
constexpr int SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
constexpr int NT = 320;                          // producer, MMA, 4 converter, 4 epilogue warps
constexpr int NCONV = 128, NEPI = 128;
constexpr uint32_t TMEM_COLS = 512;              // 2 work items x 4 xi x 64 columns
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
static_assert(OFF_RAW % 1024 == 0 && RAW_STRIDE % 1024 == 0 && OFF_W % 1024 == 0, "alignment");

struct Item {
  int b, y0, x0;
};

__device__ __forceinline__ Item item_of(int t, int H, int W) {
  const int nx = (W + OW - 1) / OW, ny = (H + OH - 1) / OH;
  Item c;
  c.b = t / (nx * ny);
  const int r = t - c.b * nx * ny;
  c.y0 = (r / nx) * OH;
  c.x0 = (r % nx) * OW;
  return c;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// chunk c (16 B, 4 channels) of halo pixel px in the 128B-swizzled raw box
__device__ __forceinline__ const float4* raw_chunk(const uint8_t* raw, int px, int c) {
  return reinterpret_cast<const float4*>(raw + px * 128 + ((c ^ (px & 7)) << 4));
}
// 16-byte chunk c4 of row r in a 128B-swizzled [rows][128 B] staging box
__device__ __forceinline__ uint32_t swz(int r, int c4) {
  return uint32_t(r * 128 + ((c4 ^ (r & 7)) << 4));
}

__global__ void __launch_bounds__(NT, 1)
    conv3x3_wino_kernel(const __grid_constant__ CUtensorMap xmap,
                        const __grid_constant__ CUtensorMap omap,
                        const __grid_constant__ CUtensorMap rmap, const ConvArgs a, int num_items) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* rms_s = reinterpret_cast<float*>(smem + OFF_SMALL);
  float* bias_s = rms_s + 328;
  float* gain_s = bias_s + 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* raw_full = bars;            // [NR]
  uint64_t* raw_empty = raw_full + NR;  // [NR]
  uint64_t* v_full = raw_empty + NR;    // [NV] transformed plane written
  uint64_t* v_empty = v_full + NV;      // [NV] MMAs done with it
  uint64_t* mma_done = v_empty + NV;    // [2] work item accumulated
  uint64_t* acc_empty = mma_done + 2;   // [2] accumulators drained
  uint64_t* res_full = acc_empty + 2;   // [4] residual sub-box landed (per epilogue warp)
  uint64_t* w_full = res_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  tc::pdl_launch_dependents();
  if (blockIdx.x >= num_items) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = tc::smem_u32(smem);
  if (tid == 0 && (sbase & 1023u)) __trap();

  if (tid < 32) bias_s[tid] = a.bias ? __ldg(a.bias + tid) : 0.f;
  else if (tid < 64) gain_s[tid - 32] = a.gain ? __ldg(a.gain + tid - 32) : 1.f;
  if (tid == 0) {
    for (int k = 0; k < NR; ++k) {
      tc::mbar_init(&raw_full[k], 1);
      tc::mbar_init(&raw_empty[k], NCONV);
    }
    for (int k = 0; k < NV; ++k) {
      tc::mbar_init(&v_full[k], NCONV);
      tc::mbar_init(&v_empty[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(&mma_done[k], 1);
      tc::mbar_init(&acc_empty[k], NEPI);
    }
    for (int k = 0; k < 4; ++k) tc::mbar_init(&res_full[k], 1);
    tc::mbar_init(w_full, 1);
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  tc::pdl_wait();  // global data only below
  if (tid == 0) {
    tc::mbar_expect_tx(w_full, W_BYTES);
    tc::bulk_load(sbase + OFF_W, a.wsplit, W_BYTES, w_full);
  }

  if (warp == 0) {
    // ---- TMA producer: one 18 x 18 x 32 halo box per work item ----
    if (lane == 0) {
      int i = 0;
      for (int t = blockIdx.x; t < num_items; t += gridDim.x, ++i) {
        const int r = i % NR;
        if (i >= NR) tc::mbar_wait(&raw_empty[r], uint32_t((i / NR - 1) & 1));
        if (LVSG_CONV_PROBE & 8) {
          tc::mbar_arrive(&raw_full[r]);
          continue;
        }
        const Item it = item_of(t, a.H, a.W);
        tc::mbar_expect_tx(&raw_full[r], RAW_BYTES);
        tc::tma_load_4d(sbase + OFF_RAW + r * RAW_STRIDE, &xmap, 0, it.x0 - 1, it.y0 - 1, it.b,
                        &raw_full[r]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: per work item 4 xi x 3 dy x 2 K steps x (N=64, N=32) ----
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    constexpr uint32_t id64 = tc::idesc_f16(128, 64);
    constexpr uint32_t id32 = tc::idesc_f16(128, 32);
    tc::mbar_wait(w_full, 0);
    int i = 0;
    for (int t = blockIdx.x; t < num_items; t += gridDim.x, ++i) {
      const int bb = i & 1;
      if (i >= 2) tc::mbar_wait(&acc_empty[bb], uint32_t(((i >> 1) - 1) & 1));
      for (int xi = 0; xi < 4; ++xi) {
        const int u = 4 * i + xi, slot = u % NV;
        tc::mbar_wait(&v_full[slot], uint32_t((u / NV) & 1));
        tc::fence_after();
        if (tc::elect_one()) {
          const uint32_t d = tm + uint32_t(bb * 256 + xi * 64);
          const uint32_t vh = sbase + OFF_V + slot * V_SLOT;
          const uint64_t ah = tc::smem_desc(vh, LBO_V, 128), al = tc::smem_desc(vh + V_HALF, LBO_V, 128);
          const uint64_t bw = tc::smem_desc(sbase + OFF_W, 64 * 16, 128);
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              if (LVSG_CONV_PROBE & 1) break;
              const uint64_t ao = uint64_t((2 * s * LBO_V + dy * 8 * 16) >> 4);
              const uint64_t bo = uint64_t((((xi * 3 + dy) * 4 + 2 * s) * 64 * 16) >> 4);
              tc::mma_f16(d, ah + ao, bw + bo, id64, (dy | s) != 0);
              tc::mma_f16(d + 32, al + ao, bw + bo, id32, 1u);
            }
          tc::commit(&v_empty[slot]);
          if (xi == 3) tc::commit(&mma_done[bb]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---- converters: raw halo -> transformed fp16 hi / lo' planes ----
    const int ct = tid - 64;
    const int j = ct & 3;  // 8-channel group of this thread's items
    float g8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) g8[k] = gain_s[8 * j + k];
    int i = 0;
    for (int t = blockIdx.x; t < num_items; t += gridDim.x, ++i) {
      const int r = i % NR;
      const uint8_t* raw = smem + OFF_RAW + r * RAW_STRIDE;
      tc::mbar_wait(&raw_full[r], uint32_t((i / NR) & 1));
      if (a.rinv) {
        // conv_mlp_residual's rms_norm: one scale per halo pixel
        named_sync(1, NCONV);  // the previous item's readers are done
        for (int px = ct; px < HALO_PX; px += NCONV) {
          float ms = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *raw_chunk(raw, px, c);
            ms = fmaf(v.x, v.x, ms);
            ms = fmaf(v.y, v.y, ms);
            ms = fmaf(v.z, v.z, ms);
            ms = fmaf(v.w, v.w, ms);
          }
          rms_s[px] = __fdiv_rn(1.0f, __fsqrt_rn(fa(fm(ms, 0.03125f), 1e-6f)));
        }
        named_sync(1, NCONV);
      }
      for (int xi = 0; xi < 4; ++xi) {
        const int u = 4 * i + xi, slot = u % NV;
        if (u >= NV) tc::mbar_wait(&v_empty[slot], uint32_t((u / NV - 1) & 1));
        uint8_t* vh = smem + OFF_V + slot * V_SLOT;
        // v = d[ka] + sgn * d[kb]
        const int ka = xi == 0 ? 0 : xi == 2 ? 2 : 1;
        const int kb = xi == 0 ? 2 : xi == 1 ? 2 : xi == 2 ? 1 : 3;
        const bool add = xi == 1;
        for (int e = ct; e < ((LVSG_CONV_PROBE & 4) ? 0 : VROWS * 4); e += NCONV) {
          const int tx = (e >> 2) & 7, hy = e >> 5;
          const int pa = hy * HW_ + 2 * tx + ka, pb = hy * HW_ + 2 * tx + kb;
          float da[8], db[8];
          {
            const float4 a0 = *raw_chunk(raw, pa, 2 * j), a1 = *raw_chunk(raw, pa, 2 * j + 1);
            const float4 b0 = *raw_chunk(raw, pb, 2 * j), b1 = *raw_chunk(raw, pb, 2 * j + 1);
            da[0] = a0.x, da[1] = a0.y, da[2] = a0.z, da[3] = a0.w;
            da[4] = a1.x, da[5] = a1.y, da[6] = a1.z, da[7] = a1.w;
            db[0] = b0.x, db[1] = b0.y, db[2] = b0.z, db[3] = b0.w;
            db[4] = b1.x, db[5] = b1.y, db[6] = b1.z, db[7] = b1.w;
          }
          if (a.rinv) {
            const float ra = rms_s[pa], rb = rms_s[pb];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              da[k] = fm(fm(da[k], ra), g8[k]);
              db[k] = fm(fm(db[k], rb), g8[k]);
            }
          }
          __align__(16) __half h[8], l[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) tc::split_f16(add ? fa(da[k], db[k]) : fsb(da[k], db[k]), h[k], l[k]);
          const int off = j * LBO_V + (hy * NTX + tx) * 16;
          *reinterpret_cast<uint4*>(vh + off) = *reinterpret_cast<uint4*>(h);
          *reinterpret_cast<uint4*>(vh + V_HALF + off) = *reinterpret_cast<uint4*>(l);
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&v_full[slot]);
      }
      tc::mbar_arrive(&raw_empty[r]);
    }
  } else {
    // ---- epilogue: inverse transform + bias / GELU / residual -> TMA store ----
    const int ew = warp - 6;   // 0..3
    const int q = warp & 3;    // TMEM lane quadrant
    const int row = q * 32 + lane;
    const int ly = (row >> 3) - 4 * q, tx = row & 7;  // local row in the warp's 4-row box
    const int sy = 4 * q;
    const uint32_t lane_base = uint32_t(q * 32) << 16;
    const uint32_t stg = sbase + OFF_STG + ew * STG_BYTES;
    uint8_t* stg_p = smem + OFF_STG + ew * STG_BYTES;
    const bool has_res = a.resid != nullptr;
    uint32_t rph = 0;
    auto res_issue = [&](int t) {
      const Item it = item_of(t, a.H, a.W);
      if (lane == 0 && it.y0 + sy < a.H) {
        tc::mbar_expect_tx(&res_full[ew], STG_BYTES);
        tc::tma_load_4d(stg, &rmap, 0, it.x0, it.y0 + sy, it.b, &res_full[ew]);
      }
    };
    if (has_res && blockIdx.x < num_items) res_issue(blockIdx.x);
    int i = 0;
    for (int t = blockIdx.x; t < num_items; t += gridDim.x, ++i) {
      const int bb = i & 1;
      tc::mbar_wait(&mma_done[bb], uint32_t((i >> 1) & 1));
      tc::fence_after();
      if (LVSG_CONV_PROBE & 2) {
        tc::mbar_arrive(&acc_empty[bb]);
        continue;
      }
      float y0[32], y1[32];
#pragma unroll
      for (int xi = 0; xi < 4; ++xi) {
        float hi[32], lo[32];
        const uint32_t col = tmem + lane_base + uint32_t(bb * 256 + xi * 64);
        tc::tmem_ld32(col, hi);
        tc::tmem_ld32(col + 32, lo);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float m = fmaf(lo[c], 1.0f / tc::kF16LoScale, hi[c]);
          if (xi == 0) {
            y0[c] = m;
          } else if (xi == 1) {
            y0[c] = fa(y0[c], m);
            y1[c] = m;
          } else if (xi == 2) {
            y0[c] = fa(y0[c], m);
            y1[c] = fsb(y1[c], m);
          } else {
            y1[c] = fsb(y1[c], m);
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&acc_empty[bb]);
      const Item it = item_of(t, a.H, a.W);
      const bool valid = it.y0 + sy < a.H;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        float u0 = y0[c], u1 = y1[c];
        if (a.bias) {
          u0 = fa(u0, bias_s[c]);
          u1 = fa(u1, bias_s[c]);
        }
        if (a.gelu) {
          u0 = gelu_ref(u0);
          u1 = gelu_ref(u1);
        }
        y0[c] = u0;
        y1[c] = u1;
      }
      const int i0 = ly * 16 + 2 * tx, i1 = i0 + 1;  // staging rows of my two pixels
      if (has_res && valid) {
        tc::mbar_wait(&res_full[ew], rph);
        rph ^= 1u;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 r0 = *reinterpret_cast<const float4*>(stg_p + swz(i0, c4));
          const float4 r1 = *reinterpret_cast<const float4*>(stg_p + swz(i1, c4));
          y0[4 * c4] = fa(r0.x, y0[4 * c4]);
          y0[4 * c4 + 1] = fa(r0.y, y0[4 * c4 + 1]);
          y0[4 * c4 + 2] = fa(r0.z, y0[4 * c4 + 2]);
          y0[4 * c4 + 3] = fa(r0.w, y0[4 * c4 + 3]);
          y1[4 * c4] = fa(r1.x, y1[4 * c4]);
          y1[4 * c4 + 1] = fa(r1.y, y1[4 * c4 + 1]);
          y1[4 * c4 + 2] = fa(r1.z, y1[4 * c4 + 2]);
          y1[4 * c4 + 3] = fa(r1.w, y1[4 * c4 + 3]);
        }
        __syncwarp();
      }
      if (valid) {
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          *reinterpret_cast<float4*>(stg_p + swz(i0, c4)) =
              make_float4(y0[4 * c4], y0[4 * c4 + 1], y0[4 * c4 + 2], y0[4 * c4 + 3]);
          *reinterpret_cast<float4*>(stg_p + swz(i1, c4)) =
              make_float4(y1[4 * c4], y1[4 * c4 + 1], y1[4 * c4 + 2], y1[4 * c4 + 3]);
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_4d(&omap, stg, 0, it.x0, it.y0 + sy, it.b);
          tc::bulk_commit();
          tc::bulk_wait_read<0>();  // the staging box is free again
        }
        __syncwarp();
      }
      // the next item's residual lands in the (now free) staging box
      if (has_res && t + int(gridDim.x) < num_items) res_issue(t + gridDim.x);
    }
    if (lane == 0) tc::bulk_wait<0>();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// Weight image [xi][dy][j][n][8 halves]: rows n < 32 = fp16 hi, 32..63 = lo' of
// u_xi(dy)[co = n & 31][ci = 8j + k8] (G g of the three dx taps of row dy).
__global__ void conv3x3_wino_weights_kernel(const ConvArgs a, __half* out) {
  pdl_grid_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W_BYTES / 2) return;
  const int k8 = e & 7, n = (e >> 3) & 63, rest = e >> 9;
  const int j = rest & 3, dy = (rest >> 2) % 3, xi = (rest >> 2) / 3;
  const int co = n & 31, ci = 8 * j + k8;
  const float* g = a.w + ((long long)co * w_cin_of(a) + a.w_ci0 + ci) * 9 + dy * 3;
  const float g0 = __ldg(g), g1 = __ldg(g + 1), g2 = __ldg(g + 2);
  const float uu = xi == 0   ? g0
                   : xi == 1 ? fm(fa(fa(g0, g1), g2), 0.5f)
                   : xi == 2 ? fm(fa(fsb(g0, g1), g2), 0.5f)
                             : g2;
  __half h, l;
  tc::split_f16(uu, h, l);
  out[e] = n < 32 ? h : l;
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

CUtensorMap make_map(const float* p, long long pstride, long long bstride, int W, int H, int B,
                     cuuint32_t bw, cuuint32_t bh) {
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  cuuint64_t dims[4] = {32, cuuint64_t(W), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(pstride) * 4, cuuint64_t(pstride) * 4 * W,
                           cuuint64_t(bstride) * 4};
  cuuint32_t box[4] = {32, bw, bh, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  if (encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(p), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed");
  return map;
}

}  // namespace

bool conv3x3_wino_supported(const ConvArgs& a) { return conv3x3_tc_supported(a) && encode_fn(); }

void conv3x3_wino_prepare(const ConvArgs& a, void* dst, cudaStream_t st) {
  static_assert(kConvWinoWeightBytes == W_BYTES, "weight image size");
  launch_k(conv3x3_wino_weights_kernel, (W_BYTES / 2 + 255) / 256, 256, 0, st, a,
           static_cast<__half*>(dst));
}

void conv3x3_wino(const ConvArgs& a, cudaStream_t st) {
  if (!a.wsplit || (reinterpret_cast<uintptr_t>(a.wsplit) & 15))
    throw CudaError("conv3x3_wino: missing or misaligned weight image (conv3x3_wino_prepare)");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3x3_wino_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES);
    attr = true;
  }
  const ConvSrc& S = a.src[0];
  const CUtensorMap xmap = make_map(S.ptr, S.pstride, S.bstride, a.W, a.H, a.B, HW_, HH_);
  const CUtensorMap omap = make_map(a.out, a.out_pstride, a.out_bstride, a.W, a.H, a.B, OW, 4);
  const CUtensorMap rmap =
      a.resid ? make_map(a.resid, a.res_pstride, a.res_bstride, a.W, a.H, a.B, OW, 4) : omap;
  const int items = a.B * ((a.H + OH - 1) / OH) * ((a.W + OW - 1) / OW);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = items < sms ? items : sms;
  launch_pdl(a.pdl != 0, conv3x3_wino_kernel, grid, NT, SMEM_BYTES, st, xmap, omap, rmap, a,
             items);
}

}  // namespace lvsg
