// Stage 2 (One-to-many attention, attention.hpp:207-252) fused on the
// sm_100a tensor core, C = 32, h <= 4 heads, M views:
//
//   n      = rms_norm(V) * g                     (SIMT, thread = texel)
//   S      = n [Wq_0 | ... | Wq_{h-1}]           tcgen05.mma kind::tf32, 3xTF32,
//                                                M=128 texels, N=32h, TMEM
//   l_im   = <S_i, Δ_m> / sqrt(C); w = softmax_m; head_i = sum_m w_im Δ_m
//                                                (SIMT over coalesced Δ[m][g][p])
//   O      = sum_i head_i Wo_i                   tcgen05.mma, 3xTF32, TMEM
//   V     += O
//
// Persistent CTAs (2 per SM), 128 threads, thread t <-> texel row t <-> TMEM
// lane t. Weights are pre-split into tf32 hi/lo and kept resident in shared
// memory in the K-major interleave layout; A operands (n, then each head)
// are staged the same way. Δ is read once for all heads' scores (S_i re-read
// from TMEM per view) and once per head for the mix, from the L2-resident
// 128-texel tile.
#include <cfloat>

#include "kernels.h"
#include "tc.cuh"

namespace lvsg {
namespace {

constexpr int C = 32;
constexpr int TILE = 128;
constexpr int NT = 128;
constexpr int NCH = C / 4;                 // 16-byte K chunks
constexpr int A_LBO = TILE * 16;           // 2048
constexpr int A_BYTES = NCH * A_LBO;       // 16 KB per plane
// TMEM per CTA: S (32h columns) then O (32 columns), rounded up to a power of
// two -- 64 / 128 / 256 columns for h = 1 / 2 / 4, which bounds how many
// CTAs share an SM's 512 columns; registers set the rest (4 / 3 / 2 CTAs).
template <int H>
constexpr uint32_t tmem_cols() {
  return H == 1 ? 64u : H == 2 ? 128u : 256u;
}
template <int H>
constexpr int ctas_per_sm() {
  return H == 1 ? 4 : H == 2 ? 3 : 2;
}

template <int H>
struct Smem {
  static constexpr int BQ_LBO = 32 * H * 16;
  static constexpr int BQ_BYTES = NCH * BQ_LBO;  // one plane
  static constexpr int BO_LBO = 32 * 16;
  static constexpr int BO_BYTES = NCH * BO_LBO;  // one head, one plane
  static constexpr int OFF_BQH = 2 * A_BYTES;
  static constexpr int OFF_BQL = OFF_BQH + BQ_BYTES;
  static constexpr int OFF_BO = OFF_BQL + BQ_BYTES;  // [head][hi|lo]
  static constexpr int OFF_BAR = OFF_BO + 2 * H * BO_BYTES;
  static constexpr int BYTES = OFF_BAR + 32;
};

__device__ __forceinline__ void put_split(float* hi, float* lo, int off, float4 v) {
  float4 h, l;
  tc::split_tf32(v.x, h.x, l.x);
  tc::split_tf32(v.y, h.y, l.y);
  tc::split_tf32(v.z, h.z, l.z);
  tc::split_tf32(v.w, h.w, l.w);
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = l;
}

// A[j][row][4] <- x[32] of this thread's row, split into tf32 hi/lo planes.
__device__ __forceinline__ void stage_row(uint8_t* smem, int row, const float* x) {
  float* hi = reinterpret_cast<float*>(smem);
  float* lo = reinterpret_cast<float*>(smem + A_BYTES);
#pragma unroll
  for (int j = 0; j < NCH; ++j)
    put_split(hi, lo, (j * A_LBO) / 4 + row * 4,
              make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]));
}

// D (N columns) (+)= Ahi*Bhi + Ahi*Blo + Alo*Bhi over K = 32.
__device__ __forceinline__ void mma3(uint32_t tmem_d, uint64_t ahi, uint64_t alo, uint64_t bhi,
                                     uint64_t blo, uint32_t bstep, uint32_t idesc, bool acc0) {
#pragma unroll
  for (int s = 0; s < NCH / 2; ++s) {
    const uint64_t ao = uint64_t((2 * s * A_LBO) >> 4);
    const uint64_t bo = uint64_t((2 * s * bstep) >> 4);
    tc::mma_tf32(tmem_d, ahi + ao, bhi + bo, idesc, (acc0 || s > 0) ? 1u : 0u);
    tc::mma_tf32(tmem_d, ahi + ao, blo + bo, idesc, 1u);
    tc::mma_tf32(tmem_d, alo + ao, bhi + bo, idesc, 1u);
  }
}

template <int H, int M>
__global__ void __launch_bounds__(NT, ctas_per_sm<H>()) attend_tc_kernel(float* V, const float* __restrict__ D,
                                                         int64_t P, const float* __restrict__ wq,
                                                         const float* __restrict__ wo,
                                                         const float* __restrict__ gain,
                                                         int zero_scores, int num_tiles) {
  using S = Smem<H>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x >= num_tiles) return;

  // resident weights, tf32 hi/lo, K-major:
  //   Bq[j][n][4]  n = 32*i + c : Wq_i[4j..4j+3][c]
  //   Bo[i][j][n][4]            : Wo[32i + 4j..][n]
  {
    float* bqh = reinterpret_cast<float*>(smem + S::OFF_BQH);
    float* bql = reinterpret_cast<float*>(smem + S::OFF_BQL);
    for (int e = tid; e < NCH * 32 * H; e += NT) {
      const int n = e % (32 * H), j = e / (32 * H);
      const int i = n / 32, c = n % 32;
      const float* src = wq + (i * C + 4 * j) * C + c;
      put_split(bqh, bql, (j * S::BQ_LBO) / 4 + n * 4,
                make_float4(__ldg(src), __ldg(src + C), __ldg(src + 2 * C), __ldg(src + 3 * C)));
    }
    for (int e = tid; e < H * NCH * 32; e += NT) {
      const int n = e % 32, j = (e / 32) % NCH, i = e / (32 * NCH);
      float* bh = reinterpret_cast<float*>(smem + S::OFF_BO + (2 * i) * S::BO_BYTES);
      float* bl = reinterpret_cast<float*>(smem + S::OFF_BO + (2 * i + 1) * S::BO_BYTES);
      const float* src = wo + (i * C + 4 * j) * C + n;
      put_split(bh, bl, (j * S::BO_LBO) / 4 + n * 4,
                make_float4(__ldg(src), __ldg(src + C), __ldg(src + 2 * C), __ldg(src + 3 * C)));
    }
  }
  if (tid == 0) {
    tc::mbar_init(bar_s, 1);
    tc::mbar_init(bar_o, 1);
    tc::mbar_init_fence();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, tmem_cols<H>());
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  const uint32_t tmem_s = tmem, tmem_o = tmem + 32 * H;

  const uint32_t sb = tc::smem_u32(smem);
  const uint64_t ahi = tc::smem_desc(sb + 0, A_LBO, 128);
  const uint64_t alo = tc::smem_desc(sb + A_BYTES, A_LBO, 128);
  const uint64_t bqh = tc::smem_desc(sb + S::OFF_BQH, S::BQ_LBO, 128);
  const uint64_t bql = tc::smem_desc(sb + S::OFF_BQL, S::BQ_LBO, 128);
  constexpr uint32_t id_s = tc::idesc_tf32(128, 32 * H);
  constexpr uint32_t id_o = tc::idesc_tf32(128, 32);
  const float inv_temp = __double2float_rn(1.0 / sqrt(double(C)));
  uint32_t ph_s = 0, ph_o = 0;

  for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    const int64_t p = int64_t(tile) * TILE + tid;
    const bool valid = p < P;
    // ---- n = rms_norm(V) * g  -> A ----
    float x[C];
    if (valid) {
      const float4* vr = reinterpret_cast<const float4*>(V + p * C);
#pragma unroll
      for (int k = 0; k < C / 4; ++k) {
        const float4 t = vr[k];
        x[4 * k] = t.x, x[4 * k + 1] = t.y, x[4 * k + 2] = t.z, x[4 * k + 3] = t.w;
      }
      float ms = 0.f;
#pragma unroll
      for (int k = 0; k < C; ++k) ms = fmaf(x[k], x[k], ms);
      const float r = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(ms, float(C)), 1e-6f)));
#pragma unroll
      for (int k = 0; k < C; ++k) x[k] = fm(fm(x[k], r), __ldg(gain + k));
    } else {
#pragma unroll
      for (int k = 0; k < C; ++k) x[k] = 0.f;
    }
    stage_row(smem, tid, x);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0) {  // whole warp, one elected lane issues (uniform descriptors)
      if (tc::elect_one()) {
        mma3(tmem_s, ahi, alo, bqh, bql, S::BQ_LBO, id_s, false);
        tc::commit(bar_s);
      }
      __syncwarp();
    }

    // ---- scores: one pass over Δ, S_i re-read from TMEM per view ----
    const float4* d4 = reinterpret_cast<const float4*>(D) + (valid ? p : 0);
    float w[H][M];
    tc::mbar_wait(bar_s, ph_s);
    ph_s ^= 1u;
    tc::fence_after();
    if (zero_scores) {
#pragma unroll
      for (int i = 0; i < H; ++i)
#pragma unroll
        for (int m = 0; m < M; ++m) w[i][m] = __fdiv_rn(1.0f, float(M));
    } else {
      // software pipeline: view m+1's Δ row is in flight while view m's
      // dot products run
      float4 nx[C / 4];
#pragma unroll
      for (int g = 0; g < C / 4; ++g)
        nx[g] = valid ? __ldg(d4 + int64_t(g) * P) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
      for (int m = 0; m < M; ++m) {
        float dm[C];
#pragma unroll
        for (int g = 0; g < C / 4; ++g) {
          const float4 t = nx[g];
          dm[4 * g] = t.x, dm[4 * g + 1] = t.y, dm[4 * g + 2] = t.z, dm[4 * g + 3] = t.w;
        }
        if (m + 1 < M) {
#pragma unroll
          for (int g = 0; g < C / 4; ++g)
            nx[g] = valid ? __ldg(d4 + (int64_t(m + 1) * (C / 4) + g) * P)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < H; ++i) {
          float si[C];
          tc::tmem_ld32(tmem_s + lane_base + uint32_t(32 * i), si);
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < C; ++c) acc = fmaf(si[c], dm[c], acc);
          // dynamic m: keep w in registers through a select chain
#pragma unroll
          for (int mm = 0; mm < M; ++mm)
            if (mm == m) w[i][mm] = fm(acc, inv_temp);
        }
      }
      // softmax over views (tape.hpp:390-404: max, exp(x - max), sum, * 1/sum)
#pragma unroll
      for (int i = 0; i < H; ++i) {
        float mx = w[i][0];
#pragma unroll
        for (int m = 1; m < M; ++m) mx = fmaxf(mx, w[i][m]);
        float sum = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          w[i][m] = expf(fsb(w[i][m], mx));
          sum = fa(sum, w[i][m]);
        }
        const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
        for (int m = 0; m < M; ++m) w[i][m] = fm(w[i][m], inv);
      }
    }

    // ---- per head: mix over Δ (L2-resident tile), stage, O += head Wo_i ----
#pragma unroll
    for (int i = 0; i < H; ++i) {
      float hd[C];
#pragma unroll
      for (int c = 0; c < C; ++c) hd[c] = 0.f;
#pragma unroll 2
      for (int m = 0; m < M; ++m) {
        float wm = w[i][0];  // select chain: w stays in registers for runtime m
#pragma unroll
        for (int mm = 1; mm < M; ++mm)
          if (mm == m) wm = w[i][mm];
#pragma unroll
        for (int g = 0; g < C / 4; ++g) {
          const float4 t = valid ? __ldg(d4 + (int64_t(m) * (C / 4) + g) * P)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
          hd[4 * g] = fmaf(wm, t.x, hd[4 * g]);
          hd[4 * g + 1] = fmaf(wm, t.y, hd[4 * g + 1]);
          hd[4 * g + 2] = fmaf(wm, t.z, hd[4 * g + 2]);
          hd[4 * g + 3] = fmaf(wm, t.w, hd[4 * g + 3]);
        }
      }
      if (i > 0) {  // the previous head's MMAs have read A
        tc::mbar_wait(bar_o, ph_o);
        ph_o ^= 1u;
      }
      stage_row(smem, tid, hd);
      tc::fence_proxy_async();
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      if (warp == 0) {
        if (tc::elect_one()) {
          const uint64_t boh = tc::smem_desc(sb + S::OFF_BO + (2 * i) * S::BO_BYTES, S::BO_LBO, 128);
          const uint64_t bol =
              tc::smem_desc(sb + S::OFF_BO + (2 * i + 1) * S::BO_BYTES, S::BO_LBO, 128);
          mma3(tmem_o, ahi, alo, boh, bol, S::BO_LBO, id_o, i > 0);
          tc::commit(bar_o);
        }
        __syncwarp();
      }
    }
    tc::mbar_wait(bar_o, ph_o);
    ph_o ^= 1u;
    tc::fence_after();
    float o[C];
    tc::tmem_ld32(tmem_o + lane_base, o);
    if (valid) {
      float4* vw = reinterpret_cast<float4*>(V + p * C);
#pragma unroll
      for (int k = 0; k < C / 4; ++k) {
        float4 t = vw[k];
        t.x = fa(t.x, o[4 * k]);
        t.y = fa(t.y, o[4 * k + 1]);
        t.z = fa(t.z, o[4 * k + 2]);
        t.w = fa(t.w, o[4 * k + 3]);
        vw[k] = t;
      }
    }
    tc::fence_before();
    __syncthreads();  // A, S and O are reused by the next tile
  }
  if (warp == 0) tc::tmem_dealloc(tmem, tmem_cols<H>());
}

template <int H, int M>
void launch(float* V, const float* D, int64_t P, const float* wq, const float* wo,
            const float* gain, int zero, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attend_tc_kernel<H, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Smem<H>::BYTES);
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = int((P + TILE - 1) / TILE);
  const int cap = ctas_per_sm<H>() * sms;
  const int grid = tiles < cap ? tiles : cap;
  attend_tc_kernel<H, M><<<grid, NT, Smem<H>::BYTES, st>>>(V, D, P, wq, wo, gain, zero, tiles);
}

}  // namespace

bool attend_tc(float* V, const float* deltas, int64_t P, int C_, int M, int heads, const float* wq,
               const float* wo, const float* gain, int zero_scores, cudaStream_t st) {
  if (C_ != C) return false;
#define LVSG_ATT(HH, MM)                                                     \
  if (heads == HH && M == MM) {                                              \
    launch<HH, MM>(V, deltas, P, wq, wo, gain, zero_scores, st);             \
    return true;                                                             \
  }
  LVSG_ATT(1, 4) LVSG_ATT(2, 4) LVSG_ATT(4, 4)
  LVSG_ATT(1, 8) LVSG_ATT(2, 8) LVSG_ATT(4, 8)
  LVSG_ATT(1, 16) LVSG_ATT(2, 16) LVSG_ATT(4, 16)
#undef LVSG_ATT
  return false;
}

}  // namespace lvsg
