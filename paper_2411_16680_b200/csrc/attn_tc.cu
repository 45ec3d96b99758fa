// Stage 2 (One-to-many attention, attention.hpp:207-252) fused on the
// sm_100a tensor core, C = 32, h <= 4 heads, M views:
//
//   n      = rms_norm(V) * g                     (SIMT, thread = texel)
//   S      = n [Wq_0 | ... | Wq_{h-1}]           tcgen05.mma kind::tf32, 3xTF32,
//                                                M=128 texels, N=32h, TMEM
//   l_im   = <S_i, Δ_m> / sqrt(C); w = softmax_m; head_i = sum_m w_im Δ_m
//   O      = sum_i head_i Wo_i                   tcgen05.mma, 3xTF32, TMEM
//   V     += O
//
// Persistent warp-specialised CTA, one per SM, 128-texel tiles:
//   w0     TMA producer: the V tile (128B-swizzled, 2 buffers) and, per view,
//          the tile's Δ slice [8 channel groups][128 texels][16 B] (8 bulk
//          copies of 2 KB from the view-major SoA Δ[m][g][p][4]) into an NS-deep ring --
//          twice per tile (scores, then mix; the second read hits L2)
//   w1     MMA issuer (one elected lane; warp-uniform descriptors)
//   w2-5   consumers, thread <-> texel row <-> TMEM lane: rms-norm, stage n,
//          S for every head held in registers through the score pass, softmax,
//          one mix pass for all heads, stage each head for O (two A buffers),
//          V + O back through the swizzled tile and one TMA store
// Weights are split into tf32 hi/lo once per CTA and stay resident in the
// K-major interleave layout.
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
constexpr int NT = 192;                    // 6 warps
constexpr int NCONS = 128;                 // consumer threads
constexpr int NCH = C / 4;                 // 16-byte K chunks
constexpr int A_LBO = TILE * 16;           // 2048
constexpr int A_PLANE = NCH * A_LBO;       // 16 KB per tf32 plane
constexpr int A_BYTES = 2 * A_PLANE;       // hi + lo
constexpr int V_BYTES = TILE * C * 4;      // 16 KB
constexpr int D_BYTES = NCH * TILE * 16;   // one view slice, 16 KB

template <int H>
constexpr uint32_t tmem_cols() {  // S (32h columns) + O (32 columns), power of two
  return H == 1 ? 64u : H == 2 ? 128u : 256u;
}

template <int H>
struct Smem {
  static constexpr int BQ_LBO = 32 * H * 16;
  static constexpr int BQ_BYTES = NCH * BQ_LBO;  // one plane
  static constexpr int BO_LBO = 32 * 16;
  static constexpr int BO_BYTES = NCH * BO_LBO;  // one head, one plane
  static constexpr int OFF_V = 0;                // 2 buffers, 1 KB aligned (swizzle)
  static constexpr int OFF_A = OFF_V + 2 * V_BYTES;
  static constexpr int OFF_BQH = OFF_A + 2 * A_BYTES;
  static constexpr int OFF_BQL = OFF_BQH + BQ_BYTES;
  static constexpr int OFF_BO = OFF_BQL + BQ_BYTES;  // [head][hi|lo]
  static constexpr int OFF_D = OFF_BO + 2 * H * BO_BYTES;
  static constexpr int BUDGET = 227 * 1024 - 512;
  static constexpr int NS = (BUDGET - OFF_D) / D_BYTES > 8 ? 8 : (BUDGET - OFF_D) / D_BYTES;
  static constexpr int OFF_BAR = OFF_D + NS * D_BYTES;
  // bars: v_full[2] v_empty[2] d_full[NS] d_empty[NS] a_full[2] a_free[2] s_done o_done
  static constexpr int NBAR = 4 + 2 * NS + 4 + 2;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16;
  static_assert(NS >= 2, "shared memory budget");
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
__device__ __forceinline__ void stage_row(uint8_t* a, int row, const float* x) {
  float* hi = reinterpret_cast<float*>(a);
  float* lo = reinterpret_cast<float*>(a + A_PLANE);
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

template <int H, int M>
__global__ void __launch_bounds__(NT, 1)
    attend_tc_kernel(const __grid_constant__ CUtensorMap vmap, const float* __restrict__ D, int64_t P,
                     const float* __restrict__ wq, const float* __restrict__ wo,
                     const float* __restrict__ gain, int zero_scores, int num_tiles) {
  using S = Smem<H>;
  constexpr int NS = S::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint64_t* v_full = bars;            // [2] V tile landed
  uint64_t* v_empty = bars + 2;       // [2] V tile stored back (buffer free)
  uint64_t* d_full = bars + 4;        // [NS] Δ slice landed
  uint64_t* d_empty = d_full + NS;    // [NS] consumers done with the slice
  uint64_t* a_full = d_empty + NS;    // [2] A operand staged
  uint64_t* a_free = a_full + 2;      // [2] MMAs done reading A
  uint64_t* s_done = a_free + 2;      // S ready
  uint64_t* o_done = s_done + 1;      // O ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::NBAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x >= num_tiles) return;
  const uint32_t sb = tc::smem_u32(smem);
  if (tid == 0 && (sb & 1023u)) __trap();  // swizzle atoms need 1 KB alignment
  const int passes = zero_scores ? 1 : 2;

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
    for (int k = 0; k < 2; ++k) {
      tc::mbar_init(&v_full[k], 1);
      tc::mbar_init(&v_empty[k], 1);
      tc::mbar_init(&a_full[k], NCONS);
      tc::mbar_init(&a_free[k], 1);
    }
    for (int k = 0; k < NS; ++k) {
      tc::mbar_init(&d_full[k], 1);
      tc::mbar_init(&d_empty[k], NCONS);
    }
    tc::mbar_init(s_done, 1);
    tc::mbar_init(o_done, 1);
    tc::mbar_init_fence();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, tmem_cols<H>());
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const uint32_t tmem_s = tmem, tmem_o = tmem + 32 * H;

  if (warp == 0) {
    // ---- producer ----
    if (lane == 0) {
      int k = 0, i = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++i) {
        const int vb = i & 1;
        if (i >= 2) tc::mbar_wait(&v_empty[vb], uint32_t(((i >> 1) - 1) & 1));
        tc::mbar_expect_tx(&v_full[vb], V_BYTES);
        tma_load_2d(sb + S::OFF_V + vb * V_BYTES, &vmap, 0, tile * TILE, &v_full[vb]);
        // Δ[m][g][p0 .. p0+n) is 8 contiguous runs of n*16 bytes: plain bulk copies
        const int64_t p0 = int64_t(tile) * TILE;
        const uint32_t run = uint32_t((P - p0 < TILE ? P - p0 : TILE) * 16);
        for (int pass = 0; pass < passes; ++pass)
          for (int m = 0; m < M; ++m, ++k) {
            const int sl = k % NS;
            if (k >= NS) tc::mbar_wait(&d_empty[sl], uint32_t((k / NS - 1) & 1));
            tc::mbar_expect_tx(&d_full[sl], run * NCH);
            for (int g = 0; g < NCH; ++g)
              tc::bulk_load(sb + S::OFF_D + sl * D_BYTES + g * TILE * 16,
                            D + ((int64_t(m) * NCH + g) * P + p0) * 4, run, &d_full[sl]);
          }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: per tile S (from A staging u), then O over the heads ----
    const uint64_t bqh = tc::smem_desc(sb + S::OFF_BQH, S::BQ_LBO, 128);
    const uint64_t bql = tc::smem_desc(sb + S::OFF_BQL, S::BQ_LBO, 128);
    constexpr uint32_t id_s = tc::idesc_tf32(128, 32 * H);
    constexpr uint32_t id_o = tc::idesc_tf32(128, 32);
    int u = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      for (int st = 0; st <= H; ++st, ++u) {
        const int b = u & 1;
        tc::mbar_wait(&a_full[b], uint32_t((u >> 1) & 1));
        tc::fence_after();
        const uint32_t ab = sb + S::OFF_A + b * A_BYTES;
        const uint64_t ahi = tc::smem_desc(ab, A_LBO, 128);
        const uint64_t alo = tc::smem_desc(ab + A_PLANE, A_LBO, 128);
        if (tc::elect_one()) {
          if (st == 0) {
            mma3(tmem_s, ahi, alo, bqh, bql, S::BQ_LBO, id_s, false);
            tc::commit(s_done);
          } else {
            const int hh = st - 1;
            const uint64_t boh =
                tc::smem_desc(sb + S::OFF_BO + (2 * hh) * S::BO_BYTES, S::BO_LBO, 128);
            const uint64_t bol =
                tc::smem_desc(sb + S::OFF_BO + (2 * hh + 1) * S::BO_BYTES, S::BO_LBO, 128);
            mma3(tmem_o, ahi, alo, boh, bol, S::BO_LBO, id_o, hh > 0);
            if (hh == H - 1) tc::commit(o_done);
          }
          tc::commit(&a_free[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- consumers ----
    const int q = warp & 3;
    const int row = q * 32 + lane;  // texel row of the tile == TMEM lane
    const uint32_t lane_base = uint32_t(q * 32) << 16;
    const float inv_temp = __double2float_rn(1.0 / sqrt(double(C)));
    float g32[C];
#pragma unroll
    for (int c = 0; c < C; ++c) g32[c] = __ldg(gain + c);
    int k = 0, u = 0, i = 0;
    auto stage = [&](const float* x) {  // A staging u (buffer u & 1)
      const int b = u & 1;
      if (u >= 2) tc::mbar_wait(&a_free[b], uint32_t(((u >> 1) - 1) & 1));
      stage_row(smem + S::OFF_A + b * A_BYTES, row, x);
      tc::fence_proxy_async();
      tc::mbar_arrive(&a_full[b]);
      ++u;
    };
    auto slice_row = [&](float* dm) {  // this texel's row of the next Δ slice
      const int sl = k % NS;
      tc::mbar_wait(&d_full[sl], uint32_t((k / NS) & 1));
      const uint8_t* d = smem + S::OFF_D + sl * D_BYTES + row * 16;
#pragma unroll
      for (int g = 0; g < NCH; ++g) {
        const float4 t = *reinterpret_cast<const float4*>(d + g * TILE * 16);
        dm[4 * g] = t.x, dm[4 * g + 1] = t.y, dm[4 * g + 2] = t.z, dm[4 * g + 3] = t.w;
      }
      tc::mbar_arrive(&d_empty[sl]);
      ++k;
    };
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++i) {
      const int vb = i & 1;
      uint8_t* vt = smem + S::OFF_V + vb * V_BYTES;
      // ---- n = rms_norm(V) * g -> A ----
      tc::mbar_wait(&v_full[vb], uint32_t((i >> 1) & 1));
      {
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
        for (int c = 0; c < C; ++c) x[c] = fm(fm(x[c], r), g32[c]);
        stage(x);
      }
      // ---- scores: S held in registers, one pass over Δ ----
      float w[H][M];
      if (zero_scores) {
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int m = 0; m < M; ++m) w[h][m] = __fdiv_rn(1.0f, float(M));
      } else {
        float sv[H][C];
        tc::mbar_wait(s_done, uint32_t(i & 1));
        tc::fence_after();
#pragma unroll
        for (int h = 0; h < H; ++h) tc::tmem_ld32(tmem_s + lane_base + uint32_t(32 * h), sv[h]);
        tc::fence_before();
#pragma unroll
        for (int m = 0; m < M; ++m) {
          float dm[C];
          slice_row(dm);
#pragma unroll
          for (int h = 0; h < H; ++h) {
            float acc = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) acc = fmaf(sv[h][c], dm[c], acc);
            w[h][m] = fm(acc, inv_temp);
          }
        }
        // softmax over views (tape.hpp:390-404: max, exp(x - max), sum, * 1/sum)
#pragma unroll
        for (int h = 0; h < H; ++h) {
          float mx = w[h][0];
#pragma unroll
          for (int m = 1; m < M; ++m) mx = fmaxf(mx, w[h][m]);
          float sum = 0.f;
#pragma unroll
          for (int m = 0; m < M; ++m) {
            w[h][m] = expf(fsb(w[h][m], mx));
            sum = fa(sum, w[h][m]);
          }
          const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
          for (int m = 0; m < M; ++m) w[h][m] = fm(w[h][m], inv);
        }
      }
      // ---- mix: every head in one pass over Δ ----
      float hd[H][C];
#pragma unroll
      for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < C; ++c) hd[h][c] = 0.f;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        float dm[C];
        slice_row(dm);
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int c = 0; c < C; ++c) hd[h][c] = fmaf(w[h][m], dm[c], hd[h][c]);
      }
      // ---- O = sum_i head_i Wo_i ----
#pragma unroll
      for (int h = 0; h < H; ++h) stage(hd[h]);
      tc::mbar_wait(o_done, uint32_t(i & 1));
      tc::fence_after();
      float o[C];
      tc::tmem_ld32(tmem_o + lane_base, o);
      tc::fence_before();
      // ---- V += O, back through the swizzled tile and one TMA store ----
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
      if (warp == 2 && lane == 0) {
        tma_store_2d(&vmap, sb + S::OFF_V + vb * V_BYTES, 0, tile * TILE);
        tc::bulk_commit();
        tc::bulk_wait_read<0>();
        tc::mbar_arrive(&v_empty[vb]);
      }
    }
    if (warp == 2 && lane == 0) tc::bulk_wait<0>();
  }
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
  // V [P][32] fp32 as a 2-D map, 128-texel boxes (128B swizzle)
  CUtensorMap vmap;
  std::memset(&vmap, 0, sizeof(vmap));
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
  const int tiles = int((P + TILE - 1) / TILE);
  const int grid = tiles < sms ? tiles : sms;
  attend_tc_kernel<H, M><<<grid, NT, Smem<H>::BYTES, st>>>(vmap, D, P, wq, wo, gain, zero, tiles);
}

}  // namespace

bool attend_tc(float* V, const float* deltas, int64_t P, int C_, int M, int heads, const float* wq,
               const float* wo, const float* gain, int zero_scores, cudaStream_t st) {
  if (C_ != C || !encode_fn() || (reinterpret_cast<uintptr_t>(V) & 15) ||
      (reinterpret_cast<uintptr_t>(deltas) & 15) || P >= (int64_t(1) << 31))
    return false;
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
