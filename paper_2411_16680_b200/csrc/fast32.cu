// C = 32 specialisations of the per-texel MLP kernels (the production
// channel count): every per-texel vector lives in registers (float4 loads),
// weights are shared-memory broadcasts. Same arithmetic order as the generic
// kernels in kernels.cu.
#include "kernels.h"

namespace lvsg {
namespace {

constexpr int C = 32;

__device__ __forceinline__ void load_row(const float* p, float* v) {
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int k = 0; k < C / 4; ++k) {
    const float4 t = __ldg(q + k);
    v[4 * k] = t.x, v[4 * k + 1] = t.y, v[4 * k + 2] = t.z, v[4 * k + 3] = t.w;
  }
}

// layer_collapse (network.hpp:440-455), one thread per output texel.
__global__ void __launch_bounds__(128) layer_collapse32_kernel(
    const float* __restrict__ V, int L2, int64_t PL, const float* __restrict__ w1,
    const float* __restrict__ b1, const float* __restrict__ w2, const float* __restrict__ b2,
    float* __restrict__ out) {
  pdl_grid_sync();
  __shared__ __align__(16) float s_w1[2 * C * 2 * C];
  __shared__ __align__(16) float s_w2[2 * C * C];
  for (int e = threadIdx.x; e < 4 * C * C; e += blockDim.x) s_w1[e] = w1[e];
  for (int e = threadIdx.x; e < 2 * C * C; e += blockDim.x) s_w2[e] = w2[e];
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)L2 * PL) return;
  const int64_t l = t / PL, q = t % PL;
  float a[C], b[C], r[C];
  load_row(V + ((2 * l) * PL + q) * C, a);
  load_row(V + ((2 * l + 1) * PL + q) * C, b);
#pragma unroll
  for (int c = 0; c < C; ++c) r[c] = 0.f;
#pragma unroll 1
  for (int j0 = 0; j0 < 2 * C; j0 += 8) {
    float hc[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) hc[jj] = 0.f;
    // h[j] = sum_k cat[k] w1[k][j], k ascending over [a ; b]
#pragma unroll
    for (int k = 0; k < 2 * C; ++k) {
      const float xk = k < C ? a[k] : b[k - C];
      const float4 wa = *reinterpret_cast<const float4*>(s_w1 + k * 2 * C + j0);
      const float4 wb = *reinterpret_cast<const float4*>(s_w1 + k * 2 * C + j0 + 4);
      hc[0] = fmaf(xk, wa.x, hc[0]);
      hc[1] = fmaf(xk, wa.y, hc[1]);
      hc[2] = fmaf(xk, wa.z, hc[2]);
      hc[3] = fmaf(xk, wa.w, hc[3]);
      hc[4] = fmaf(xk, wb.x, hc[4]);
      hc[5] = fmaf(xk, wb.y, hc[5]);
      hc[6] = fmaf(xk, wb.z, hc[6]);
      hc[7] = fmaf(xk, wb.w, hc[7]);
    }
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const float hv = gelu_ref(fa(hc[jj], __ldg(b1 + j0 + jj)));
      const float4* wr = reinterpret_cast<const float4*>(s_w2 + (j0 + jj) * C);
#pragma unroll
      for (int c4 = 0; c4 < C / 4; ++c4) {
        const float4 w = wr[c4];
        r[4 * c4] = fmaf(hv, w.x, r[4 * c4]);
        r[4 * c4 + 1] = fmaf(hv, w.y, r[4 * c4 + 1]);
        r[4 * c4 + 2] = fmaf(hv, w.z, r[4 * c4 + 2]);
        r[4 * c4 + 3] = fmaf(hv, w.w, r[4 * c4 + 3]);
      }
    }
  }
  float4* o = reinterpret_cast<float4*>(out + t * C);
#pragma unroll
  for (int c4 = 0; c4 < C / 4; ++c4) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * c4 + k;
      v[k] = fa(fm(fa(a[c], b[c]), 0.5f), fa(r[c], __ldg(b2 + c)));
    }
    o[c4] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// blend_w [32][32] by value (parameter space): the q = n W_blend products
// take their weights as constant-bank / uniform-register operands.
struct BlendParam {
  float w[C * C];
};

// decode_blend_logits (network.hpp:539-549) for C = 32, M views.
template <int M, bool PW>
__global__ void __launch_bounds__(128) blend_logits32_kernel(const float* __restrict__ V,
                                                             const float* __restrict__ D, int64_t P,
                                                             const float* __restrict__ bw,
                                                             const float* __restrict__ gain,
                                                             float* __restrict__ logits,
                                                             const __grid_constant__ BlendParam pw) {
  pdl_grid_sync();
  __shared__ __align__(16) float s_bw[PW ? 4 : C * C];
  if (!PW) {
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) s_bw[e] = bw[e];
    __syncthreads();
  }
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  float n[C], q[C];
  load_row(V + p * C, n);
  float ms = 0.f;
#pragma unroll
  for (int k = 0; k < C; ++k) ms = fmaf(n[k], n[k], ms);
  const float r = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(ms, float(C)), 1e-6f)));
#pragma unroll
  for (int k = 0; k < C; ++k) n[k] = fm(fm(n[k], r), __ldg(gain + k));
  // q = n W_blend as packed f32x2 FMAs over output-channel pairs (FFMA2,
  // the same per-lane roundings)
  float2 q2[C / 2];
#pragma unroll
  for (int c = 0; c < C / 2; ++c) q2[c] = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const float2 nk = make_float2(n[k], n[k]);
#pragma unroll
    for (int c4 = 0; c4 < C / 4; ++c4) {
      const float4 w = PW ? make_float4(pw.w[k * C + 4 * c4], pw.w[k * C + 4 * c4 + 1],
                                        pw.w[k * C + 4 * c4 + 2], pw.w[k * C + 4 * c4 + 3])
                          : reinterpret_cast<const float4*>(s_bw + k * C)[c4];
      q2[2 * c4] = __ffma2_rn(nk, make_float2(w.x, w.y), q2[2 * c4]);
      q2[2 * c4 + 1] = __ffma2_rn(nk, make_float2(w.z, w.w), q2[2 * c4 + 1]);
    }
  }
#pragma unroll
  for (int c = 0; c < C / 2; ++c) q[2 * c] = q2[c].x, q[2 * c + 1] = q2[c].y;
  const float inv_temp = __double2float_rn(1.0 / sqrt(double(C)));
  float out[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const float* dm = D + ((int64_t)m * P + p) * C;  // Δ[m][p][32]: one 128-byte row
    float acc = 0.f;
#pragma unroll
    for (int c8 = 0; c8 < C / 8; ++c8) {
      float t[8];
      ldg256(dm + 8 * c8, t);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = fmaf(q[8 * c8 + k], t[k], acc);
    }
    out[m] = fm(acc, inv_temp);
  }
#pragma unroll
  for (int m = 0; m < M; ++m) logits[p * M + m] = out[m];
}

// render_to_input_view decode for C = Ca = 32: payload [a(32), sigma],
// activated depth and the world point, one thread per texel.
// The three heads by value: [k][36] = appear(32) | sigma | depth | 0 0.
struct DecodeParam {
  float w[C * (C + 4)];
};

// PW: weights from `pw` (constant-bank FMA operands), else staged in shared
// memory; 32-bit texel indexing (the caller checks P < 2^31).
template <bool PW>
__global__ void __launch_bounds__(128) decode_payload32_kernel(
    const float* __restrict__ V, int L, int H, int W, const float* __restrict__ w_appear,
    const float* __restrict__ w_sigma, const float* __restrict__ w_depth, DepthAct act,
    DevRayCam rc, float* __restrict__ payload, float* __restrict__ depth,
    float* __restrict__ points, const __grid_constant__ DecodeParam pw) {
  pdl_grid_sync();
  constexpr int KW = C + 4;  // appear | sigma | depth | pad (16-byte rows)
  __shared__ __align__(16) float s_w[PW ? 4 : C * KW];
  if (!PW) {
    for (int e = threadIdx.x; e < C * KW; e += blockDim.x) {
      const int k = e / KW, c = e % KW;
      s_w[e] = c < C ? w_appear[k * C + c] : (c == C ? w_sigma[k] : (c == C + 1 ? w_depth[k] : 0.f));
    }
    __syncthreads();
  }
  const int P = L * H * W;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  float v[C], acc[KW];
  load_row(V + p * C, v);
  // packed f32x2 FMAs over output-channel pairs (sm_100 FFMA2: the same
  // per-lane roundings as fmaf), the input channel broadcast
  float2 acc2[KW / 2];
#pragma unroll
  for (int c = 0; c < KW / 2; ++c) acc2[c] = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const float2 vk = make_float2(v[k], v[k]);
#pragma unroll
    for (int c4 = 0; c4 < KW / 4; ++c4) {
      const float4 w = PW ? make_float4(pw.w[k * KW + 4 * c4], pw.w[k * KW + 4 * c4 + 1],
                                        pw.w[k * KW + 4 * c4 + 2], pw.w[k * KW + 4 * c4 + 3])
                          : reinterpret_cast<const float4*>(s_w + k * KW)[c4];
      acc2[2 * c4] = __ffma2_rn(vk, make_float2(w.x, w.y), acc2[2 * c4]);
      acc2[2 * c4 + 1] = __ffma2_rn(vk, make_float2(w.z, w.w), acc2[2 * c4 + 1]);
    }
  }
#pragma unroll
  for (int c = 0; c < KW / 2; ++c) acc[2 * c] = acc2[c].x, acc[2 * c + 1] = acc2[c].y;
  // payload row padded to 40 floats (32-byte rows): [a(32), sigma, 0 x 7]
  float4* pay = reinterpret_cast<float4*>(payload + (int64_t)p * (C + 8));
#pragma unroll
  for (int c4 = 0; c4 < C / 4; ++c4)
    pay[c4] = make_float4(sigmoid_ref(acc[4 * c4]), sigmoid_ref(acc[4 * c4 + 1]),
                          sigmoid_ref(acc[4 * c4 + 2]), sigmoid_ref(acc[4 * c4 + 3]));
  pay[C / 4] = make_float4(sigmoid_ref(acc[C]), 0.f, 0.f, 0.f);
  pay[C / 4 + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int q = p / W, j = p - q * W;
  const int l = q / H, i = q - l * H;
  const float d = activate_depth(acc[C + 1], l, act);
  depth[p] = d;
  float pt[3];
  world_point(rc, i, j, d, pt);
  points[(int64_t)p * 3 + 0] = pt[0];
  points[(int64_t)p * 3 + 1] = pt[1];
  points[(int64_t)p * 3 + 2] = pt[2];
}

inline int blocks_for(int64_t n, int t) { return int((n + t - 1) / t); }

}  // namespace

bool layer_collapse32(const float* V, int L, int64_t PL, int C_, const float* w1, const float* b1,
                      const float* w2, const float* b2, float* out, cudaStream_t st) {
  if (C_ != C) return false;
  const int L2 = L / 2;
  launch_k(layer_collapse32_kernel, blocks_for(L2 * PL, 128), 128, 0, st, V, L2, PL, w1, b1, w2, b2, out);
  return true;
}

bool blend_logits32(const float* V, const float* deltas, int64_t P, int C_, int M,
                    const float* blend_w, const float* gain, float* logits, cudaStream_t st,
                    const float* blend_w_host) {
  if (C_ != C) return false;
  const int g = blocks_for(P, 128);
  BlendParam pw;
  if (blend_w_host)
    for (int e = 0; e < C * C; ++e) pw.w[e] = blend_w_host[e];
  const bool h = blend_w_host != nullptr;
#define LVSG_BL(MM)                                                                             \
  if (h)                                                                                         \
    launch_k(blend_logits32_kernel<MM, true>, g, 128, 0, st, V, deltas, P, blend_w, gain, logits, pw); \
  else                                                                                           \
    launch_k(blend_logits32_kernel<MM, false>, g, 128, 0, st, V, deltas, P, blend_w, gain, logits, pw);
  switch (M) {
    case 2: LVSG_BL(2) return true;
    case 4: LVSG_BL(4) return true;
    case 8: LVSG_BL(8) return true;
    case 16: LVSG_BL(16) return true;
    default: return false;
  }
#undef LVSG_BL
}

bool decode_payload32(const float* V, int L, int H, int W, int C_, const float* w_appear, int Ca,
                      const float* w_sigma, const float* w_depth, const DepthAct& act,
                      const DevRayCam& rc, float* payload, float* depth, float* points,
                      cudaStream_t st, const float* w_host) {
  const int64_t P = (int64_t)L * H * W;
  if (C_ != C || Ca != C || P * (C + 4) >= (int64_t(1) << 31)) return false;
  DecodeParam pw;
  if (w_host) {
    for (int e = 0; e < C * (C + 4); ++e) pw.w[e] = w_host[e];
    launch_k(decode_payload32_kernel<true>, blocks_for(P, 128), 128, 0, st, V, L, H, W, w_appear,
             w_sigma, w_depth, act, rc, payload, depth, points, pw);
  } else {
    launch_k(decode_payload32_kernel<false>, blocks_for(P, 128), 128, 0, st, V, L, H, W, w_appear,
             w_sigma, w_depth, act, rc, payload, depth, points, pw);
  }
  return true;
}

}  // namespace lvsg
