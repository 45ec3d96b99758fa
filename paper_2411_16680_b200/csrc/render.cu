// Stage 3 + Stage 4 fused: bilinear x s upsample of the LDM pre-activation
// maps, activation (Eq. 4 depth, sigmoid density, softmax blend over views),
// per-layer reprojection into every input view with the 4-tap f64 colour
// gather, beta renormalisation over valid views, and back-to-front
// over-compositing into the output frame. The activated 1080p LDM is never
// materialised.
//
// Reference semantics: upsample_activate (ldm.hpp:249-271), resize_bilinear
// (tape.hpp:858-917), render_target -> world_points + blended_layer_colors +
// over_composite (ldm.hpp:98-199, geometry.hpp:84-171).
#include <algorithm>
#include <cfloat>

#include "kernels.h"

namespace lvsg {
namespace {

constexpr int kMaxViews = 32;
#ifndef LVSG_RENDER_X2
#define LVSG_RENDER_X2 1
#endif

struct Taps {
  int y0, y1, x0, x1;
  float fy, fx;
};

__device__ __forceinline__ float sample(const float* map, int W, const Taps& t) {
  return lerp2(__ldg(map + t.y0 * W + t.x0), __ldg(map + t.y0 * W + t.x1),
               __ldg(map + t.y1 * W + t.x0), __ldg(map + t.y1 * W + t.x1), t.fx, t.fy);
}

// Activated LDM sample of layer l at output pixel: depth, sigma, beta[M].
// MM > 0: compile-time view count (every per-view array stays in registers);
// G: MM is only an upper bound of the runtime count a.M (views >= a.M are
// skipped, beta[m >= a.M] = 0).
template <int MM, bool G = false>
__device__ __forceinline__ void ldm_sample(const RenderArgs& a, int l, const Taps& t, float& depth,
                                           float& sigma, float* beta) {
  const int64_t plane = (int64_t)a.H * a.W;
  depth = activate_depth(sample(a.pre_d + l * plane, a.W, t), l, a.act);
  sigma = sigmoid_ref(sample(a.pre_s + l * plane, a.W, t));
  const int M = MM > 0 && !G ? MM : a.M;
  const float* lg = a.logits + l * plane * M;
  float mx = 0.f;
  if (G) {
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (m >= M) {
        beta[m] = 0.f;
        continue;
      }
      const float v = lerp2(__ldg(lg + ((int64_t)t.y0 * a.W + t.x0) * M + m),
                            __ldg(lg + ((int64_t)t.y0 * a.W + t.x1) * M + m),
                            __ldg(lg + ((int64_t)t.y1 * a.W + t.x0) * M + m),
                            __ldg(lg + ((int64_t)t.y1 * a.W + t.x1) * M + m), t.fx, t.fy);
      beta[m] = v;
      mx = m == 0 ? v : fmaxf(mx, v);
    }
    float sum = 0.f;
#pragma unroll
    for (int m = 0; m < MM; ++m)
      if (m < M) {
        beta[m] = expf(fsb(beta[m], mx));
        sum = fa(sum, beta[m]);
      }
    const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
    for (int m = 0; m < MM; ++m) beta[m] = fm(beta[m], inv);
    return;
  }
  if (MM > 0 && MM % 4 == 0) {  // each tap's M logits as float4 runs
    const float4* q00 = reinterpret_cast<const float4*>(lg + ((int64_t)t.y0 * a.W + t.x0) * M);
    const float4* q10 = reinterpret_cast<const float4*>(lg + ((int64_t)t.y0 * a.W + t.x1) * M);
    const float4* q01 = reinterpret_cast<const float4*>(lg + ((int64_t)t.y1 * a.W + t.x0) * M);
    const float4* q11 = reinterpret_cast<const float4*>(lg + ((int64_t)t.y1 * a.W + t.x1) * M);
#pragma unroll
    for (int g = 0; g < (MM > 0 ? MM : 4) / 4; ++g) {
      const float4 A = __ldg(q00 + g), B = __ldg(q10 + g), Cc = __ldg(q01 + g), D = __ldg(q11 + g);
      const float v[4] = {lerp2(A.x, B.x, Cc.x, D.x, t.fx, t.fy), lerp2(A.y, B.y, Cc.y, D.y, t.fx, t.fy),
                          lerp2(A.z, B.z, Cc.z, D.z, t.fx, t.fy), lerp2(A.w, B.w, Cc.w, D.w, t.fx, t.fy)};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        beta[4 * g + k] = v[k];
        mx = (g == 0 && k == 0) ? v[k] : fmaxf(mx, v[k]);
      }
    }
  } else {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const float v = lerp2(__ldg(lg + ((int64_t)t.y0 * a.W + t.x0) * M + m),
                            __ldg(lg + ((int64_t)t.y0 * a.W + t.x1) * M + m),
                            __ldg(lg + ((int64_t)t.y1 * a.W + t.x0) * M + m),
                            __ldg(lg + ((int64_t)t.y1 * a.W + t.x1) * M + m), t.fx, t.fy);
      beta[m] = v;
      mx = m == 0 ? v : fmaxf(mx, v);
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    beta[m] = expf(fsb(beta[m], mx));
    sum = fa(sum, beta[m]);
  }
  const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
  for (int m = 0; m < M; ++m) beta[m] = fm(beta[m], inv);
}

__device__ __forceinline__ Taps taps_for(const RenderArgs& a, int i, int j) {
  Taps t;
  resize_tap(i, a.H, a.Ho, t.y0, t.y1, t.fy);
  resize_tap(j, a.W, a.Wo, t.x0, t.x1, t.fx);
  return t;
}

// blended_layer_colors (ldm.hpp:158-189) for a compile-time view count:
// acc = sum_m beta_m mask_m c_m and wsum = sum_m beta_m mask_m (k ascending),
// with the cameras in the kernel's parameter space. The caller scales acc
// by 1/(wsum + 1e-8) once (the reference scales each beta first: ~1 ulp
// apart, floating-point work); no per-view colour stays live across the
// loop. EXACT = false takes each footprint from the fast path and returns
// the mask of views whose decisions it could not take (the caller then
// re-runs the layer with EXACT = true: the reference's operation order for
// every view). Taps and validity are the reference's either way; weights
// are f32 from the f64 fractions and the colour an f32 FMA chain (~2 ulp of
// the reference's f64 blend).
template <int MM, bool G, bool EXACT>
__device__ __forceinline__ unsigned blend_views(const RenderArgs& a, const FastCam* fc,
                                                const float pt[3], const float* beta, float acc[3],
                                                float& wsum) {
  unsigned need = 0;
  acc[0] = acc[1] = acc[2] = 0.f;
  wsum = 0.f;
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    if (G && m >= a.M) break;
    Footprint f;
    if (EXACT)
      f = project_footprint_nb(a.pc[m], pt);
    else if (!project_footprint_fast(fc[m], pt, f))
      need |= 1u << m;  // f: invalid, in-range taps
    LVSG_CHECK(f.x0 >= 0 && f.x1 < a.Wr && f.x0 <= f.x1 && f.y0 >= 0 && f.y1 < a.Hr &&
               f.y0 <= f.y1);
    const float fx = __double2float_rn(f.fx), fy = __double2float_rn(f.fy);
    const float gx = 1.0f - fx, gy = 1.0f - fy;
    const int r0 = f.y0 * a.Wr, r1 = f.y1 * a.Wr;  // one view < 2^31 floats
    const float bm = f.valid ? beta[m] : 0.f;
    const float* img = a.images + (int64_t)m * a.Hr * a.Wr * 3;
    const float* p00 = img + (r0 + f.x0) * 3;
    const float* p10 = img + (r0 + f.x1) * 3;
    const float* p01 = img + (r1 + f.x0) * 3;
    const float* p11 = img + (r1 + f.x1) * 3;
#if LVSG_RENDER_X2
    // red and green as packed f32x2 ops (sm_100 FMUL2 / FFMA2: the same
    // per-lane roundings as the scalar chain blue keeps; frames
    // bit-identical). The resize lerps stay scalar: ptxas contracts a packed
    // mul.rn.f32x2 feeding an add.rn.f32x2 into one FFMA2, which would change
    // their (uncontracted, tape.hpp:890-894) rounding
    const float2 wa = __fmul2_rn(make_float2(gx, fx), make_float2(gy, gy));  // w00, w10
    const float2 wb = __fmul2_rn(make_float2(gx, fx), make_float2(fy, fy));  // w01, w11
    float2 t = __fmul2_rn(make_float2(wa.x, wa.x), make_float2(__ldg(p00), __ldg(p00 + 1)));
    t = __ffma2_rn(make_float2(wa.y, wa.y), make_float2(__ldg(p10), __ldg(p10 + 1)), t);
    t = __ffma2_rn(make_float2(wb.x, wb.x), make_float2(__ldg(p01), __ldg(p01 + 1)), t);
    t = __ffma2_rn(make_float2(wb.y, wb.y), make_float2(__ldg(p11), __ldg(p11 + 1)), t);
    const float2 rg = __ffma2_rn(make_float2(bm, bm), t, make_float2(acc[0], acc[1]));
    acc[0] = rg.x, acc[1] = rg.y;
    acc[2] = fmaf(bm, fmaf(wb.y, __ldg(p11 + 2),
                           fmaf(wb.x, __ldg(p01 + 2), fmaf(wa.y, __ldg(p10 + 2), wa.x * __ldg(p00 + 2)))),
                  acc[2]);
#else
    const float w[4] = {gx * gy, fx * gy, gx * fy, fx * fy};
#pragma unroll
    for (int k = 0; k < 3; ++k)
      acc[k] = fmaf(bm, fmaf(w[3], __ldg(p11 + k),
                             fmaf(w[2], __ldg(p01 + k), fmaf(w[1], __ldg(p10 + k), w[0] * __ldg(p00 + k)))),
                    acc[k]);
#endif
    wsum = fa(wsum, bm);
  }
  return need;
}

// One thread per output pixel of the row band. MM > 0: the view count is a
// compile-time constant, the cameras are read from the kernel's parameter
// space (a.pc: constant-bank operands of the f64 instructions) and each
// view's footprint is branch-free (taps always in range; an invalid view's
// colour and weight are zeroed by select). MM == 0: cameras staged in shared
// memory, branchy footprint.
template <int MM, bool G = false>
__global__ void __launch_bounds__(128, MM >= 16 ? 4 : 8)
    render_fused_kernel(const __grid_constant__ RenderArgs a) {
  pdl_grid_sync();
  extern __shared__ DevCam s_cams[];
  if (MM == 0) {
    for (int m = threadIdx.x; m < a.M; m += blockDim.x) s_cams[m] = a.cams[m];
    __syncthreads();
  }
  const FastCam* fc = a.fc;  // (shared-memory copies measured slower: 818 vs 782 us)
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int rows = a.row1 - a.row0;
  if (idx >= (int64_t)rows * a.Wo) return;
  const int i = a.row0 + int(idx / a.Wo), j = int(idx % a.Wo);
  const Taps t = taps_for(a, i, j);
  const int M = MM > 0 ? MM : a.M;
  double dir[3];
  world_dir(a.rc, i, j, dir);
  float o[3] = {0.f, 0.f, 0.f};
  float beta[MM > 0 ? MM : kMaxViews];
  int bad = 0;
  const int64_t img_stride = (int64_t)a.Hr * a.Wr * 3;
  for (int l = 0; l < a.L; ++l) {
    float depth, sigma;
    ldm_sample<MM, G>(a, l, t, depth, sigma, beta);
    const double dv = double(depth);
    bad |= (dv < a.slack_lo || dv > a.slack_hi);
    float pt[3];
    world_point_dir(a.rc, dir, depth, pt);
    float rgb[3] = {0.f, 0.f, 0.f};
    if constexpr (MM > 0) {
      float acc[3], wsum;
      if (blend_views<MM, G, false>(a, fc, pt, beta, acc, wsum))
        blend_views<MM, G, true>(a, fc, pt, beta, acc, wsum);  // rare: a decision within 1e-7 px
      const float r = __fdiv_rn(1.0f, fa(wsum, 1e-8f));
#pragma unroll
      for (int k = 0; k < 3; ++k) rgb[k] = fm(acc[k], r);
    } else {
      // blended_layer_colors: beta * mask, wsum (k ascending from 0),
      // 1/(wsum+1e-8), then sum_m (beta_m r) c_m -- the reference's order
      float col[kMaxViews][3];
      float wsum = 0.f;
      for (int m = 0; m < M; ++m) {
        const float* img = a.images + m * img_stride;
        const Footprint f = project_footprint(s_cams[m], pt);
        if (f.valid) {
          double wd[4];
          bilinear_weights(f, wd);
          float w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) w[k] = __double2float_rn(wd[k]);
          const float* p00 = img + ((int64_t)f.y0 * a.Wr + f.x0) * 3;
          const float* p10 = img + ((int64_t)f.y0 * a.Wr + f.x1) * 3;
          const float* p01 = img + ((int64_t)f.y1 * a.Wr + f.x0) * 3;
          const float* p11 = img + ((int64_t)f.y1 * a.Wr + f.x1) * 3;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            col[m][k] = fmaf(w[3], __ldg(p11 + k),
                             fmaf(w[2], __ldg(p01 + k), fmaf(w[1], __ldg(p10 + k), w[0] * __ldg(p00 + k))));
          beta[m] = fm(beta[m], 1.0f);
        } else {
          col[m][0] = col[m][1] = col[m][2] = 0.f;
          beta[m] = fm(beta[m], 0.0f);
        }
        wsum = fa(wsum, fm(beta[m], 1.0f));
      }
      const float r = __fdiv_rn(1.0f, fa(wsum, 1e-8f));
      for (int m = 0; m < M; ++m) {
        const float b = fm(beta[m], r);
#pragma unroll
        for (int k = 0; k < 3; ++k) rgb[k] = fa(rgb[k], fm(b, col[m][k]));
      }
    }
    // over_composite: o = v*a + (1-a)*o, layer 0 (far) first
#pragma unroll
    for (int k = 0; k < 3; ++k) o[k] = fa(fm(rgb[k], sigma), fm(fsb(1.0f, sigma), o[k]));
  }
  if (bad && a.bad_depth) atomicOr(a.bad_depth, 1);
  float* out = a.rgb + idx * 3;
  out[0] = o[0];
  out[1] = o[1];
  out[2] = o[2];
}

__global__ void upsample_activate_kernel(const RenderArgs a, float* depth, float* density,
                                         float* blend) {
  pdl_grid_sync();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t plane = (int64_t)a.Ho * a.Wo;
  if (idx >= plane * a.L) return;
  const int l = int(idx / plane);
  const int64_t pix = idx % plane;
  const int i = int(pix / a.Wo), j = int(pix % a.Wo);
  const Taps t = taps_for(a, i, j);
  float beta[kMaxViews];
  float d, s;
  ldm_sample<0>(a, l, t, d, s, beta);
  depth[idx] = d;
  density[idx] = s;
  for (int m = 0; m < a.M; ++m) blend[idx * a.M + m] = beta[m];
}

// ForwardResult.rgb under direct_rgb (network.hpp:596-601): the appearance
// head pre_a = V w_appear [L,H,W,3] resized bilinearly to the output grid
// (the same taps and f32 lerps as the LDM maps), sigmoid, over-composited
// back to front with the activated density sigmoid(resize(pre_s)). One
// thread per output pixel.
__global__ void direct_rgb_kernel(const RenderArgs a, const float* __restrict__ pre_a,
                                  float* __restrict__ out) {
  pdl_grid_sync();
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)a.Ho * a.Wo) return;
  const int i = int(idx / a.Wo), j = int(idx % a.Wo);
  const Taps t = taps_for(a, i, j);
  const int64_t plane = (int64_t)a.H * a.W;
  const int64_t q00 = (int64_t)t.y0 * a.W + t.x0, q10 = (int64_t)t.y0 * a.W + t.x1;
  const int64_t q01 = (int64_t)t.y1 * a.W + t.x0, q11 = (int64_t)t.y1 * a.W + t.x1;
  float o[3] = {0.f, 0.f, 0.f};
  for (int l = 0; l < a.L; ++l) {
    const float s = sigmoid_ref(sample(a.pre_s + l * plane, a.W, t));
    const float* pa = pre_a + l * plane * 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float x = lerp2(__ldg(pa + q00 * 3 + k), __ldg(pa + q10 * 3 + k), __ldg(pa + q01 * 3 + k),
                            __ldg(pa + q11 * 3 + k), t.fx, t.fy);
      const float v = sigmoid_ref(x);
      o[k] = fa(fm(v, s), fm(fsb(1.0f, s), o[k]));
    }
  }
  out[idx * 3 + 0] = o[0];
  out[idx * 3 + 1] = o[1];
  out[idx * 3 + 2] = o[2];
}

inline int blocks_for(int64_t n, int t) { return int((n + t - 1) / t); }

}  // namespace

FastCam fast_cam(const DevCam& d) {
  FastCam c;
  for (int j = 0; j < 3; ++j) {
    c.A[0 * 3 + j] = d.fx * d.R[0 * 3 + j] + d.cx * d.R[2 * 3 + j];
    c.A[1 * 3 + j] = d.fy * d.R[1 * 3 + j] + d.cy * d.R[2 * 3 + j];
    c.A[2 * 3 + j] = d.R[2 * 3 + j];
  }
  c.b[0] = d.fx * d.t[0] + d.cx * d.t[2];
  c.b[1] = d.fy * d.t[1] + d.cy * d.t[2];
  c.b[2] = d.t[2];
  c.wm = d.wm;
  c.hm = d.hm;
  c.hu = d.hu;
  c.hv = d.hv;
  c.W = d.W;
  c.H = d.H;
  // f32 decision bounds (kDecisionEpsF): the f32 roundings of the f64
  // bounds, moved by the band. Views wider or taller than 8192 px: nothing
  // is clearly inside or outside, every decision takes the exact path.
  const double lo = 0.5 - 1e-4, e = double(kDecisionEpsF);
  if (d.W > 8192 || d.H > 8192) {
    c.in_lo = FLT_MAX;
    c.in_u = c.in_v = -FLT_MAX;
    c.out_lo = -FLT_MAX;
    c.out_u = c.out_v = FLT_MAX;
    return c;
  }
  c.in_lo = float(lo + e);
  c.in_u = float(d.hu - e);
  c.in_v = float(d.hv - e);
  c.out_lo = float(lo - e);
  c.out_u = float(d.hu + e);
  c.out_v = float(d.hv + e);
  return c;
}

void render_fused(const RenderArgs& a, cudaStream_t st) {
  const int64_t n = (int64_t)(a.row1 - a.row0) * a.Wo;
  const int g = blocks_for(n, 128);
  // exact view-count kernels for M in {4, 8, 16}; other M <= 32 run the
  // next larger one with a runtime bound; all of them take the cameras by
  // value (pc); without them (pc_valid = 0) the generic kernel
  const bool pc = a.pc_valid && a.M >= 1 && a.M <= kRenderParamViews;
  const int mm = !pc ? 0 : (a.M == 4 || a.M == 8 || a.M == 16) ? a.M : -a.M;
  const size_t sm = mm ? 0 : a.M * sizeof(DevCam);  // <0> stages the cameras in smem
  switch (mm) {
    case 4: launch_k(render_fused_kernel<4>, g, 128, sm, st, a); break;
    case 8: launch_k(render_fused_kernel<8>, g, 128, sm, st, a); break;
    case 16: launch_k(render_fused_kernel<16>, g, 128, sm, st, a); break;
    case 0: launch_k(render_fused_kernel<0>, g, 128, sm, st, a); break;
    default:
      if (a.M < 8)
        launch_k(render_fused_kernel<8, true>, g, 128, sm, st, a);
      else if (a.M < 16)
        launch_k(render_fused_kernel<16, true>, g, 128, sm, st, a);
      else
        launch_k(render_fused_kernel<32, true>, g, 128, sm, st, a);
  }
}

void upsample_activate(const RenderArgs& a, float* depth, float* density, float* blend,
                       cudaStream_t st) {
  const int64_t n = (int64_t)a.L * a.Ho * a.Wo;
  launch_k(upsample_activate_kernel, blocks_for(n, 128), 128, 0, st, a, depth, density, blend);
}

void direct_rgb(const RenderArgs& a, const float* pre_a, float* out, cudaStream_t st) {
  const int64_t n = (int64_t)a.Ho * a.Wo;
  launch_k(direct_rgb_kernel, blocks_for(n, 128), 128, 0, st, a, pre_a, out);
}

}  // namespace lvsg
