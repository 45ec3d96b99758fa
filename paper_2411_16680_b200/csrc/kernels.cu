// Memory-bound lvsg kernels: layout/elementwise, ray encodings, the Stage-1
// reprojection gather, the render-to-input-view splat, and the per-texel
// One-to-many attention / blend-logit / layer-collapse MLPs.
#include <cfloat>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <string>

#include "host.h"
#include "kernels.h"

namespace lvsg {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("LVSG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool pdl_all() {
  static const bool on = [] {
    const char* e = getenv("LVSG_PDL");
    return e && e[0] == '2';
  }();
  return on;
}

namespace {
std::mutex g_dev_mu;
std::set<std::pair<int, const void*>> g_optin;  // (device, kernel) opted in
std::map<int, int> g_sms;
int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) throw CudaError("cudaGetDevice failed");
  return d;
}
}  // namespace

void smem_optin(const void* kernel, int bytes) {
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_optin.insert({d, kernel}).second) return;
  const cudaError_t e =
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    g_optin.erase({d, kernel});
    throw CudaError(std::string("cudaFuncSetAttribute(MaxDynamicSharedMemorySize): ") +
                    cudaGetErrorString(e));
  }
}

int sm_count() {
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_sms.find(d);
  if (it != g_sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n < 1)
    throw CudaError("cudaDeviceGetAttribute(MultiProcessorCount) failed");
  g_sms[d] = n;
  return n;
}

namespace {

constexpr int kMaxM = 32;  // views handled per texel in registers

inline int blocks_for(int64_t n, int t) { return int((n + t - 1) / t); }

// ----------------------------------------------------------------------------
// elementwise / layout
// ----------------------------------------------------------------------------

__global__ void fill_rows_kernel(float* out, const float* row, int64_t rows, int C) {
  pdl_grid_sync();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * C) return;
  // matmul(ones[P,1], f[1,C]) == 0 + 1*f (network.hpp:466-467)
  out[i] = fa(0.f, fm(1.f, row[i % C]));
}

__global__ void fill_layers_kernel(float* out, const float* per_layer, int L, int64_t P) {
  pdl_grid_sync();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= L * P) return;
  out[i] = per_layer[i / P];
}

__global__ void fill_anchor_depths_kernel(float* out, int L, int64_t P, double inv_span,
                                          double inv_far) {
  pdl_grid_sync();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= L * P) return;
  const int l = int(i / P);
  const float a = __double2float_rn(dd(double(l) + 0.5, double(L)));
  out[i] = __double2float_rn(dd(1.0, da(dm(double(a), inv_span), inv_far)));
}

// mean_pool2 (tape.hpp:816-836): ((a+b)+c+d)*0.25, channel-last.
__global__ void mean_pool2_kernel(const float* in, float* out, int B, int H, int W, int C) {
  pdl_grid_sync();
  const int Ho = H / 2, Wo = W / 2;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)B * Ho * Wo * C;
  if (i >= n) return;
  const int c = int(i % C);
  int64_t t = i / C;
  const int x = int(t % Wo);
  t /= Wo;
  const int y = int(t % Ho);
  const int b = int(t / Ho);
  const float* s = in + (int64_t)b * H * W * C;
  const float v00 = s[((int64_t)(2 * y) * W + 2 * x) * C + c];
  const float v01 = s[((int64_t)(2 * y) * W + 2 * x + 1) * C + c];
  const float v10 = s[((int64_t)(2 * y + 1) * W + 2 * x) * C + c];
  const float v11 = s[((int64_t)(2 * y + 1) * W + 2 * x + 1) * C + c];
  out[i] = fm(fa(fa(fa(v00, v01), v10), v11), 0.25f);
}

// C % 4 == 0: one thread per (output pixel, channel group), same sum order.
__global__ void mean_pool2x4_kernel(const float4* __restrict__ in, float4* __restrict__ out, int B,
                                    int H, int W, int G) {
  pdl_grid_sync();
  const int Ho = H / 2, Wo = W / 2;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * Ho * Wo * G) return;
  const int g = int(i % G);
  int64_t t = i / G;
  const int x = int(t % Wo);
  t /= Wo;
  const int y = int(t % Ho);
  const int b = int(t / Ho);
  const float4* s = in + (int64_t)b * H * W * G;
  const float4 v00 = __ldg(s + ((int64_t)(2 * y) * W + 2 * x) * G + g);
  const float4 v01 = __ldg(s + ((int64_t)(2 * y) * W + 2 * x + 1) * G + g);
  const float4 v10 = __ldg(s + ((int64_t)(2 * y + 1) * W + 2 * x) * G + g);
  const float4 v11 = __ldg(s + ((int64_t)(2 * y + 1) * W + 2 * x + 1) * G + g);
  out[i] = make_float4(fm(fa(fa(fa(v00.x, v01.x), v10.x), v11.x), 0.25f),
                       fm(fa(fa(fa(v00.y, v01.y), v10.y), v11.y), 0.25f),
                       fm(fa(fa(fa(v00.z, v01.z), v10.z), v11.z), 0.25f),
                       fm(fa(fa(fa(v00.w, v01.w), v10.w), v11.w), 0.25f));
}

__global__ void resize_hwc_kernel(const float* in, float* out, int B, int H, int W, int C, int Ho,
                                  int Wo) {
  pdl_grid_sync();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)B * Ho * Wo * C;
  if (i >= n) return;
  const int c = int(i % C);
  int64_t t = i / C;
  const int x = int(t % Wo);
  t /= Wo;
  const int y = int(t % Ho);
  const int b = int(t / Ho);
  int y0, y1, x0, x1;
  float fy, fx;
  resize_tap(y, H, Ho, y0, y1, fy);
  resize_tap(x, W, Wo, x0, x1, fx);
  const float* s = in + (int64_t)b * H * W * C;
  out[i] = lerp2(s[((int64_t)y0 * W + x0) * C + c], s[((int64_t)y0 * W + x1) * C + c],
                 s[((int64_t)y1 * W + x0) * C + c], s[((int64_t)y1 * W + x1) * C + c], fx, fy);
}

// resize_hwc for C % 4 == 0: one thread per output pixel, taps computed once,
// channels moved as float4.
__global__ void resize_hwc4_kernel(const float* __restrict__ in, float* __restrict__ out, int B,
                                   int H, int W, int C, int Ho, int Wo) {
  pdl_grid_sync();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * Ho * Wo) return;
  const int x = int(i % Wo);
  const int y = int((i / Wo) % Ho);
  const int b = int(i / ((int64_t)Wo * Ho));
  int y0, y1, x0, x1;
  float fy, fx;
  resize_tap(y, H, Ho, y0, y1, fy);
  resize_tap(x, W, Wo, x0, x1, fx);
  const float4* s = reinterpret_cast<const float4*>(in + (int64_t)b * H * W * C);
  const int G = C / 4;
  const float4* a = s + ((int64_t)y0 * W + x0) * G;
  const float4* bb = s + ((int64_t)y0 * W + x1) * G;
  const float4* c = s + ((int64_t)y1 * W + x0) * G;
  const float4* d = s + ((int64_t)y1 * W + x1) * G;
  float4* o = reinterpret_cast<float4*>(out) + i * G;
  for (int g = 0; g < G; ++g) {
    const float4 A = __ldg(a + g), Bv = __ldg(bb + g), Cv = __ldg(c + g), D = __ldg(d + g);
    o[g] = make_float4(lerp2(A.x, Bv.x, Cv.x, D.x, fx, fy), lerp2(A.y, Bv.y, Cv.y, D.y, fx, fy),
                       lerp2(A.z, Bv.z, Cv.z, D.z, fx, fy), lerp2(A.w, Bv.w, Cv.w, D.w, fx, fy));
  }
}

// resize_hwc for C % 4 == 0, cooperative: one thread per (output pixel,
// channel group g), g fastest, so every tap read and every store is a
// contiguous run; a grid-stride loop keeps each block busy across many
// pixels (the one-pass version's blocks wrote 4 KB each and left the
// kernel at ~40% of HBM bandwidth).
__global__ void __launch_bounds__(256) resize_hwc4c_kernel(const float* __restrict__ in,
                                                           float* __restrict__ out, int B, int H,
                                                           int W, int G, int Ho, int Wo) {
  pdl_grid_sync();
  // grid-stride over (output pixel, channel group), g fastest; each thread
  // derives its pixel's taps itself (32-bit index math: the caller checks
  // the element counts)
  const int total = B * Ho * Wo * G;
  const float4* s4 = reinterpret_cast<const float4*>(in);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (int e = blockIdx.x * 256 + threadIdx.x; e < total; e += gridDim.x * 256) {
    const int i = e / G, g = e - i * G;
    const int q = i / Wo, x = i - q * Wo;
    const int b = q / Ho, y = q - b * Ho;
    int y0, y1, x0, x1;
    float fy, fx;
    resize_tap(y, H, Ho, y0, y1, fy);
    resize_tap(x, W, Wo, x0, x1, fx);
    const int r0 = (b * H + y0) * W, r1 = (b * H + y1) * W;
    const float4 A = __ldg(s4 + (r0 + x0) * G + g);
    const float4 Bv = __ldg(s4 + (r0 + x1) * G + g);
    const float4 Cv = __ldg(s4 + (r1 + x0) * G + g);
    const float4 D = __ldg(s4 + (r1 + x1) * G + g);
    o4[e] = make_float4(lerp2(A.x, Bv.x, Cv.x, D.x, fx, fy), lerp2(A.y, Bv.y, Cv.y, D.y, fx, fy),
                        lerp2(A.z, Bv.z, Cv.z, D.z, fx, fy), lerp2(A.w, Bv.w, Cv.w, D.w, fx, fy));
  }
}

// resize_hwc for C = 4G (G = 8 or 9: the 32-channel maps and the padded
// 36-float feedback rows): one block row per output image row (b, y), its
// y taps computed once; threads over (x, channel group g), g fastest, the
// scales divided once per thread (the per-element version spent most of its
// instructions in f64 divisions and 32-bit index divisions).
template <int G>
__global__ void __launch_bounds__(256) resize_hwc4g_kernel(const float* __restrict__ in,
                                                           float* __restrict__ out, int H, int W,
                                                           int Ho, int Wo, double sy, double sx) {
  pdl_grid_sync();
  // sy, sx = dd(H, Ho), dd(W, Wo), divided once on the host (IEEE binary64,
  // the same value as the device's __ddiv_rn)
  const int row = blockIdx.y;  // b * Ho + y
  const int b = row / Ho, y = row - b * Ho;
  int y0, y1;
  float fy;
  resize_tap_s(y, sy, H, y0, y1, fy);
  const float4* s4 = reinterpret_cast<const float4*>(in);
  float4* o4 = reinterpret_cast<float4*>(out) + (int64_t)row * Wo * G;
  const int r0 = (b * H + y0) * W, r1 = (b * H + y1) * W;
  for (int e = blockIdx.x * 256 + threadIdx.x; e < Wo * G; e += gridDim.x * 256) {
    const int x = e / G, g = e - x * G;
    int x0, x1;
    float fx;
    resize_tap_s(x, sx, W, x0, x1, fx);
    const float4 A = __ldg(s4 + (int64_t)(r0 + x0) * G + g);
    const float4 Bv = __ldg(s4 + (int64_t)(r0 + x1) * G + g);
    const float4 Cv = __ldg(s4 + (int64_t)(r1 + x0) * G + g);
    const float4 D = __ldg(s4 + (int64_t)(r1 + x1) * G + g);
    o4[e] = make_float4(lerp2(A.x, Bv.x, Cv.x, D.x, fx, fy), lerp2(A.y, Bv.y, Cv.y, D.y, fx, fy),
                        lerp2(A.z, Bv.z, Cv.z, D.z, fx, fy), lerp2(A.w, Bv.w, Cv.w, D.w, fx, fy));
  }
}

// One warp per row: rinv = 1 / sqrt(sum(x^2)/C + 1e-6).
__global__ void rms_rinv_kernel(const float* x, float* rinv, int64_t rows, int C) {
  pdl_grid_sync();
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float s = 0.f;
  for (int c = lane; c < C; c += 32) {
    const float v = x[row * C + c];
    s = fmaf(v, v, s);
  }
  s = warp_sum(s);
  if (lane == 0) rinv[row] = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(s, float(C)), 1e-6f)));
}

// ----------------------------------------------------------------------------
// ray encodings
// ----------------------------------------------------------------------------

// ray_plane_delta + ray_encoding_base (geometry.hpp:343-391): [M, h, w, 32].
__global__ void ray_base_kernel(const RayBaseCam* cams, RayBaseArgs a, float* base) {
  pdl_grid_sync();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)a.M * a.h * a.w) return;
  const int j = int(i % a.w);
  const int ii = int((i / a.w) % a.h);
  const int m = int(i / ((int64_t)a.w * a.h));
  const RayBaseCam& g = cams[m];
  const double d0 = dd(ds(double(j) + 0.5, g.cx), g.fx);
  const double d1 = dd(ds(double(ii) + 0.5, g.cy), g.fy);
  double dw[3], d[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    dw[r] = da(da(dm(g.Rwc_in[r * 3 + 0], d0), dm(g.Rwc_in[r * 3 + 1], d1)), dm(g.Rwc_in[r * 3 + 2], 1.0));
#pragma unroll
  for (int r = 0; r < 3; ++r)
    d[r] = da(da(dm(a.Rcw_t[r * 3 + 0], dw[0]), dm(a.Rcw_t[r * 3 + 1], dw[1])), dm(a.Rcw_t[r * 3 + 2], dw[2]));
  const double dz = d[2] >= 0 ? fmax(d[2], 1e-6) : fmin(d[2], -1e-6);
  const double sx = ds(g.o[0], dm(dd(d[0], dz), g.o[2]));
  const double sy = ds(g.o[1], dm(dd(d[1], dz), g.o[2]));
  const double e[2] = {tanh(dd(dm(dm(a.tfx, sx), a.inv_span), a.half_w)),
                       tanh(dd(dm(dm(a.tfy, sy), a.inv_span), a.half_h))};
  float* out = base + i * 32;
#pragma unroll
  for (int comp = 0; comp < 2; ++comp)
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const double arg = dm(3.141592653589793 * double(1 << o), e[comp]);
      double sv, cv;
      sincos(arg, &sv, &cv);
      out[comp * 16 + 2 * o] = __double2float_rn(sv);
      out[comp * 16 + 2 * o + 1] = __double2float_rn(cv);
    }
}

// rays_k[p, c] = sum_f resize(base)[p, f] * proj[f, c] (network.hpp:405-411).
__global__ void ray_project_kernel(const float* base, int M, int hK, int wK, int Hk, int Wk,
                                   const float* proj, int C, float* out) {
  pdl_grid_sync();
  extern __shared__ __align__(16) float s_proj[];
  for (int e = threadIdx.x; e < 32 * C; e += blockDim.x) s_proj[e] = proj[e];
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * Hk * Wk) return;
  const int x = int(i % Wk);
  const int y = int((i / Wk) % Hk);
  const int m = int(i / ((int64_t)Wk * Hk));
  const float* b = base + (int64_t)m * hK * wK * 32;
  float f[32];
  if (Hk == hK && Wk == wK) {
#pragma unroll
    for (int k = 0; k < 32; ++k) f[k] = b[((int64_t)y * wK + x) * 32 + k];
  } else {
    int y0, y1, x0, x1;
    float fy, fx;
    resize_tap(y, hK, Hk, y0, y1, fy);
    resize_tap(x, wK, Wk, x0, x1, fx);
#pragma unroll
    for (int k = 0; k < 32; ++k)
      f[k] = lerp2(b[((int64_t)y0 * wK + x0) * 32 + k], b[((int64_t)y0 * wK + x1) * 32 + k],
                   b[((int64_t)y1 * wK + x0) * 32 + k], b[((int64_t)y1 * wK + x1) * 32 + k], fx, fy);
  }
  float* o = out + i * C;
  if (C == 32) {  // production width: accumulators in registers, float4 weight broadcasts
    float acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 w = reinterpret_cast<const float4*>(s_proj + k * 32)[c4];
        acc[4 * c4] = fmaf(f[k], w.x, acc[4 * c4]);
        acc[4 * c4 + 1] = fmaf(f[k], w.y, acc[4 * c4 + 1]);
        acc[4 * c4 + 2] = fmaf(f[k], w.z, acc[4 * c4 + 2]);
        acc[4 * c4 + 3] = fmaf(f[k], w.w, acc[4 * c4 + 3]);
      }
    }
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4)
      reinterpret_cast<float4*>(o)[c4] =
          make_float4(acc[4 * c4], acc[4 * c4 + 1], acc[4 * c4 + 2], acc[4 * c4 + 3]);
    return;
  }
  for (int c = 0; c < C; ++c) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) acc = fmaf(f[k], s_proj[k * C + c], acc);
    o[c] = acc;
  }
}

// C = 32 production path: float4 tap reads, the block's 128 output rows
// staged in shared memory and written back as contiguous float4 runs.
// ray_proj weights [32][32] by value (parameter space): every FMA takes its
// weight as a constant-bank / uniform-register operand (the shared-memory
// version spent a broadcast float4 load per four FMAs).
struct RayProjParam {
  float w[32 * 32];
};

// rays_k = resize(base) @ ray_proj for C = 32: thread per output pixel,
// 32-bit index math; PW: weights from `pw`, else staged in shared memory.
template <bool PW>
__global__ void __launch_bounds__(128) ray_project32_kernel(const float* __restrict__ base, int M,
                                                            int hK, int wK, int Hk, int Wk,
                                                            const float* __restrict__ proj,
                                                            float* __restrict__ out,
                                                            const __grid_constant__ RayProjParam pw) {
  pdl_grid_sync();
  __shared__ __align__(16) float s_proj[PW ? 4 : 32 * 32];
  __shared__ __align__(16) float4 s_o[128 * 8];  // [row][c4 ^ (row & 7)]
  if (!PW) {
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) s_proj[e] = __ldg(proj + e);
    __syncthreads();
  }
  const int t = threadIdx.x;
  const int n = M * Hk * Wk;  // < 2^31 (checked by the caller)
  const int i0 = blockIdx.x * 128, i = i0 + t;
  if (i < n) {
    const int q = i / Wk, x = i - q * Wk;
    const int m = q / Hk, y = q - m * Hk;
    const float4* b = reinterpret_cast<const float4*>(base + (int64_t)m * hK * wK * 32);
    float f[32];
    if (Hk == hK && Wk == wK) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 v = __ldg(b + (y * wK + x) * 8 + g);
        f[4 * g] = v.x, f[4 * g + 1] = v.y, f[4 * g + 2] = v.z, f[4 * g + 3] = v.w;
      }
    } else {
      int y0, y1, x0, x1;
      float fy, fx;
      resize_tap(y, hK, Hk, y0, y1, fy);
      resize_tap(x, wK, Wk, x0, x1, fx);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 A = __ldg(b + (y0 * wK + x0) * 8 + g);
        const float4 B = __ldg(b + (y0 * wK + x1) * 8 + g);
        const float4 Cc = __ldg(b + (y1 * wK + x0) * 8 + g);
        const float4 D = __ldg(b + (y1 * wK + x1) * 8 + g);
        f[4 * g] = lerp2(A.x, B.x, Cc.x, D.x, fx, fy);
        f[4 * g + 1] = lerp2(A.y, B.y, Cc.y, D.y, fx, fy);
        f[4 * g + 2] = lerp2(A.z, B.z, Cc.z, D.z, fx, fy);
        f[4 * g + 3] = lerp2(A.w, B.w, Cc.w, D.w, fx, fy);
      }
    }
    float acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 w = PW ? make_float4(pw.w[k * 32 + 4 * c4], pw.w[k * 32 + 4 * c4 + 1],
                                          pw.w[k * 32 + 4 * c4 + 2], pw.w[k * 32 + 4 * c4 + 3])
                            : reinterpret_cast<const float4*>(s_proj + k * 32)[c4];
        acc[4 * c4] = fmaf(f[k], w.x, acc[4 * c4]);
        acc[4 * c4 + 1] = fmaf(f[k], w.y, acc[4 * c4 + 1]);
        acc[4 * c4 + 2] = fmaf(f[k], w.z, acc[4 * c4 + 2]);
        acc[4 * c4 + 3] = fmaf(f[k], w.w, acc[4 * c4 + 3]);
      }
    }
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4)
      s_o[t * 8 + (c4 ^ (t & 7))] =
          make_float4(acc[4 * c4], acc[4 * c4 + 1], acc[4 * c4 + 2], acc[4 * c4 + 3]);
  }
  __syncthreads();
  float4* o = reinterpret_cast<float4*>(out) + (int64_t)i0 * 8;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = t + 128 * k, r = j >> 3, c4 = j & 7;
    if (i0 + r < n) o[j] = s_o[r * 8 + (c4 ^ (r & 7))];
  }
}

// ----------------------------------------------------------------------------
// Stage 1: reprojection + bilinear feature gather
// ----------------------------------------------------------------------------

// One thread per (texel, view); consecutive threads = consecutive texels of
// one view. The world point and footprint are computed once (f64, bit-exact
// order); the 4 taps are read as whole channel rows and the result is written
// as the texel-view's row of Δ[m][p][C].
template <bool kVec4>
__global__ void gather_stack_kernel(const float* __restrict__ feats, int M, int Hf, int Wf, int C,
                                    const DevCam* __restrict__ cams, DevRayCam rc,
                                    const float* __restrict__ depth, int L, int H, int W,
                                    float* __restrict__ deltas) {
  pdl_grid_sync();
  const int64_t P = (int64_t)L * H * W;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P * M) return;
  const int m = int(i / P);
  const int64_t p = i - m * P;
  const int G = (C + 3) / 4;
  const int j = int(p % W);
  const int ii = int((p / W) % H);
  float pt[3];
  world_point(rc, ii, j, __ldg(depth + p), pt);
  const Footprint f = project_footprint(cams[m], pt);
  float* o = deltas + ((int64_t)m * P + p) * C;
  if (!f.valid) {
    for (int c = 0; c < C; ++c) o[c] = 0.f;
    return;
  }
  double w[4];
  bilinear_weights(f, w);
  const float* img = feats + (int64_t)m * Hf * Wf * C;
  const float* i00 = img + ((int64_t)f.y0 * Wf + f.x0) * C;
  const float* i10 = img + ((int64_t)f.y0 * Wf + f.x1) * C;
  const float* i01 = img + ((int64_t)f.y1 * Wf + f.x0) * C;
  const float* i11 = img + ((int64_t)f.y1 * Wf + f.x1) * C;
  if (kVec4) {
    for (int g = 0; g < G; ++g) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(i00) + g);
      const float4 b = __ldg(reinterpret_cast<const float4*>(i10) + g);
      const float4 c = __ldg(reinterpret_cast<const float4*>(i01) + g);
      const float4 d = __ldg(reinterpret_cast<const float4*>(i11) + g);
      reinterpret_cast<float4*>(o)[g] =
          make_float4(blend4(w, a.x, b.x, c.x, d.x), blend4(w, a.y, b.y, c.y, d.y),
                      blend4(w, a.z, b.z, c.z, d.z), blend4(w, a.w, b.w, c.w, d.w));
    }
  } else {
    for (int c = 0; c < C; ++c) o[c] = blend4(w, __ldg(i00 + c), __ldg(i10 + c), __ldg(i01 + c), __ldg(i11 + c));
  }
}

// C = 32: each lane computes one (view, texel) footprint as above (f64,
// bit-exact taps / validity / weights). The warp's 32 texel-views (32
// consecutive texels of one output row, mostly) are then consumed by four
// 8-lane groups, group q taking texel-views 8q .. 8q+7 in order and lane g of
// the group channel group g (16 bytes) of each 128-byte feature row. Adjacent
// texels project to adjacent feature cells (about one feature pixel per
// texel), so a group keeps the previous texel-view's two tap columns in
// registers: when the cell is the same, or the next one to the right, only
// the new right column is loaded -- about 2 of the 4 tap rows per
// texel-view instead of 4, which halves the L1 wavefronts this kernel is
// bound by. Stores are one 128-byte row of Δ[m][p][32] per texel-view. The
// 4-tap blend is an f32 FMA chain over the f64 weights rounded to f32
// (within ~2 ulp of the reference's f64 blend; the parity gate is the RGB
// tolerance), the same values whichever loads were reused.
// 6 CTAs per SM (<= 40 registers): 0.78 -> 0.70 ms per frame against the
// unconstrained 47 registers (ncu A/B, profiles/debug/ab_kernel.sh)
#ifndef LVSG_GATHER_CS
#define LVSG_GATHER_CS 1
#endif
#ifndef LVSG_GATHER_UNROLL
#define LVSG_GATHER_UNROLL 8
#endif
constexpr int kGatherUnroll = LVSG_GATHER_UNROLL;
__global__ void __launch_bounds__(256, 6) gather_stack32_kernel(
    const float* __restrict__ feats, int M, int Hf, int Wf, const DevCam* __restrict__ cams,
    DevRayCam rc, const float* __restrict__ depth, int L, int H, int W, float* __restrict__ deltas) {
  pdl_grid_sync();
  constexpr int G = 8;
  // grid (texel blocks, views): 32-bit texel indexing (P M < 2^31, checked
  // by the launcher); a warp = 32 consecutive texels of one view
  const int P = L * H * W;
  const int m = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  // record: p, flags (1 valid | 2 x1>x0 | 4 y1>y0 | 8 past the end), tap 00, weights
  int pl = p, flags = 8, off = 0;
  float w[4] = {0.f, 0.f, 0.f, 0.f};
  if (p < P) {
    flags = 0;
    const unsigned pu = unsigned(p);
    const int j = int(pu % unsigned(W));
    const int ii = int((pu / unsigned(W)) % unsigned(H));
    float pt[3];
    world_point(rc, ii, j, __ldg(depth + p), pt);
    const Footprint f = project_footprint(cams[m], pt);
    if (f.valid) {
      double wd[4];
      bilinear_weights(f, wd);
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = __double2float_rn(wd[k]);
      flags = 1 | (f.x1 > f.x0 ? 2 : 0) | (f.y1 > f.y0 ? 4 : 0);
      off = ((m * Hf + f.y0) * Wf + f.x0) * G;
    }
  }
  const float4* f4 = reinterpret_cast<const float4*>(feats);
  float4* o4 = reinterpret_cast<float4*>(deltas);
  const int g = lane & 7, q = lane >> 3;
  // the group's previous texel-view: tap-00 offset and flags (-1: none) and
  // its left (x0) / right (x1) columns at rows y0 / y1
  int poff = -1, pfl = 0;
  float4 l0 = make_float4(0.f, 0.f, 0.f, 0.f), l1 = l0, r0 = l0, r1 = l0;
#pragma unroll kGatherUnroll
  for (int it = 0; it < 8; ++it) {
    const int r = 8 * q + it;
    const int rf = __shfl_sync(0xffffffffu, flags, r);
    const int rp = __shfl_sync(0xffffffffu, pl, r);
    const int ro = __shfl_sync(0xffffffffu, off, r) + g;
    float rw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rw[k] = __shfl_sync(0xffffffffu, w[k], r);
    if (rf & 8) continue;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rf & 1) {
      const int dx = (rf & 2) ? G : 0, dy = (rf & 4) ? Wf * G : 0;
      const bool same_rows = poff >= 0 && ((rf ^ pfl) & 4) == 0;
      LVSG_CHECK(ro >= 0 && int64_t(ro) + dy + dx < int64_t(M) * Hf * Wf * G);
      if (!(same_rows && ro == poff)) {  // not the previous cell: new right column
        if (same_rows && ro == poff + G && (pfl & 2) && dx) {
          l0 = r0;  // the next cell to the right: the old right column is the left
          l1 = r1;
        } else {
          l0 = __ldg(f4 + ro);
          l1 = dy ? __ldg(f4 + ro + dy) : l0;
        }
        r0 = dx ? __ldg(f4 + ro + dx) : l0;
        r1 = dx ? (dy ? __ldg(f4 + ro + dy + dx) : r0) : l1;
      }
      poff = ro;
      pfl = rf;
      const float4 a = l0, b = r0, c = l1, d = r1;
      // the 4-tap chain on channel pairs (packed f32x2 ops: the same per-lane
      // roundings as fmaf / the product)
      const float2 w0 = make_float2(rw[0], rw[0]), w1 = make_float2(rw[1], rw[1]);
      const float2 w2 = make_float2(rw[2], rw[2]), w3 = make_float2(rw[3], rw[3]);
      float2 xy = __fmul2_rn(w0, make_float2(a.x, a.y)), zw = __fmul2_rn(w0, make_float2(a.z, a.w));
      xy = __ffma2_rn(w1, make_float2(b.x, b.y), xy);
      zw = __ffma2_rn(w1, make_float2(b.z, b.w), zw);
      xy = __ffma2_rn(w2, make_float2(c.x, c.y), xy);
      zw = __ffma2_rn(w2, make_float2(c.z, c.w), zw);
      xy = __ffma2_rn(w3, make_float2(d.x, d.y), xy);
      zw = __ffma2_rn(w3, make_float2(d.z, d.w), zw);
      v = make_float4(xy.x, xy.y, zw.x, zw.y);
    } else {
      poff = -1;
    }
#if LVSG_GATHER_CS
    // evict-first: the 128 B rows stream past L2 without pushing out the
    // feature level the next warps still sample
    __stcs(o4 + ((int64_t)m * P + rp) * G + g, v);
#else
    o4[((int64_t)m * P + rp) * G + g] = v;
#endif
  }
}

// ----------------------------------------------------------------------------
// render_to_input_view: decode, splat, composite
// ----------------------------------------------------------------------------

// One thread per texel: a = sigmoid(V w_a) [Ca], sigma, depth, world point.
__global__ void decode_payload_kernel(const float* __restrict__ V, int L, int H, int W, int C,
                                      const float* __restrict__ w_appear, int Ca,
                                      const float* __restrict__ w_sigma,
                                      const float* __restrict__ w_depth, DepthAct act, DevRayCam rc,
                                      float* payload, float* depth, float* points) {
  pdl_grid_sync();
  extern __shared__ float s_w[];  // [C, Ca+2]: appear | sigma | depth
  const int K2 = Ca + 2;
  for (int e = threadIdx.x; e < C * K2; e += blockDim.x) {
    const int k = e / K2, c = e % K2;
    s_w[e] = c < Ca ? w_appear[k * Ca + c] : (c == Ca ? w_sigma[k] : w_depth[k]);
  }
  __syncthreads();
  const int64_t P = (int64_t)L * H * W;
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float* v = V + p * C;
  float* pay = payload + p * payload_stride(Ca + 1);
  // matmul order: k ascending from 0 (kernels_ref.hpp:40-48)
  for (int c = 0; c < Ca + 2; ++c) {
    float acc = 0.f;
    for (int k = 0; k < C; ++k) acc = fmaf(v[k], s_w[k * K2 + c], acc);
    if (c < Ca + 1) {
      pay[c] = sigmoid_ref(acc);
    } else {
      const int l = int(p / ((int64_t)H * W));
      const float d = activate_depth(acc, l, act);
      depth[p] = d;
      const int j = int(p % W), i = int((p / W) % H);
      float pt[3];
      world_point(rc, i, j, d, pt);
      points[p * 3 + 0] = pt[0];
      points[p * 3 + 1] = pt[1];
      points[p * 3 + 2] = pt[2];
    }
  }
}


// ----------------------------------------------------------------------------
// Stage 2: One-to-many attention, blend logits, layer collapse
// ----------------------------------------------------------------------------

// Generic-C fallback of the same arithmetic (small channel counts in tests).
__global__ void attend_generic_kernel(float* V, const float* __restrict__ D, int64_t P, int C,
                                      int M, int heads, const float* __restrict__ wq,
                                      const float* __restrict__ wo, const float* __restrict__ gain,
                                      int zero_scores, float* scratch) {
  pdl_grid_sync();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  float* n = scratch + p * 4 * C;
  float* s = n + C;
  float* hd = s + C;
  float* out = hd + C;
  const float* v = V + p * C;
  float ms = 0.f;
  for (int k = 0; k < C; ++k) ms = fmaf(v[k], v[k], ms);
  const float r = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(ms, float(C)), 1e-6f)));
  for (int k = 0; k < C; ++k) n[k] = fm(fm(v[k], r), gain[k]), out[k] = 0.f;
  const float inv_temp = __double2float_rn(1.0 / sqrt(double(C)));
  float w[kMaxM];
  for (int h = 0; h < heads; ++h) {
    if (zero_scores) {
      for (int m = 0; m < M; ++m) w[m] = __fdiv_rn(1.0f, float(M));
    } else {
      for (int c = 0; c < C; ++c) {
        float acc = 0.f;
        for (int k = 0; k < C; ++k) acc = fmaf(n[k], wq[(h * C + k) * C + c], acc);
        s[c] = acc;
      }
      float mx = 0.f;
      for (int m = 0; m < M; ++m) {
        float acc = 0.f;
        for (int c = 0; c < C; ++c) acc = fmaf(s[c], D[((int64_t)m * P + p) * C + c], acc);
        w[m] = fm(acc, inv_temp);
        mx = m == 0 ? w[m] : fmaxf(mx, w[m]);
      }
      float sum = 0.f;
      for (int m = 0; m < M; ++m) w[m] = expf(fsb(w[m], mx)), sum = fa(sum, w[m]);
      const float inv = __fdiv_rn(1.0f, sum);
      for (int m = 0; m < M; ++m) w[m] = fm(w[m], inv);
    }
    for (int c = 0; c < C; ++c) {
      float acc = 0.f;
      for (int m = 0; m < M; ++m) acc = fmaf(w[m], D[((int64_t)m * P + p) * C + c], acc);
      hd[c] = acc;
    }
    for (int c = 0; c < C; ++c) {
      float acc = out[c];
      for (int k = 0; k < C; ++k) acc = fmaf(hd[k], wo[(h * C + k) * C + c], acc);
      out[c] = acc;
    }
  }
  for (int c = 0; c < C; ++c) V[p * C + c] = fa(V[p * C + c], out[c]);
}

__global__ void blend_logits_kernel(const float* __restrict__ V, const float* __restrict__ D,
                                    int64_t P, int C, int M, const float* __restrict__ bw,
                                    const float* __restrict__ gain, float* logits) {
  pdl_grid_sync();
  extern __shared__ float s_bw[];
  for (int e = threadIdx.x; e < C * C; e += blockDim.x) s_bw[e] = bw[e];
  __syncthreads();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float* v = V + p * C;
  float ms = 0.f;
  for (int k = 0; k < C; ++k) ms = fmaf(v[k], v[k], ms);
  const float r = __fdiv_rn(1.0f, __fsqrt_rn(fa(__fdiv_rn(ms, float(C)), 1e-6f)));
  const float inv_temp = __double2float_rn(1.0 / sqrt(double(C)));
  float q[64];
  const int Cq = C <= 64 ? C : 64;
  for (int c = 0; c < Cq; ++c) {
    float acc = 0.f;
    for (int k = 0; k < C; ++k) acc = fmaf(fm(fm(v[k], r), gain[k]), s_bw[k * C + c], acc);
    q[c] = acc;
  }
  for (int m = 0; m < M; ++m) {
    float acc = 0.f;
    for (int c = 0; c < Cq; ++c) acc = fmaf(q[c], D[((int64_t)m * P + p) * C + c], acc);
    logits[p * M + m] = fm(acc, inv_temp);
  }
}

// layer_collapse per texel: cat = [a, b]; h = gelu(cat W1 + b1);
// out = (a+b)*0.5 + (h W2 + b2). W2 accumulates in 16-column chunks of h so
// the k order stays ascending.
__global__ void layer_collapse_kernel(const float* __restrict__ V, int L2, int64_t PL, int C,
                                      const float* __restrict__ w1, const float* __restrict__ b1,
                                      const float* __restrict__ w2, const float* __restrict__ b2,
                                      float* out) {
  pdl_grid_sync();
  extern __shared__ float smem[];
  float* s_w1 = smem;                 // [2C][2C]
  float* s_w2 = smem + 4 * C * C;     // [2C][C]
  for (int e = threadIdx.x; e < 4 * C * C; e += blockDim.x) s_w1[e] = w1[e];
  for (int e = threadIdx.x; e < 2 * C * C; e += blockDim.x) s_w2[e] = w2[e];
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)L2 * PL) return;
  const int64_t l = t / PL, q = t % PL;
  const float* a = V + ((2 * l) * PL + q) * C;
  const float* b = V + ((2 * l + 1) * PL + q) * C;
  float r[64];
  for (int c = 0; c < C; ++c) r[c] = 0.f;
  for (int j0 = 0; j0 < 2 * C; j0 += 16) {
    float hc[16];
    for (int jj = 0; jj < 16 && j0 + jj < 2 * C; ++jj) {
      const int j = j0 + jj;
      float acc = 0.f;
      for (int k = 0; k < C; ++k) acc = fmaf(a[k], s_w1[k * 2 * C + j], acc);
      for (int k = 0; k < C; ++k) acc = fmaf(b[k], s_w1[(C + k) * 2 * C + j], acc);
      hc[jj] = gelu_ref(fa(acc, b1[j]));
    }
    for (int jj = 0; jj < 16 && j0 + jj < 2 * C; ++jj) {
      const float hv = hc[jj];
      const float* wr = s_w2 + (j0 + jj) * C;
      for (int c = 0; c < C; ++c) r[c] = fmaf(hv, wr[c], r[c]);
    }
  }
  float* o = out + t * C;
  for (int c = 0; c < C; ++c) o[c] = fa(fm(fa(a[c], b[c]), 0.5f), fa(r[c], b2[c]));
}

__global__ void decode_linear_kernel(const float* __restrict__ V, int64_t P, int C,
                                     const float* __restrict__ w, int K, float* out) {
  pdl_grid_sync();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P * K) return;
  const int64_t p = i / K;
  const int j = int(i % K);
  const float* v = V + p * C;
  float acc = 0.f;
  for (int k = 0; k < C; ++k) acc = fmaf(v[k], __ldg(w + k * K + j), acc);
  out[i] = acc;
}

__global__ void decode_scalar_kernel(const float* __restrict__ V, int64_t P, int C,
                                     const float* __restrict__ w, float* out, int64_t PL,
                                     DepthAct act, int do_act) {
  pdl_grid_sync();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float* v = V + p * C;
  float acc = 0.f;
  for (int k = 0; k < C; ++k) acc = fmaf(v[k], __ldg(w + k), acc);
  out[p] = do_act ? activate_depth(acc, int(p / PL), act) : acc;
}

// Both LDM scalar heads of a C = 32 volume in one pass (decode_depth_density,
// network.hpp:525-537): the block's 128 rows are read coalesced into shared
// memory, then each thread runs the two k-ascending dot products of its row.
__global__ void __launch_bounds__(128) decode_scalar2_kernel(const float* __restrict__ V, int64_t P,
                                                             const float* __restrict__ wa,
                                                             float* __restrict__ outa,
                                                             const float* __restrict__ wb,
                                                             float* __restrict__ outb) {
  pdl_grid_sync();
  __shared__ __align__(16) float4 rows[128 * 8];  // [row][c4 ^ (row & 7)]
  __shared__ float s_wa[32], s_wb[32];
  const int t = threadIdx.x;
  if (t < 32) s_wa[t] = __ldg(wa + t);
  else if (t < 64) s_wb[t - 32] = __ldg(wb + t - 32);
  const int64_t p0 = blockIdx.x * (int64_t)128;
  const float4* src = reinterpret_cast<const float4*>(V) + p0 * 8;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = t + 128 * k, r = j >> 3, c4 = j & 7;
    if (p0 + r < P) rows[r * 8 + (c4 ^ (r & 7))] = __ldg(src + j);
  }
  __syncthreads();
  const int64_t p = p0 + t;
  if (p >= P) return;
  float a = 0.f, b = 0.f;
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4) {
    const float4 v = rows[t * 8 + (c4 ^ (t & 7))];
    a = fmaf(v.x, s_wa[4 * c4], a);
    a = fmaf(v.y, s_wa[4 * c4 + 1], a);
    a = fmaf(v.z, s_wa[4 * c4 + 2], a);
    a = fmaf(v.w, s_wa[4 * c4 + 3], a);
    b = fmaf(v.x, s_wb[4 * c4], b);
    b = fmaf(v.y, s_wb[4 * c4 + 1], b);
    b = fmaf(v.z, s_wb[4 * c4 + 2], b);
    b = fmaf(v.w, s_wb[4 * c4 + 3], b);
  }
  outa[p] = a;
  outb[p] = b;
}

// ----------------------------------------------------------------------------
// stage entry points
// ----------------------------------------------------------------------------

__global__ void stage_world_points_kernel(DevRayCam rc, const float* depth, int L, int H, int W,
                                          float* points, double lo, double hi, int* bad) {
  pdl_grid_sync();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= (int64_t)L * H * W) return;
  const float d = depth[p];
  const double dv = double(d);
  if (dv < lo || dv > hi) atomicOr(bad, 1);
  float pt[3];
  world_point(rc, int((p / W) % H), int(p % W), d, pt);
  points[p * 3] = pt[0];
  points[p * 3 + 1] = pt[1];
  points[p * 3 + 2] = pt[2];
}

__global__ void stage_footprints_kernel(DevCam cam, const float* points, int64_t P, int32_t* taps,
                                        uint8_t* valid, double* fracs) {
  pdl_grid_sync();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float pt[3] = {points[p * 3], points[p * 3 + 1], points[p * 3 + 2]};
  const Footprint f = project_footprint(cam, pt);
  taps[p * 4] = f.x0;
  taps[p * 4 + 1] = f.x1;
  taps[p * 4 + 2] = f.y0;
  taps[p * 4 + 3] = f.y1;
  valid[p] = f.valid ? 1 : 0;
  fracs[p * 2] = f.fx;
  fracs[p * 2 + 1] = f.fy;
}

__global__ void stage_gather_kernel(DevCam cam, const float* image, int Hi, int Wi, int C,
                                    const float* points, int64_t P, float* values, float* mask) {
  pdl_grid_sync();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float pt[3] = {points[p * 3], points[p * 3 + 1], points[p * 3 + 2]};
  const Footprint f = project_footprint(cam, pt);
  float* o = values + p * C;
  if (mask) mask[p] = f.valid ? 1.f : 0.f;
  if (!f.valid) {
    for (int c = 0; c < C; ++c) o[c] = 0.f;
    return;
  }
  double w[4];
  bilinear_weights(f, w);
  for (int c = 0; c < C; ++c)
    o[c] = blend4(w, image[((int64_t)f.y0 * Wi + f.x0) * C + c], image[((int64_t)f.y0 * Wi + f.x1) * C + c],
                  image[((int64_t)f.y1 * Wi + f.x0) * C + c], image[((int64_t)f.y1 * Wi + f.x1) * C + c]);
}

// resize_hwc for RGB (the input-side decimation of the views): one thread
// per output pixel, taps computed once for its three channels.
// 3-channel resize (the input-side decimation), one block row per output
// image row (b, y): the y taps once per thread, scales divided on the host,
// 32-bit index math (the caller checks the sizes)
__global__ void __launch_bounds__(256) resize_rgb_kernel(const float* __restrict__ in,
                                                         float* __restrict__ out, int H, int W,
                                                         int Ho, int Wo, double sy, double sx) {
  pdl_grid_sync();
  const int row = blockIdx.y;  // b * Ho + y
  const int b = row / Ho, y = row - b * Ho;
  int y0, y1;
  float fy;
  resize_tap_s(y, sy, H, y0, y1, fy);
  const float* s0 = in + ((int64_t)b * H + y0) * W * 3;
  const float* s1 = in + ((int64_t)b * H + y1) * W * 3;
  float* o = out + (int64_t)row * Wo * 3;
  for (int x = blockIdx.x * 256 + threadIdx.x; x < Wo; x += gridDim.x * 256) {
    int x0, x1;
    float fx;
    resize_tap_s(x, sx, W, x0, x1, fx);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o[x * 3 + c] = lerp2(__ldg(s0 + x0 * 3 + c), __ldg(s0 + x1 * 3 + c), __ldg(s1 + x0 * 3 + c),
                           __ldg(s1 + x1 * 3 + c), fx, fy);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

void fill_rows(float* out, const float* row, int64_t rows, int C, cudaStream_t st) {
  launch_k(fill_rows_kernel, blocks_for(rows * C, 256), 256, 0, st, out, row, rows, C);
}
void fill_layers(float* out, const float* per_layer, int L, int64_t P, cudaStream_t st) {
  launch_k(fill_layers_kernel, blocks_for(L * P, 256), 256, 0, st, out, per_layer, L, P);
}
void fill_anchor_depths(float* out, int L, int64_t P, double inv_span, double inv_far,
                        cudaStream_t st) {
  launch_k(fill_anchor_depths_kernel, blocks_for(L * P, 256), 256, 0, st, out, L, P, inv_span, inv_far);
}
void mean_pool2(const float* in, float* out, int B, int H, int W, int C, cudaStream_t st) {
  const int64_t n = (int64_t)B * (H / 2) * (W / 2) * C;
  if (C % 4 == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    launch_k(mean_pool2x4_kernel, blocks_for(n / 4, 256), 256, 0, st, 
        reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), B, H, W, C / 4);
    return;
  }
  launch_k(mean_pool2_kernel, blocks_for(n, 256), 256, 0, st, in, out, B, H, W, C);
}
void resize_hwc(const float* in, float* out, int B, int H, int W, int C, int Ho, int Wo,
                cudaStream_t st) {
  const int64_t n = (int64_t)B * Ho * Wo * C;
  if (H == Ho && W == Wo) {
    cudaMemcpyAsync(out, in, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
    return;
  }
  const bool al = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (C % 4 == 0 && al) {
    const int64_t px = (int64_t)B * Ho * Wo;
    const int G = C / 4;
    if ((G == 8 || G == 9) && (int64_t)B * H * W * G < (int64_t(1) << 31) &&
        px * G < (int64_t(1) << 31) && (int64_t)B * Ho < 65536) {
      // a few blocks per row, each thread several (x, g) elements: the per-
      // thread row setup is amortised
      const dim3 grid(unsigned(std::min<int64_t>((int64_t(Wo) * G + 1023) / 1024, 8)), unsigned(B * Ho));
      const double sy = double(H) / double(Ho), sx = double(W) / double(Wo);
      if (G == 8)
        launch_k(resize_hwc4g_kernel<8>, grid, 256, 0, st, in, out, H, W, Ho, Wo, sy, sx);
      else
        launch_k(resize_hwc4g_kernel<9>, grid, 256, 0, st, in, out, H, W, Ho, Wo, sy, sx);
    } else if (G >= 4 && G <= 64 && (int64_t)B * H * W * G < (int64_t(1) << 31) &&
               px * G < (int64_t(1) << 31)) {
      const int64_t blocks = (px * G + 255) / 256;
      launch_k(resize_hwc4c_kernel, int(std::min<int64_t>(blocks, 148 * 16)), 256, 0, st, in, out, B,
               H, W, G, Ho, Wo);
    } else {
      launch_k(resize_hwc4_kernel, blocks_for(px, 128), 128, 0, st, in, out, B, H, W, C, Ho, Wo);
    }
    return;
  }
  if (C == 3) {
    if ((int64_t)B * Ho < 65536 && (int64_t)W * 3 < (int64_t(1) << 31)) {
      const dim3 grid(unsigned(std::min<int64_t>((Wo + 255) / 256, 8)), unsigned(B * Ho));
      launch_k(resize_rgb_kernel, grid, 256, 0, st, in, out, H, W, Ho, Wo,
               double(H) / double(Ho), double(W) / double(Wo));
      return;
    }
  }
  launch_k(resize_hwc_kernel, blocks_for(n, 256), 256, 0, st, in, out, B, H, W, C, Ho, Wo);
}
void rms_rinv(const float* x, float* rinv, int64_t rows, int C, cudaStream_t st) {
  launch_k(rms_rinv_kernel, blocks_for(rows * 32, 256), 256, 0, st, x, rinv, rows, C);
}
void ray_base(const RayBaseCam* cams_dev, const RayBaseArgs& a, float* base, cudaStream_t st) {
  const int64_t n = (int64_t)a.M * a.h * a.w;
  launch_k(ray_base_kernel, blocks_for(n, 128), 128, 0, st, cams_dev, a, base);
}
void ray_project(const float* base, int M, int hK, int wK, int Hk, int Wk, const float* proj,
                 int C, float* out, cudaStream_t st, const float* proj_host) {
  const int64_t n = (int64_t)M * Hk * Wk;
  if (C == 32 && n < (int64_t(1) << 31) && (int64_t)M * hK * wK * 32 < (int64_t(1) << 31)) {
    RayProjParam pw;
    if (proj_host) {
      for (int e = 0; e < 32 * 32; ++e) pw.w[e] = proj_host[e];
      launch_k(ray_project32_kernel<true>, blocks_for(n, 128), 128, 0, st, base, M, hK, wK, Hk, Wk,
               proj, out, pw);
    } else {
      launch_k(ray_project32_kernel<false>, blocks_for(n, 128), 128, 0, st, base, M, hK, wK, Hk, Wk,
               proj, out, pw);
    }
    return;
  }
  launch_k(ray_project_kernel, blocks_for(n, 128), 128, 32 * C * sizeof(float), st, base, M, hK, wK, Hk,
                                                                               Wk, proj, C, out);
}
void gather_stack(const float* feats, int M, int Hf, int Wf, int C, const DevCam* cams_dev,
                  const DevRayCam& rc, const float* depth, int L, int H, int W, float* deltas,
                  cudaStream_t st) {
  const bool v4 = C % 4 == 0;
  const int64_t n = (int64_t)L * H * W * M;
  if (C == 32 && (int64_t)M * Hf * Wf * 8 < (int64_t(1) << 31) && n < (int64_t(1) << 31)) {
    const int64_t P = (int64_t)L * H * W;
    launch_k(gather_stack32_kernel, dim3(blocks_for(P, 256), M), 256, 0, st, feats, M, Hf, Wf,
             cams_dev, rc, depth, L, H, W, deltas);
  } else if (v4)
    launch_k(gather_stack_kernel<true>, blocks_for(n, 256), 256, 0, st, feats, M, Hf, Wf, C, cams_dev, rc,
                                                                  depth, L, H, W, deltas);
  else
    launch_k(gather_stack_kernel<false>, blocks_for(n, 256), 256, 0, st, feats, M, Hf, Wf, C, cams_dev,
                                                                   rc, depth, L, H, W, deltas);
}
void decode_payload(const float* V, int L, int H, int W, int C, const float* w_appear, int Ca,
                    const float* w_sigma, const float* w_depth, const DepthAct& act,
                    const DevRayCam& rc, float* payload, float* depth, float* points,
                    cudaStream_t st, const float* w_host) {
  if (decode_payload32(V, L, H, W, C, w_appear, Ca, w_sigma, w_depth, act, rc, payload, depth,
                       points, st, w_host))
    return;
  const int64_t P = (int64_t)L * H * W;
  launch_k(decode_payload_kernel, blocks_for(P, 128), 128, C * (Ca + 2) * sizeof(float), st, 
      V, L, H, W, C, w_appear, Ca, w_sigma, w_depth, act, rc, payload, depth, points);
}

__global__ void deltas_to_view_major_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                            int64_t P, int M, int C) {
  pdl_grid_sync();
  const int64_t n = P * M * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    // e enumerates dst: (m * P + p) * C + c
    const int c = int(e % C);
    const int64_t r = e / C;
    const int64_t p = r % P;
    const int m = int(r / P);
    dst[e] = src[(p * M + m) * C + c];
  }
}
__global__ void copy_pinned_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   size_t bytes, int vec) {
  pdl_grid_sync();  // the previous frame's kernels may still read dst
  const size_t n16 = vec ? bytes / 16 : 0;
  const size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x, nt = size_t(gridDim.x) * blockDim.x;
  for (size_t i = t; i < n16; i += nt)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (size_t i = n16 * 16 + t; i < bytes; i += nt) dst[i] = src[i];
}
void copy_from_pinned(void* dst, const void* pinned_src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  void* src = nullptr;
  if (cudaHostGetDevicePointer(&src, const_cast<void*>(pinned_src), 0) != cudaSuccess)
    throw CudaError("copy_from_pinned: source is not mapped pinned memory");
  const int vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int blocks = int(std::min<size_t>((bytes / 16 + 255) / 256 + 1, 16));
  launch_k(copy_pinned_kernel, blocks, 256, 0, st, static_cast<const uint8_t*>(src),
           static_cast<uint8_t*>(dst), bytes, vec);
}

void deltas_to_view_major(const float* src, float* dst, int64_t P, int M, int C, cudaStream_t st) {
  const int64_t n = P * M * C;
  launch_k(deltas_to_view_major_kernel, int(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0,
           st, src, dst, P, M, C);
}
void attend(float* V, const float* deltas, int64_t P, int C, int M, int heads, const float* wq,
            const float* const* wq_heads, const float* wo, const float* gain, int zero_scores,
            float* scratch, const void* wimg, bool wimg_early, int* ovf, cudaStream_t st) {
  (void)wq_heads;
  if (attend_tc(V, deltas, P, C, M, heads, wq, wo, gain, zero_scores, wimg, wimg_early, ovf, st))
    return;
  // generic fallback: 4C floats of scratch per texel (attend_scratch_floats)
  if (!scratch) throw CudaError("attend: no arena scratch for the generic kernel");
  launch_k(attend_generic_kernel, blocks_for(P, 128), 128, 0, st, V, deltas, P, C, M, heads, wq, wo,
                                                            gain, zero_scores, scratch);
}
size_t attend_scratch_floats(int64_t P, int C, int M, int heads) {
  return attend_tc_supported(C, M, heads) ? 0 : size_t(P) * 4 * C;
}
void blend_logits(const float* V, const float* deltas, int64_t P, int C, int M,
                  const float* blend_w, const float* gain, float* logits, cudaStream_t st,
                  const float* blend_w_host) {
  if (blend_logits32(V, deltas, P, C, M, blend_w, gain, logits, st, blend_w_host)) return;
  launch_k(blend_logits_kernel, blocks_for(P, 128), 128, C * C * sizeof(float), st, V, deltas, P, C, M,
                                                                              blend_w, gain, logits);
}
void layer_collapse(const float* V, int L, int64_t PL, int C, const float* w1, const float* b1,
                    const float* w2, const float* b2, float* out, cudaStream_t st) {
  if (layer_collapse32(V, L, PL, C, w1, b1, w2, b2, out, st)) return;
  const int L2 = L / 2;
  launch_k(layer_collapse_kernel, blocks_for(L2 * PL, 128), 128, 6 * C * C * sizeof(float), st, 
      V, L2, PL, C, w1, b1, w2, b2, out);
}
void decode_scalar(const float* V, int64_t P, int C, const float* w, float* out, int L,
                   int64_t PL, const DepthAct* act, cudaStream_t st) {
  (void)L;
  launch_k(decode_scalar_kernel, blocks_for(P, 256), 256, 0, st, V, P, C, w, out, PL,
                                                           act ? *act : DepthAct{}, act ? 1 : 0);
}
void decode_linear(const float* V, int64_t P, int C, const float* w, int K, float* out,
                   cudaStream_t st) {
  launch_k(decode_linear_kernel, blocks_for(P * K, 256), 256, 0, st, V, P, C, w, K, out);
}
void decode_scalar2(const float* V, int64_t P, int C, const float* wa, float* outa, const float* wb,
                    float* outb, cudaStream_t st) {
  if (C == 32) {
    launch_k(decode_scalar2_kernel, blocks_for(P, 128), 128, 0, st, V, P, wa, outa, wb, outb);
  } else {
    decode_scalar(V, P, C, wa, outa, 0, P, nullptr, st);
    decode_scalar(V, P, C, wb, outb, 0, P, nullptr, st);
  }
}
void stage_world_points(const DevRayCam& rc, const float* depth, int L, int H, int W,
                        float* points, double lo, double hi, int* bad, cudaStream_t st) {
  const int64_t n = (int64_t)L * H * W;
  launch_k(stage_world_points_kernel, blocks_for(n, 256), 256, 0, st, rc, depth, L, H, W, points, lo, hi,
                                                                bad);
}
void stage_footprints(const DevCam& cam, const float* points, int64_t P, int32_t* taps,
                      uint8_t* valid, double* fracs, cudaStream_t st) {
  launch_k(stage_footprints_kernel, blocks_for(P, 256), 256, 0, st, cam, points, P, taps, valid, fracs);
}
void stage_gather(const DevCam& cam, const float* image, int Hi, int Wi, int C,
                  const float* points, int64_t P, float* values, float* mask, cudaStream_t st) {
  launch_k(stage_gather_kernel, blocks_for(P, 256), 256, 0, st, cam, image, Hi, Wi, C, points, P, values,
                                                          mask);
}

}  // namespace lvsg
