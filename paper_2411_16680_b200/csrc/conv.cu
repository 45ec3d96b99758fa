// conv3x3 on channel-last fp32 maps: SIMT implicit GEMM.
//
// Semantics: kernels_ref.hpp:72-96 (y = b + sum_{ci,di,dj} w*x with zero
// padding), accumulated in the reference's (ci, dy, dx) order starting from
// the bias, with FFMA (fp32-accurate; see SURVEY.md §7 hard part 2 for why the
// solve path stays fp32 at 1080p).
//
// Tiling: one CTA = 8x32 output pixels x 32 output channels, 128 threads.
// Warp w owns couts [8w, 8w+8); lane (r = lane/4, q = lane%4) owns the 8
// pixels of row r, columns [8q, 8q+8). Input channels stream through shared
// memory 8 at a time as a (8+2)x(32+2) halo tile (row pitch 36 floats so every
// lane's 8-wide window is 16-byte aligned and conflict-free); the 9x8x32
// weight slab is read with warp-broadcast LDS.128.
#include <cstdlib>

#include "kernels.h"

namespace lvsg {
namespace {

constexpr int TH = 8, TW = 32, CK = 8, HP = TH + 2, WP = 36, COT = 32;
constexpr int NT = 128;

__device__ __forceinline__ float load_src(const ConvArgs& a, int b, int pix, int ch) {
  // channel -> source (concat_last order)
  int c = ch;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s < a.nsrc) {
      const ConvSrc& S = a.src[s];
      if (c < S.C) return __ldg(S.ptr + (long long)b * S.bstride + (long long)pix * S.pstride + c);
      c -= S.C;
    }
  }
  return 0.f;
}

__global__ void __launch_bounds__(NT) conv3x3_kernel(const ConvArgs a) {
  pdl_grid_sync();
  __shared__ __align__(16) float s_in[CK * HP * WP];
  __shared__ __align__(16) float s_w[9 * CK * COT];

  const int tiles_x = (a.W + TW - 1) / TW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int x0 = tx * TW, y0 = ty * TH;
  const int co_base = blockIdx.y * COT;
  const int b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, q = lane & 3;
  const int cw = co_base + warp * 8;  // first cout of this warp

  float acc[8][8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int co = cw + c;
    const float bv = (a.bias && co < a.Cout) ? __ldg(a.bias + co) : 0.f;
#pragma unroll
    for (int p = 0; p < 8; ++p) acc[p][c] = bv;
  }

  const int HW = a.H * a.W;
  for (int c0 = 0; c0 < a.Cin; c0 += CK) {
    __syncthreads();
    // stage the input halo tile: element e -> (pixel, channel-in-chunk)
    for (int e = tid; e < HP * (TW + 2) * CK; e += NT) {
      const int ch = e % CK, pix = e / CK;
      const int hy = pix / (TW + 2), hx = pix % (TW + 2);
      const int gy = y0 - 1 + hy, gx = x0 - 1 + hx, gc = c0 + ch;
      float v = 0.f;
      if (gy >= 0 && gy < a.H && gx >= 0 && gx < a.W && gc < a.Cin) {
        const int gp = gy * a.W + gx;
        v = load_src(a, b, gp, gc);
        if (a.rinv) v = fm(fm(v, __ldg(a.rinv + (long long)b * HW + gp)), __ldg(a.gain + gc));
      }
      s_in[(ch * HP + hy) * WP + hx] = v;
    }
    // stage the weight slab [tap][ci][co]
    for (int e = tid; e < 9 * CK * COT; e += NT) {
      const int tap = e % 9, rest = e / 9;
      const int ci = rest % CK, co = rest / CK;
      const int gci = c0 + ci, gco = co_base + co;
      float v = 0.f;
      if (gci < a.Cin && gco < a.Cout)
        v = __ldg(a.w + ((long long)gco * w_cin_of(a) + a.w_ci0 + gci) * 9 + tap);
      s_w[(tap * CK + ci) * COT + co] = v;
    }
    __syncthreads();
#pragma unroll 2
    for (int ci = 0; ci < CK; ++ci) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
        const float* row = s_in + (ci * HP + r + dy) * WP + 8 * q;
        const float4 v0 = *reinterpret_cast<const float4*>(row);
        const float4 v1 = *reinterpret_cast<const float4*>(row + 4);
        const float2 v2 = *reinterpret_cast<const float2*>(row + 8);
        const float xin[10] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y};
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const float* wr = s_w + ((dy * 3 + dx) * CK + ci) * COT + warp * 8;
          const float4 wa = *reinterpret_cast<const float4*>(wr);
          const float4 wb = *reinterpret_cast<const float4*>(wr + 4);
          const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
          for (int p = 0; p < 8; ++p)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[p][c] = fmaf(xin[p + dx], wv[c], acc[p][c]);
        }
      }
    }
  }

  // epilogue: GELU, residual, store
  const int gy = y0 + r;
  if (gy >= a.H) return;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int gx = x0 + 8 * q + p;
    if (gx >= a.W) continue;
    const long long pix = (long long)gy * a.W + gx;
    float* o = a.out + (long long)b * a.out_bstride + pix * a.out_pstride;
    const float* rs = a.resid ? a.resid + (long long)b * a.res_bstride + pix * a.res_pstride : nullptr;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int co = cw + c;
      if (co >= a.Cout) continue;
      float y = acc[p][c];
      if (a.gelu) y = gelu_ref(y);
      if (rs) y = fa(rs[co], y);
      o[co] = y;
    }
  }
}

// Stem weights by value: [k = ci*9+tap][32] and the bias (zero when the
// conv has none), in the kernel's parameter space.
struct StemParam {
  float w[27 * 32];
  float b[32];
};

// Few-input-channel conv (Cin = CI in {1, 3} -> Cout = 32): the encoder
// stem (encode_inputs network.hpp:390) and the feedback-alpha slice of the
// update stems. One thread per output pixel, the 9*CI taps in registers,
// weights [k = ci*9+tap][32], k ascending from the bias like the reference;
// optional residual (accumulating slices). PW: the weights come from the
// parameter block `pw` (constant-bank FMA operands: the shared-memory
// version is bound by its 27*8 weight loads per pixel); else they are
// staged in shared memory and read as broadcast float4s.
template <int CI, bool PW>
__global__ void __launch_bounds__(128) conv3x3_stem_kernel(const ConvArgs a,
                                                           const __grid_constant__ StemParam pw) {
  pdl_grid_sync();
  __shared__ __align__(16) float s_w[PW ? 4 : 9 * CI * 32];
  __shared__ float s_b[32];
  __shared__ __align__(16) float4 s_o[128 * 8];  // [pixel][c4 ^ (pixel & 7)]
  if (!PW) {
    for (int e = threadIdx.x; e < 9 * CI * 32; e += blockDim.x) {
      const int co = e % 32, k = e / 32;
      s_w[e] = __ldg(a.w + ((long long)co * w_cin_of(a) + a.w_ci0) * 9 + k);
    }
    if (threadIdx.x < 32) s_b[threadIdx.x] = a.bias ? __ldg(a.bias + threadIdx.x) : 0.f;
    __syncthreads();
  }
  const int64_t HW = (int64_t)a.H * a.W;
  const int64_t n = HW * a.B;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x;
  const int64_t i = i0 + threadIdx.x;
  const int t = threadIdx.x;
  // the block's 128 consecutive pixels: one 64-bit division per block, then
  // 32-bit arithmetic per thread (the carry loop also covers images smaller
  // than a block)
  const int b_blk = int(i0 / HW);
  const int pix_blk = int(i0 - b_blk * HW);
  auto locate = [&](int k, int& b, int& pix) {  // pixel i0 + k -> (image, pixel)
    b = b_blk;
    pix = pix_blk + k;
    while (pix >= HW) pix -= int(HW), ++b;
  };
  if (i < n) {
    int b, pix;
    locate(t, b, pix);
    const int y = pix / a.W, x = pix - (pix / a.W) * a.W;
    const ConvSrc& S = a.src[0];
    const float* src = S.ptr + (long long)b * S.bstride + (long long)pix * S.pstride;
    const int row = a.W * S.pstride;
    float xin[9 * CI];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int yy = y + dy - 1, xx = x + dx - 1;
        const bool ok = yy >= 0 && yy < a.H && xx >= 0 && xx < a.W;
        const float* p = src + ((dy - 1) * row + (dx - 1) * S.pstride);
#pragma unroll
        for (int ci = 0; ci < CI; ++ci) xin[ci * 9 + dy * 3 + dx] = ok ? __ldg(p + ci) : 0.f;
      }
    float acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = PW ? pw.b[c] : s_b[c];
#pragma unroll
    for (int k = 0; k < 9 * CI; ++k) {
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 w = PW ? make_float4(pw.w[k * 32 + 4 * c4], pw.w[k * 32 + 4 * c4 + 1],
                                          pw.w[k * 32 + 4 * c4 + 2], pw.w[k * 32 + 4 * c4 + 3])
                            : reinterpret_cast<const float4*>(s_w + k * 32)[c4];
        acc[4 * c4] = fmaf(xin[k], w.x, acc[4 * c4]);
        acc[4 * c4 + 1] = fmaf(xin[k], w.y, acc[4 * c4 + 1]);
        acc[4 * c4 + 2] = fmaf(xin[k], w.z, acc[4 * c4 + 2]);
        acc[4 * c4 + 3] = fmaf(xin[k], w.w, acc[4 * c4 + 3]);
      }
    }
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
      float v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = a.gelu ? gelu_ref(acc[4 * c4 + k]) : acc[4 * c4 + k];
      s_o[t * 8 + (c4 ^ (t & 7))] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  __syncthreads();
  // coalesced write-back of the block's consecutive pixels (+ residual), one
  // float4 per thread per step: 8 threads cover one pixel's 128 bytes
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = t + 128 * k, pl = j >> 3, c4 = j & 7;
    const int64_t ip = i0 + pl;
    if (ip >= n) continue;
    int b, pix;
    locate(pl, b, pix);
    float4 v = s_o[pl * 8 + (c4 ^ (pl & 7))];
    if (a.resid) {
      const float4 r = __ldg(reinterpret_cast<const float4*>(a.resid + (long long)b * a.res_bstride +
                                                              (long long)pix * a.res_pstride) + c4);
      v = make_float4(fa(r.x, v.x), fa(r.y, v.y), fa(r.z, v.z), fa(r.w, v.w));
    }
    reinterpret_cast<float4*>(a.out + (long long)b * a.out_bstride + (long long)pix * a.out_pstride)[c4] = v;
  }
}

// The encoder stem (Cin = 3, weights by value as in conv3x3_stem_kernel<3,
// true>) with two horizontally adjacent output pixels per thread: each
// constant-bank weight feeds two FMAs and the two pixels share 8 of their
// 12 tap columns. Requires an even W (pairs never straddle a row or an
// image); same per-pixel arithmetic and order as the one-pixel kernel.
#ifndef LVSG_STEM_FFMA2
#define LVSG_STEM_FFMA2 1
#endif
__global__ void __launch_bounds__(128) conv3x3_stem3x2_kernel(const ConvArgs a,
                                                              const __grid_constant__ StemParam pw) {
  pdl_grid_sync();
  __shared__ __align__(16) float4 s_o[256 * 8];  // [pixel][c4 ^ (pixel & 7)]
  const int64_t HW = (int64_t)a.H * a.W;
  const int64_t n = HW * a.B;
  const int64_t i0 = blockIdx.x * (int64_t)256;
  const int t = threadIdx.x;
  const int b_blk = int(i0 / HW);
  const int pix_blk = int(i0 - b_blk * HW);
  auto locate = [&](int k, int& b, int& pix) {  // pixel i0 + k -> (image, pixel)
    b = b_blk;
    pix = pix_blk + k;
    while (pix >= HW) pix -= int(HW), ++b;
  };
  if (i0 + 2 * t < n) {
    int b, pix;
    locate(2 * t, b, pix);
    const int y = pix / a.W, x = pix - y * a.W;  // x even
    const ConvSrc& S = a.src[0];
    const float* src = S.ptr + (long long)b * S.bstride + (long long)pix * S.pstride;
    const int row = a.W * S.pstride;
    float xin[3][4][3];  // [dy][column x-1 .. x+2][ci]
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int cx = 0; cx < 4; ++cx) {
        const int yy = y + dy - 1, xx = x + cx - 1;
        const bool ok = yy >= 0 && yy < a.H && xx >= 0 && xx < a.W;
        const float* p = src + ((dy - 1) * row + (cx - 1) * S.pstride);
#pragma unroll
        for (int ci = 0; ci < 3; ++ci) xin[dy][cx][ci] = ok ? __ldg(p + ci) : 0.f;
      }
    float acc0[32], acc1[32];
#if LVSG_STEM_FFMA2
    // packed f32x2 FMAs over channel pairs (sm_100 FFMA2: two IEEE fmas per
    // instruction, the same roundings): half the FMA instructions
    float2 a0[16], a1[16];
#pragma unroll
    for (int c2 = 0; c2 < 16; ++c2) a0[c2] = a1[c2] = make_float2(pw.b[2 * c2], pw.b[2 * c2 + 1]);
#pragma unroll
    for (int ci = 0; ci < 3; ++ci)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int k = ci * 9 + dy * 3 + dx;
          const float2 x0 = make_float2(xin[dy][dx][ci], xin[dy][dx][ci]);
          const float2 x1 = make_float2(xin[dy][dx + 1][ci], xin[dy][dx + 1][ci]);
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            const float2 w = make_float2(pw.w[k * 32 + 2 * c2], pw.w[k * 32 + 2 * c2 + 1]);
            a0[c2] = __ffma2_rn(x0, w, a0[c2]);
            a1[c2] = __ffma2_rn(x1, w, a1[c2]);
          }
        }
#pragma unroll
    for (int c2 = 0; c2 < 16; ++c2) {
      acc0[2 * c2] = a0[c2].x, acc0[2 * c2 + 1] = a0[c2].y;
      acc1[2 * c2] = a1[c2].x, acc1[2 * c2 + 1] = a1[c2].y;
    }
#else
#pragma unroll
    for (int c = 0; c < 32; ++c) acc0[c] = acc1[c] = pw.b[c];
#pragma unroll
    for (int ci = 0; ci < 3; ++ci)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int k = ci * 9 + dy * 3 + dx;
          const float x0 = xin[dy][dx][ci], x1 = xin[dy][dx + 1][ci];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            acc0[c] = fmaf(x0, pw.w[k * 32 + c], acc0[c]);
            acc1[c] = fmaf(x1, pw.w[k * 32 + c], acc1[c]);
          }
        }
#endif
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
      const int p0 = 2 * t, p1 = 2 * t + 1;
      s_o[p0 * 8 + (c4 ^ (p0 & 7))] = make_float4(acc0[4 * c4], acc0[4 * c4 + 1], acc0[4 * c4 + 2],
                                                  acc0[4 * c4 + 3]);
      s_o[p1 * 8 + (c4 ^ (p1 & 7))] = make_float4(acc1[4 * c4], acc1[4 * c4 + 1], acc1[4 * c4 + 2],
                                                  acc1[4 * c4 + 3]);
    }
  }
  __syncthreads();
  if (a.out_bstride == HW * 32 && !a.resid) {
    // contiguous [B*H*W, 32] output (the encoder stem): the block's 256
    // pixels are one linear 32 KB run
    float4* dst = reinterpret_cast<float4*>(a.out) + i0 * 8;
    const int np = n - i0 < 256 ? int(n - i0) : 256;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      const int j = t + 128 * k, pl = j >> 3, c4 = j & 7;
      if (pl < np) dst[j] = s_o[pl * 8 + (c4 ^ (pl & 7))];
    }
    return;
  }
  // coalesced write-back (+ residual): 8 threads per pixel's 128 bytes
#pragma unroll 4
  for (int k = 0; k < 16; ++k) {
    const int j = t + 128 * k, pl = j >> 3, c4 = j & 7;
    if (i0 + pl >= n) continue;
    int b, pix;
    locate(pl, b, pix);
    float4 v = s_o[pl * 8 + (c4 ^ (pl & 7))];
    if (a.resid) {
      const float4 r = __ldg(reinterpret_cast<const float4*>(a.resid + (long long)b * a.res_bstride +
                                                              (long long)pix * a.res_pstride) + c4);
      v = make_float4(fa(r.x, v.x), fa(r.y, v.y), fa(r.z, v.z), fa(r.w, v.w));
    }
    reinterpret_cast<float4*>(a.out + (long long)b * a.out_bstride + (long long)pix * a.out_pstride)[c4] = v;
  }
}

bool stem_supported(const ConvArgs& a) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return (a.Cin == 1 || a.Cin == 3) && a.Cout == 32 && a.nsrc == 1 && !a.rinv &&
         a.out_pstride == 32 && al(a.out) && a.out_bstride % 4 == 0 &&
         (!a.resid || (al(a.resid) && a.res_pstride % 4 == 0 && a.res_bstride % 4 == 0));
}

}  // namespace

int conv3x3_path(const ConvArgs& a, int impl) {
  static const int env = [] {
    const char* e = getenv("LVSG_CONV");
    return e && e[0] == 's' ? 1 : 0;  // LVSG_CONV=simt
  }();
  if (impl == 0) impl = env ? env : 2;
  if (impl == 1 || !conv3x3_tc_supported(a)) return 1;
  return 2;
}

bool conv3x3_uses_tc(const ConvArgs& a, int impl) { return conv3x3_path(a, impl) >= 2; }

void conv3x3(const ConvArgs& a, cudaStream_t st, int impl) {
  const int path = conv3x3_path(a, impl);
  if (path == 2) {
    conv3x3_tc(a, st);
  } else if (impl != 1 && stem_supported(a)) {
    const int64_t n = (int64_t)a.B * a.H * a.W;
    const int g = int((n + 127) / 128);
    StemParam pw;
    if (a.Cin == 3 && a.stem_host && a.w_ci0 == 0 && w_cin_of(a) == 3) {
      for (int co = 0; co < 32; ++co) {
        for (int k = 0; k < 27; ++k) pw.w[k * 32 + co] = a.stem_host[co * 27 + k];
        pw.b[co] = a.bias ? a.stem_host[27 * 32 + co] : 0.f;
      }
      if (a.W % 2 == 0 && !a.gelu)
        launch_k(conv3x3_stem3x2_kernel, int((n + 255) / 256), 128, 0, st, a, pw);
      else
        launch_k(conv3x3_stem_kernel<3, true>, g, 128, 0, st, a, pw);
    } else if (a.Cin == 3) {
      launch_k(conv3x3_stem_kernel<3, false>, g, 128, 0, st, a, pw);
    } else {
      launch_k(conv3x3_stem_kernel<1, false>, g, 128, 0, st, a, pw);
    }
  } else {
    conv3x3_simt(a, st);
  }
}

void conv3x3_simt(const ConvArgs& a, cudaStream_t st) {
  const int tiles = ((a.W + TW - 1) / TW) * ((a.H + TH - 1) / TH);
  dim3 grid(tiles, (a.Cout + COT - 1) / COT, a.B);
  launch_k(conv3x3_kernel, grid, NT, 0, st, a);
}

}  // namespace lvsg
