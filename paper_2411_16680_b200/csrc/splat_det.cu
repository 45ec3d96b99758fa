// Deterministic render-to-input-view splat (owner computes): every view
// pixel sums its own contributions in the reference's order, so a frame is
// bit-identical from run to run and every accumulator sees the same f32
// additions, in the same sequence, as splat_accumulate (geometry.hpp:
// 230-264: for l, for texel s ascending, for tap k ascending:
// dst[c] += T(w_k) * val[p, c], then dst[K] += T(w_k)).
//
// Per update step (P = L*H*W texels, M views, bins = M*L*Hv*Wv destination
// pixels):
//   1. splat_count: one thread per (texel, view) pair computes the f64
//      footprint once (the gather's rule), stores it (dest of tap 0, tap
//      offsets, f32 weights) and counts each valid tap into its bin, keeping
//      the count before it (the tap's rank in the bin);
//   2. a three-pass exclusive scan of the bin counts gives each bin its run
//      in the entry array;
//   3. splat_fill: each valid tap writes (key p*4+k, f32 weight) to slot
//      off[bin] + rank of its bin's run (slot order inside a run is
//      arbitrary);
//   4. splat_reduce_composite: one thread per (view pixel, 4-channel group)
//      sorts, layer by layer, its bin's run by key (= the reference's (s, k)
//      order; short runs in registers), accumulates the payload rows,
//      normalises by
//      max(wsum, 1e-4) (splat_project) and over-composites colour and alpha
//      back to front (ldm.hpp:236-243), writing the feedback row.
// It replaces splat_coop + splat_composite (fp32 vector atomics, whose
// accumulation order and hence low bits changed between runs) and the
// accumulator memset.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace lvsg {
namespace {

constexpr int kScanBlock = 1024;  // bins per first-level scan block (256 threads x 4)

__global__ void __launch_bounds__(256) splat_count_kernel(const float* __restrict__ points,
                                                          int L, int PL,
                                                          const DevCam* __restrict__ cams, int M,
                                                          int Hv, int Wv, int* __restrict__ cnt,
                                                          int2* __restrict__ fp_i,
                                                          float4* __restrict__ fp_w,
                                                          int4* __restrict__ rank) {
  pdl_grid_sync();
  const int64_t P = (int64_t)L * PL;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // pair (p, m), m fastest
  if (i >= P * M) return;
  const int m = int(i % M);
  const int64_t p = i / M;
  const int l = int(p / PL);
  const float pt[3] = {__ldg(points + p * 3), __ldg(points + p * 3 + 1), __ldg(points + p * 3 + 2)};
  const Footprint f = project_footprint(cams[m], pt);
  if (!f.valid) {
    fp_i[i] = make_int2(-1, 0);
    return;
  }
  double wd[4];
  bilinear_weights(f, wd);
  const int dx = f.x1 - f.x0, dy = (f.y1 - f.y0) * Wv;
  const int d0 = int(((int64_t)m * L + l) * Hv * Wv + (int64_t)f.y0 * Wv + f.x0);
  fp_i[i] = make_int2(d0, dx | (dy << 1));
  fp_w[i] = make_float4(__double2float_rn(wd[0]), __double2float_rn(wd[1]),
                        __double2float_rn(wd[2]), __double2float_rn(wd[3]));
  // each tap's position in its bin's run (the count before it): the fill
  // then writes entry slots without a second round of atomics
  int4 r;
  r.x = atomicAdd(cnt + d0, 1);
  r.y = atomicAdd(cnt + d0 + dx, 1);
  r.z = atomicAdd(cnt + d0 + dy, 1);
  r.w = atomicAdd(cnt + d0 + dy + dx, 1);
  rank[i] = r;
}

// exclusive scan, pass 1: per-block scan of kScanBlock counts (in place into
// off) and the block totals
__global__ void __launch_bounds__(256) scan_blocks_kernel(const int* __restrict__ cnt, int n,
                                                          int* __restrict__ off,
                                                          int* __restrict__ block_sum) {
  pdl_grid_sync();
  __shared__ int s_warp[8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int base = blockIdx.x * kScanBlock + t * 4;
  int v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = base + k < n ? cnt[base + k] : 0;
  const int tot = v[0] + v[1] + v[2] + v[3];
  int incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  int wpre = 0;
  for (int k = 0; k < w; ++k) wpre += s_warp[k];
  int run = wpre + incl - tot;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (base + k < n) off[base + k] = run;
    run += v[k];
  }
  if (t == 255) block_sum[blockIdx.x] = wpre + incl;
}

// pass 2: one block scans the block totals (exclusive, in place)
__global__ void __launch_bounds__(1024) scan_sums_kernel(int* __restrict__ block_sum, int nb) {
  pdl_grid_sync();
  __shared__ int s_warp[32];
  __shared__ int s_carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int v = b0 + t < nb ? block_sum[b0 + t] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    int wpre = 0;
    for (int k = 0; k < w; ++k) wpre += s_warp[k];
    const int carry = s_carry;
    if (b0 + t < nb) block_sum[b0 + t] = carry + wpre + incl - v;
    __syncthreads();
    if (t == 1023) s_carry = carry + wpre + incl;
    __syncthreads();
  }
}

// pass 3: add each block's base
__global__ void __launch_bounds__(256) scan_add_kernel(int* __restrict__ off, int n,
                                                       const int* __restrict__ block_sum) {
  pdl_grid_sync();
  const int base = blockIdx.x * kScanBlock;
  const int add = block_sum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = base + threadIdx.x + 256 * k;
    if (i < n) off[i] += add;
  }
}

__global__ void __launch_bounds__(256) splat_fill_kernel(int64_t pairs, int64_t bins, int M,
                                                         const int2* __restrict__ fp_i,
                                                         const float4* __restrict__ fp_w,
                                                         const int4* __restrict__ rank,
                                                         const int* __restrict__ off,
                                                         int2* __restrict__ ent) {
  pdl_grid_sync();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= pairs) return;
  const int2 f = fp_i[i];
  if (f.x < 0) return;
  const float4 w = fp_w[i];
  const int4 r = rank[i];
  const int p4 = int(i / M) * 4;
  const int dx = f.y & 1, dy = f.y >> 1;
  const int d[4] = {f.x, f.x + dx, f.x + dy, f.x + dy + dx};
  const int rk[4] = {r.x, r.y, r.z, r.w};
  const float wk[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    LVSG_CHECK(d[k] >= 0 && d[k] < bins);
    const int slot = __ldg(off + d[k]) + rk[k];
    LVSG_CHECK(slot >= 0 && slot < 4 * pairs);
    ent[slot] = make_int2(p4 + k, __float_as_int(wk[k]));
  }
}

// One thread per (view m, pixel, channel group g of G = PS/4), the G lanes
// of a pixel adjacent, kRedPix pixels per block. Each lane accumulates its
// four channels of the run (sorted (texel, tap) order) and the weight sum;
// the alpha (sigma) channel K-1 is accumulated by the lane that owns it and
// shared through shared memory for the composite. ppb pixels per block
// (<= kRedPixMax, blockDim = ppb * G <= 288).
constexpr int kRedPixMax = 64;
#ifndef LVSG_SPLAT_PL3
#define LVSG_SPLAT_PL3 3  // lanes per (view pixel, layer) in splat_reduce_pl3 (0: off)
#endif
constexpr int kRun = 8;  // runs up to this long are sorted in registers

__device__ __forceinline__ void cswap(int2& a, int2& b) {
  const bool sw = a.x > b.x;
  const int2 lo = sw ? b : a, hi = sw ? a : b;
  a = lo;
  b = hi;
}
// Batcher odd-even merge sorting networks on the keys (.x)
__device__ __forceinline__ void sort4(int2* e) {
  cswap(e[0], e[1]); cswap(e[2], e[3]); cswap(e[0], e[2]); cswap(e[1], e[3]); cswap(e[1], e[2]);
}
__device__ __forceinline__ void sort8(int2* e) {
  cswap(e[0], e[1]); cswap(e[2], e[3]); cswap(e[4], e[5]); cswap(e[6], e[7]);
  cswap(e[0], e[2]); cswap(e[1], e[3]); cswap(e[4], e[6]); cswap(e[5], e[7]);
  cswap(e[1], e[2]); cswap(e[5], e[6]);
  cswap(e[0], e[4]); cswap(e[1], e[5]); cswap(e[2], e[6]); cswap(e[3], e[7]);
  cswap(e[2], e[4]); cswap(e[3], e[5]);
  cswap(e[1], e[2]); cswap(e[3], e[4]); cswap(e[5], e[6]);
}

__global__ void __launch_bounds__(288) splat_reduce_composite_kernel(
    const float* __restrict__ payload, int K, int M, int L, int Hv, int Wv,
    const int* __restrict__ off, const int* __restrict__ cnt, const int2* __restrict__ ent,
    float* __restrict__ out, int ppb, int64_t n_ent, int64_t P) {
  pdl_grid_sync();
  __shared__ float s_sig[kRedPixMax];
  const int PS = pay_stride(K), G = PS / 4;
  const int64_t PV = (int64_t)Hv * Wv;
  const int lp = threadIdx.x / G, g = threadIdx.x - lp * G;
  const int64_t t = (int64_t)blockIdx.x * ppb + lp;  // (m, pixel)
  const bool live = lp < ppb && t < (int64_t)M * PV;
  const int64_t pix = live ? t % PV : 0;
  const int m = live ? int(t / PV) : 0;
  const int Ca = K - 1, gs = Ca / 4, ks = Ca % 4;
  const int GP = payload_stride(K) / 4;  // float4 per payload row
  const float4* pay4 = reinterpret_cast<const float4*>(payload);
  float o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int l = 0; l < L; ++l) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, ws = 0.f;
    auto add = [&](const int2 en, const float4 v) {
      const float w = __int_as_float(en.y);
      acc[0] = fa(acc[0], fm(w, v.x));
      acc[1] = fa(acc[1], fm(w, v.y));
      acc[2] = fa(acc[2], fm(w, v.z));
      acc[3] = fa(acc[3], fm(w, v.w));
      ws = fa(ws, w);
    };
    if (live) {
      const int64_t bin = ((int64_t)m * L + l) * PV + pix;
      const int n = __ldg(cnt + bin), b0 = __ldg(off + bin);
      LVSG_CHECK(n >= 0 && b0 >= 0 && (int64_t)b0 + n <= n_ent);
      if (n <= kRun) {
        // short run (the common case): entries into registers, sorted by a
        // fixed network, then every payload load in flight at once
        int2 e[kRun];
#pragma unroll
        for (int k = 0; k < kRun; ++k) e[k] = k < n ? __ldg(ent + b0 + k) : make_int2(0x7fffffff, 0);
        if (n > 4) {
          sort8(e);
        } else if (n > 1) {
          sort4(e);
        }
        float4 v[kRun];
#pragma unroll
        for (int k = 0; k < kRun; ++k)
          if (k < n) v[k] = __ldg(pay4 + (int64_t)(e[k].x >> 2) * GP + g);
#pragma unroll
        for (int k = 0; k < kRun; ++k)
          if (k < n) add(e[k], v[k]);
      } else {
        // long run: ascending keys by repeated minimum search
        int last = -1;
        for (int q = 0; q < n; ++q) {
          int2 best = make_int2(0x7fffffff, 0);
          for (int j = 0; j < n; ++j) {
            const int2 ej = __ldg(ent + b0 + j);
            if (ej.x > last && ej.x < best.x) best = ej;
          }
          last = best.x;
          add(best, __ldg(pay4 + (int64_t)(best.x >> 2) * GP + g));
        }
      }
      if (g == gs) s_sig[lp] = acc[ks];
    }
    __syncthreads();
    // splat_project: * 1/max(wsum, eps); over_composite colour / alpha
    const float nrm = __fdiv_rn(1.0f, ws > 1e-4f ? ws : 1e-4f);
    const float s = fm(live ? s_sig[lp] : 0.f, nrm);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * g + k;
      const float v = c < Ca ? fm(acc[k], nrm) : 1.0f;
      o[k] = fa(fm(v, s), fm(fsb(1.0f, s), o[k]));
    }
    __syncthreads();
  }
  if (!live) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (4 * g + k >= K) o[k] = 0.f;
  reinterpret_cast<float4*>(out)[t * G + g] = make_float4(o[0], o[1], o[2], o[3]);
}

// One thread per (view m, pixel, layer): the run of a layer's bin is summed
// in parallel across layers (the early steps have 24 layers over small view
// images, where a thread per pixel walking the layers in sequence left the
// SMs nearly empty); the normalised values go through shared memory and
// the back-to-front composite then runs per (pixel, channel group) in the
// reference's layer order. Same additions, same order, as
// splat_reduce_composite_kernel.
template <int NG>
__global__ void __launch_bounds__(192) splat_reduce_pl_kernel(
    const float* __restrict__ payload, int K, int M, int L, int Hv, int Wv,
    const int* __restrict__ off, const int* __restrict__ cnt, const int2* __restrict__ ent,
    float* __restrict__ out, int ppb, int64_t n_ent, int64_t P) {
  pdl_grid_sync();
  extern __shared__ float s_val[];  // [ppb][L][NG*4]: normalised channels, [Ca] = alpha
  const int64_t PV = (int64_t)Hv * Wv;
  const int Ca = K - 1;
  const int GP = payload_stride(K) / 4;  // float4 per payload row (>= NG)
  const int64_t t0 = (int64_t)blockIdx.x * ppb;  // first (m, pixel) of the block
  const int lp = threadIdx.x / L, l = threadIdx.x - lp * L;
  const int64_t t = t0 + lp;
  if (lp < ppb && t < (int64_t)M * PV) {
    const int64_t pix = t % PV;
    const int m = int(t / PV);
    float acc[NG * 4];
#pragma unroll
    for (int c = 0; c < NG * 4; ++c) acc[c] = 0.f;
    float ws = 0.f;
    auto add = [&](const int2 en) {
      // the payload row (32-byte aligned, payload_stride floats): the first
      // 32 channels by four 256-bit loads, the rest by 16-byte loads
      const float w = __int_as_float(en.y);
      LVSG_CHECK(en.x >= 0 && (en.x >> 2) < P);
      const float* row = payload + (int64_t)(en.x >> 2) * (4 * GP);
      float v[NG * 4];
#pragma unroll
      for (int q = 0; q < NG / 2; ++q) ldg256(row + 8 * q, v + 8 * q);
#pragma unroll
      for (int q = 2 * (NG / 2); q < NG; ++q) {
        const float4 t4 = __ldg(reinterpret_cast<const float4*>(row) + q);
        v[4 * q] = t4.x, v[4 * q + 1] = t4.y, v[4 * q + 2] = t4.z, v[4 * q + 3] = t4.w;
      }
#pragma unroll
      for (int c = 0; c < NG * 4; ++c) acc[c] = fa(acc[c], fm(w, v[c]));
      ws = fa(ws, w);
    };
    const int64_t bin = ((int64_t)m * L + l) * PV + pix;
    const int n = __ldg(cnt + bin), b0 = __ldg(off + bin);
    LVSG_CHECK(n >= 0 && b0 >= 0 && (int64_t)b0 + n <= n_ent);
    if (n <= 4) {
      int2 e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = k < n ? __ldg(ent + b0 + k) : make_int2(0x7fffffff, 0);
      sort4(e);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n) add(e[k]);
    } else if (n <= 8) {  // the sorting network again, in registers
      int2 e[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = k < n ? __ldg(ent + b0 + k) : make_int2(0x7fffffff, 0);
      sort8(e);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < n) add(e[k]);
    } else {
      int last = -1;  // ascending keys by repeated minimum search
      for (int r = 0; r < n; ++r) {
        int2 best = make_int2(0x7fffffff, 0);
        for (int j = 0; j < n; ++j) {
          const int2 ej = __ldg(ent + b0 + j);
          if (ej.x > last && ej.x < best.x) best = ej;
        }
        last = best.x;
        add(best);
      }
    }
    // splat_project: * 1/max(wsum, eps)
    const float nrm = __fdiv_rn(1.0f, ws > 1e-4f ? ws : 1e-4f);
    float4* dst = reinterpret_cast<float4*>(s_val + ((int64_t)lp * L + l) * NG * 4);
#pragma unroll
    for (int q = 0; q < NG; ++q)
      dst[q] = make_float4(fm(acc[4 * q], nrm), fm(acc[4 * q + 1], nrm), fm(acc[4 * q + 2], nrm),
                           fm(acc[4 * q + 3], nrm));
  }
  __syncthreads();
  // over_composite colour / alpha, layer 0 (far) first
  for (int u = threadIdx.x; u < ppb * NG; u += blockDim.x) {
    const int p = u / NG, g = u - p * NG;
    const int64_t tt = t0 + p;
    if (tt >= (int64_t)M * PV) break;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int ll = 0; ll < L; ++ll) {
      const float* vv = s_val + ((int64_t)p * L + ll) * NG * 4;
      const float s = vv[Ca];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = 4 * g + k;
        const float v = c < Ca ? vv[c] : 1.0f;
        o[k] = fa(fm(v, s), fm(fsb(1.0f, s), o[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * g + k >= K) o[k] = 0.f;
    reinterpret_cast<float4*>(out)[tt * NG + g] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// The same reduction with three lanes per (view pixel, layer): each lane
// sums 12 of the 36 payload channels (three 16-byte loads per entry), so a
// warp's loads of an entry's row are one contiguous 144-byte run instead of
// 32 lanes each fetching its own row. The run is sorted by each of the three
// lanes (the same network), and every channel is accumulated in the same
// sorted order as splat_reduce_pl_kernel: identical sums.
template <int NL>
__global__ void __launch_bounds__(192) splat_reduce_pl3_kernel(
    const float* __restrict__ payload, int K, int M, int L, int Hv, int Wv,
    const int* __restrict__ off, const int* __restrict__ cnt, const int2* __restrict__ ent,
    float* __restrict__ out, int ppb, int64_t n_ent, int64_t P) {
  pdl_grid_sync();
  constexpr int NG = 9, CL = 36 / NL, NQ = CL / 4;  // 36 channels, CL per lane
  extern __shared__ float s_val[];  // [ppb][L][36]: normalised channels, [Ca] = alpha
  const int64_t PV = (int64_t)Hv * Wv;
  const int Ca = K - 1;
  const int GP = payload_stride(K) / 4;  // float4 per payload row
  const int64_t t0 = (int64_t)blockIdx.x * ppb;
  const int part = threadIdx.x % NL, bt = threadIdx.x / NL;
  const int lp = bt / L, l = bt - lp * L;
  const int64_t t = t0 + lp;
  if (lp < ppb && t < (int64_t)M * PV) {
    const int64_t pix = t % PV;
    const int m = int(t / PV);
    float acc[CL];
#pragma unroll
    for (int c = 0; c < CL; ++c) acc[c] = 0.f;
    float ws = 0.f;
    auto add = [&](const int2 en) {
      const float w = __int_as_float(en.y);
      LVSG_CHECK(en.x >= 0 && (en.x >> 2) < P);
      const float4* row = reinterpret_cast<const float4*>(payload) + (int64_t)(en.x >> 2) * GP + NQ * part;
      float v[CL];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 t4 = __ldg(row + q);
        v[4 * q] = t4.x, v[4 * q + 1] = t4.y, v[4 * q + 2] = t4.z, v[4 * q + 3] = t4.w;
      }
#pragma unroll
      for (int c = 0; c < CL; ++c) acc[c] = fa(acc[c], fm(w, v[c]));
      ws = fa(ws, w);
    };
    const int64_t bin = ((int64_t)m * L + l) * PV + pix;
    const int n = __ldg(cnt + bin), b0 = __ldg(off + bin);
    LVSG_CHECK(n >= 0 && b0 >= 0 && (int64_t)b0 + n <= n_ent);
    if (n <= 4) {
      int2 e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = k < n ? __ldg(ent + b0 + k) : make_int2(0x7fffffff, 0);
      sort4(e);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n) add(e[k]);
    } else if (n <= 8) {
      int2 e[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = k < n ? __ldg(ent + b0 + k) : make_int2(0x7fffffff, 0);
      sort8(e);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < n) add(e[k]);
    } else {
      int last = -1;  // ascending keys by repeated minimum search
      for (int r = 0; r < n; ++r) {
        int2 best = make_int2(0x7fffffff, 0);
        for (int j = 0; j < n; ++j) {
          const int2 ej = __ldg(ent + b0 + j);
          if (ej.x > last && ej.x < best.x) best = ej;
        }
        last = best.x;
        add(best);
      }
    }
    const float nrm = __fdiv_rn(1.0f, ws > 1e-4f ? ws : 1e-4f);
    float4* dst = reinterpret_cast<float4*>(s_val + ((int64_t)lp * L + l) * NG * 4) + NQ * part;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      dst[q] = make_float4(fm(acc[4 * q], nrm), fm(acc[4 * q + 1], nrm), fm(acc[4 * q + 2], nrm),
                           fm(acc[4 * q + 3], nrm));
  }
  __syncthreads();
  // over_composite colour / alpha, layer 0 (far) first
  for (int u = threadIdx.x; u < ppb * NG; u += blockDim.x) {
    const int p = u / NG, g = u - p * NG;
    const int64_t tt = t0 + p;
    if (tt >= (int64_t)M * PV) break;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int ll = 0; ll < L; ++ll) {
      const float* vv = s_val + ((int64_t)p * L + ll) * NG * 4;
      const float s = vv[Ca];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = 4 * g + k;
        const float v = c < Ca ? vv[c] : 1.0f;
        o[k] = fa(fm(v, s), fm(fsb(1.0f, s), o[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (4 * g + k >= K) o[k] = 0.f;
    reinterpret_cast<float4*>(out)[tt * NG + g] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

inline int blocks_for(int64_t n, int t) { return int((n + t - 1) / t); }

}  // namespace

size_t splat_det_scratch_ints(int64_t pairs, int64_t bins) {
  const int64_t nb = (bins + kScanBlock - 1) / kScanBlock;
  // cnt, off [bins]; block sums; entries (int2) [4 pairs]; fp_i (int2),
  // fp_w (float4) and tap ranks (int4) [pairs]
  return size_t(2 * bins + nb + 8 * pairs + 2 * pairs + 4 * pairs + 4 * pairs + 16);
}

void splat_det(const float* payload, const float* points, int L, int PL, int K,
               const DevCam* cams_dev, int M, int Hv, int Wv, int* scratch, float* out,
               cudaStream_t st) {
  const int64_t pairs = (int64_t)L * PL * M;
  const int64_t bins = (int64_t)M * L * Hv * Wv;
  const int nb = int((bins + kScanBlock - 1) / kScanBlock);
  int* cnt = scratch;
  int* off = cnt + bins;
  int* bsum = off + bins;
  // 16-byte alignment for the int2 / float4 / int4 records
  uintptr_t a = reinterpret_cast<uintptr_t>(bsum + nb);
  a = (a + 15) & ~uintptr_t(15);
  float4* fp_w = reinterpret_cast<float4*>(a);
  int4* rank = reinterpret_cast<int4*>(fp_w + pairs);
  int2* ent = reinterpret_cast<int2*>(rank + pairs);
  int2* fp_i = ent + 4 * pairs;
  cudaMemsetAsync(cnt, 0, size_t(bins) * sizeof(int), st);  // errors surface at the caller's check
  launch_k(splat_count_kernel, blocks_for(pairs, 256), 256, 0, st, points, L, PL, cams_dev, M, Hv,
           Wv, cnt, fp_i, fp_w, rank);
  launch_k(scan_blocks_kernel, nb, 256, 0, st, (const int*)cnt, int(bins), off, bsum);
  launch_k(scan_sums_kernel, 1, 1024, 0, st, bsum, nb);
  launch_k(scan_add_kernel, nb, 256, 0, st, off, int(bins), (const int*)bsum);
  launch_k(splat_fill_kernel, blocks_for(pairs, 256), 256, 0, st, pairs, bins, M, (const int2*)fp_i,
           (const float4*)fp_w, (const int4*)rank, (const int*)off, ent);
  const int G = pay_stride(K) / 4;
  if (G == 9 && L <= 192 / LVSG_SPLAT_PL3 && LVSG_SPLAT_PL3) {  // C = 32: lanes per (view pixel, layer)
    constexpr int NL = LVSG_SPLAT_PL3 > 0 ? LVSG_SPLAT_PL3 : 1;
    const int ppb = std::max(1, 192 / NL / L);
    const size_t smem = size_t(ppb) * L * 36 * sizeof(float);
    launch_k(splat_reduce_pl3_kernel<NL>, blocks_for((int64_t)M * Hv * Wv, ppb), NL * ppb * L, smem, st,
             payload, K, M, L, Hv, Wv, (const int*)off, (const int*)cnt, (const int2*)ent, out, ppb,
             4 * pairs, pairs / M);
    return;
  }
  if (G == 9 && L <= 192) {  // C = 32 configs: one thread per (view pixel, layer)
    const int ppb = std::max(1, 192 / L);
    const size_t smem = size_t(ppb) * L * 36 * sizeof(float);
    smem_optin(reinterpret_cast<const void*>(splat_reduce_pl_kernel<9>), 192 * 36 * 4);
    launch_k(splat_reduce_pl_kernel<9>, blocks_for((int64_t)M * Hv * Wv, ppb), ppb * L, smem, st,
             payload, K, M, L, Hv, Wv, (const int*)off, (const int*)cnt, (const int2*)ent, out, ppb,
             4 * pairs, pairs / M);
    return;
  }
  const int ppb = std::max(1, std::min(kRedPixMax, 288 / G));
  launch_k(splat_reduce_composite_kernel, blocks_for((int64_t)M * Hv * Wv, ppb), ppb * G, 0, st,
           payload, K, M, L, Hv, Wv, (const int*)off, (const int*)cnt, (const int2*)ent, out, ppb,
           4 * pairs, pairs / M);
}

}  // namespace lvsg
