// Stage 1 gather (backproject_stack, network.hpp:421-436; gather_backproject,
// geometry.hpp:138-224) for C = 32, staged through shared memory.
//
// The per-(texel, view) footprints of a 4 x 64 texel tile of one layer land
// in a compact window of view m's feature map (the rig views see the target
// frustum at about the texel scale: a texel row maps onto one or two feature
// rows, neighbouring texels onto neighbouring pixels). The CTA computes the
// 256 footprints (f64, the gather's bit-exact rule), reduces their bounding
// box, and brings the window in with one bulk async copy per feature row
// (cp.async.bulk: L2 -> shared memory without the L1 load pipeline). The
// 4-tap blends then read 128-byte pixel rows from shared memory, 8 lanes per
// texel so each quarter-warp reads one whole row (conflict-free). A window
// larger than kTileCap pixels (depth discontinuities, grazing views) falls
// back to the same blend on global loads. Values and the view-major SoA Δ
// layout [M][8][P][4] are those of gather_stack32_kernel, bit for bit.
//
// Why: the global-load version is bound by L1 data-pipe wavefronts (one per
// 32-byte sector of each of the four taps, ~94% of peak on the largest
// step, profiles/); from shared memory a tap row costs one wavefront per
// quarter-warp.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "tc.cuh"

namespace lvsg {
namespace {

using namespace tc;

constexpr int kTileW = 64, kTileH = 4;     // texels per CTA tile (one layer)
constexpr int kTileCap = 640;              // window pixels staged (80 KB)

__global__ void __launch_bounds__(256, 2) gather_tile32_kernel(
    const float* __restrict__ feats, int M, int Hf, int Wf, const DevCam* __restrict__ cams,
    DevRayCam rc, const float* __restrict__ depth, int L, int H, int W, float* __restrict__ deltas) {
  constexpr int G = 8;
  extern __shared__ __align__(128) float4 s_win[];  // [kTileCap][8]
  __shared__ uint64_t s_bar;
  __shared__ int s_box[4][8];
  pdl_grid_sync();
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int m = blockIdx.z;
  const int l = blockIdx.y / ((H + kTileH - 1) / kTileH);
  const int ty = blockIdx.y - l * ((H + kTileH - 1) / kTileH);
  const int ii = ty * kTileH + t / kTileW, j = blockIdx.x * kTileW + t % kTileW;
  const int64_t P = (int64_t)L * H * W;
  // per-texel record: flags (1 valid | 2 x1>x0 | 4 y1>y0 | 8 outside), tap
  // 00 pixel, weights
  int flags = 8, x0 = 0, y0 = 0, pl = 0;
  float w[4] = {0.f, 0.f, 0.f, 0.f};
  if (ii < H && j < W) {
    pl = int(((int64_t)l * H + ii) * W + j);
    flags = 0;
    float pt[3];
    world_point(rc, ii, j, __ldg(depth + pl), pt);
    const Footprint f = project_footprint(cams[m], pt);
    if (f.valid) {
      double wd[4];
      bilinear_weights(f, wd);
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = __double2float_rn(wd[k]);
      flags = 1 | (f.x1 > f.x0 ? 2 : 0) | (f.y1 > f.y0 ? 4 : 0);
      x0 = f.x0;
      y0 = f.y0;
    }
  }
  // bounding box of the valid footprints (x1 <= x0 + 1, y1 <= y0 + 1)
  const bool v = flags & 1;
  int bx0 = __reduce_min_sync(0xffffffffu, v ? x0 : 0x7fffffff);
  int by0 = __reduce_min_sync(0xffffffffu, v ? y0 : 0x7fffffff);
  int bx1 = __reduce_max_sync(0xffffffffu, v ? x0 + ((flags >> 1) & 1) : -1);
  int by1 = __reduce_max_sync(0xffffffffu, v ? y0 + ((flags >> 2) & 1) : -1);
  if (lane == 0) {
    s_box[0][wid] = bx0;
    s_box[1][wid] = by0;
    s_box[2][wid] = bx1;
    s_box[3][wid] = by1;
  }
  if (t == 0) {
    mbar_init(&s_bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  bx0 = s_box[0][0], by0 = s_box[1][0], bx1 = s_box[2][0], by1 = s_box[3][0];
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    bx0 = min(bx0, s_box[0][k]);
    by0 = min(by0, s_box[1][k]);
    bx1 = max(bx1, s_box[2][k]);
    by1 = max(by1, s_box[3][k]);
  }
  const int bw = bx1 - bx0 + 1, bh = by1 - by0 + 1;
  const bool staged = bx1 >= 0 && bw * bh <= kTileCap;
  const float4* f4 = reinterpret_cast<const float4*>(feats);
  if (staged) {
    if (t == 0) {
      mbar_expect_tx(&s_bar, uint32_t(bw * bh * 128));
      for (int r = 0; r < bh; ++r)
        bulk_load(smem_u32(s_win + r * bw * G),
                  f4 + ((int64_t)(m * Hf + by0 + r) * Wf + bx0) * G, uint32_t(bw * 128), &s_bar);
    }
    mbar_wait(&s_bar, 0);
  }
  // tap-00 offset in float4 units: window-relative when staged
  const int off = staged ? ((y0 - by0) * bw + (x0 - bx0)) * G : ((m * Hf + y0) * Wf + x0) * G;
  const int dyw = (staged ? bw : Wf) * G;
  const float4* src = staged ? s_win : f4;
  float4* o4 = reinterpret_cast<float4*>(deltas);
  const int g = lane & 7;
#pragma unroll 2
  for (int it = 0; it < 8; ++it) {
    const int r = 4 * it + (lane >> 3);
    const int rf = __shfl_sync(0xffffffffu, flags, r);
    const int rp = __shfl_sync(0xffffffffu, pl, r);
    const int ro = __shfl_sync(0xffffffffu, off, r) + g;
    float rw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rw[k] = __shfl_sync(0xffffffffu, w[k], r);
    if (rf & 8) continue;
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rf & 1) {
      const int dx = (rf & 2) ? G : 0, dy = (rf & 4) ? dyw : 0;
      float4 a, b, c, d;
      if (staged) {
        a = src[ro];
        b = src[ro + dx];
        c = src[ro + dy];
        d = src[ro + dy + dx];
      } else {
        a = __ldg(src + ro);
        b = __ldg(src + ro + dx);
        c = __ldg(src + ro + dy);
        d = __ldg(src + ro + dy + dx);
      }
      val.x = fmaf(rw[3], d.x, fmaf(rw[2], c.x, fmaf(rw[1], b.x, rw[0] * a.x)));
      val.y = fmaf(rw[3], d.y, fmaf(rw[2], c.y, fmaf(rw[1], b.y, rw[0] * a.y)));
      val.z = fmaf(rw[3], d.z, fmaf(rw[2], c.z, fmaf(rw[1], b.z, rw[0] * a.z)));
      val.w = fmaf(rw[3], d.w, fmaf(rw[2], c.w, fmaf(rw[1], b.w, rw[0] * a.w)));
    }
    o4[((int64_t)m * G + g) * P + rp] = val;
  }
}

// Persistent, double-buffered variant: each CTA walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ...; while tile k is blended from one window
// buffer, tile k+1's footprints are computed and its window is already in
// flight into the other (bulk copies complete on that buffer's mbarrier).
constexpr int kPipeCap = 448;  // window pixels per buffer (56 KB); 2 buffers per CTA

struct TileRec {
  int flags, x0, y0, pl;
  float w[4];
};

__device__ __forceinline__ TileRec tile_footprint(const DevCam* __restrict__ cams, const DevRayCam& rc,
                                                  const float* __restrict__ depth, int m, int l,
                                                  int ty, int tx, int H, int W) {
  const int t = threadIdx.x;
  const int ii = ty * kTileH + t / kTileW, j = tx * kTileW + t % kTileW;
  TileRec r{8, 0, 0, 0, {0.f, 0.f, 0.f, 0.f}};
  if (ii < H && j < W) {
    r.pl = int(((int64_t)l * H + ii) * W + j);
    r.flags = 0;
    float pt[3];
    world_point(rc, ii, j, __ldg(depth + r.pl), pt);
    const Footprint f = project_footprint(cams[m], pt);
    if (f.valid) {
      double wd[4];
      bilinear_weights(f, wd);
#pragma unroll
      for (int k = 0; k < 4; ++k) r.w[k] = __double2float_rn(wd[k]);
      r.flags = 1 | (f.x1 > f.x0 ? 2 : 0) | (f.y1 > f.y0 ? 4 : 0);
      r.x0 = f.x0;
      r.y0 = f.y0;
    }
  }
  return r;
}

// Block-wide bounding box of the valid footprints (all threads get it).
// s_box must not be in use by another reduction of the same block.
__device__ __forceinline__ int4 tile_bbox(const TileRec& r, int (*s_box)[8]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool v = r.flags & 1;
  int bx0 = __reduce_min_sync(0xffffffffu, v ? r.x0 : 0x7fffffff);
  int by0 = __reduce_min_sync(0xffffffffu, v ? r.y0 : 0x7fffffff);
  int bx1 = __reduce_max_sync(0xffffffffu, v ? r.x0 + ((r.flags >> 1) & 1) : -1);
  int by1 = __reduce_max_sync(0xffffffffu, v ? r.y0 + ((r.flags >> 2) & 1) : -1);
  if (lane == 0) {
    s_box[0][wid] = bx0;
    s_box[1][wid] = by0;
    s_box[2][wid] = bx1;
    s_box[3][wid] = by1;
  }
  __syncthreads();
  bx0 = s_box[0][0], by0 = s_box[1][0], bx1 = s_box[2][0], by1 = s_box[3][0];
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    bx0 = min(bx0, s_box[0][k]);
    by0 = min(by0, s_box[1][k]);
    bx1 = max(bx1, s_box[2][k]);
    by1 = max(by1, s_box[3][k]);
  }
  return make_int4(bx0, by0, bx1, by1);
}

__global__ void __launch_bounds__(256, 2) gather_pipe32_kernel(
    const float* __restrict__ feats, int M, int Hf, int Wf, const DevCam* __restrict__ cams,
    DevRayCam rc, const float* __restrict__ depth, int L, int H, int W, float* __restrict__ deltas,
    int tiles_x, int tiles_y, int ntiles) {
  constexpr int G = 8;
  extern __shared__ __align__(128) float4 s_buf[];  // [2][kPipeCap][8]
  __shared__ uint64_t s_bar[2];
  __shared__ int s_box[2][4][8];
  pdl_grid_sync();
  const int t = threadIdx.x, lane = t & 31;
  const int64_t P = (int64_t)L * H * W;
  const float4* f4 = reinterpret_cast<const float4*>(feats);
  float4* o4 = reinterpret_cast<float4*>(deltas);
  if (t == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  auto decode = [&](int k, int& m, int& l, int& ty, int& tx) {
    tx = k % tiles_x;
    int r = k / tiles_x;
    ty = r % tiles_y;
    r /= tiles_y;
    l = r % L;
    m = r / L;
  };
  // stage tile k into buffer b: footprints, bbox, bulk copies; returns the
  // record and whether the window is staged (all threads agree)
  auto stage = [&](int k, int b, TileRec& rec, int4& box, int& mm) -> bool {
    int l, ty, tx;
    decode(k, mm, l, ty, tx);
    rec = tile_footprint(cams, rc, depth, mm, l, ty, tx, H, W);
    box = tile_bbox(rec, s_box[b]);
    const int bw = box.z - box.x + 1, bh = box.w - box.y + 1;
    const bool staged = box.z >= 0 && bw * bh <= kPipeCap;
    if (staged && t == 0) {
      float4* dst = s_buf + b * kPipeCap * G;
      fence_proxy_async();  // the buffer's earlier generic-proxy reads before the async writes
      mbar_expect_tx(&s_bar[b], uint32_t(bw * bh * 128));
      for (int r = 0; r < bh; ++r)
        bulk_load(smem_u32(dst + r * bw * G), f4 + ((int64_t)(mm * Hf + box.y + r) * Wf + box.x) * G,
                  uint32_t(bw * 128), &s_bar[b]);
    }
    return staged;
  };
  int k = blockIdx.x, b = 0;
  uint32_t phase[2] = {0, 0};
  TileRec rec;
  int4 box;
  int m = 0;
  bool staged = k < ntiles ? stage(k, 0, rec, box, m) : false;
  while (k < ntiles) {
    const int kn = k + gridDim.x;
    TileRec nrec;
    int4 nbox;
    int nm = 0;
    bool nstaged = false;
    if (kn < ntiles) nstaged = stage(kn, b ^ 1, nrec, nbox, nm);
    if (staged) {
      mbar_wait(&s_bar[b], phase[b]);
      phase[b] ^= 1;
    }
    const int bw = box.z - box.x + 1;
    const int off = staged ? ((rec.y0 - box.y) * bw + (rec.x0 - box.x)) * G
                           : ((m * Hf + rec.y0) * Wf + rec.x0) * G;
    const int dyw = (staged ? bw : Wf) * G;
    const float4* src = staged ? s_buf + b * kPipeCap * G : f4;
    const int g = lane & 7;
#pragma unroll 2
    for (int it = 0; it < 8; ++it) {
      const int r = 4 * it + (lane >> 3);
      const int rf = __shfl_sync(0xffffffffu, rec.flags, r);
      const int rp = __shfl_sync(0xffffffffu, rec.pl, r);
      const int ro = __shfl_sync(0xffffffffu, off, r) + g;
      float rw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) rw[q] = __shfl_sync(0xffffffffu, rec.w[q], r);
      if (rf & 8) continue;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rf & 1) {
        const int dx = (rf & 2) ? G : 0, dy = (rf & 4) ? dyw : 0;
        float4 a, bb, c, d;
        if (staged) {
          a = src[ro];
          bb = src[ro + dx];
          c = src[ro + dy];
          d = src[ro + dy + dx];
        } else {
          a = __ldg(src + ro);
          bb = __ldg(src + ro + dx);
          c = __ldg(src + ro + dy);
          d = __ldg(src + ro + dy + dx);
        }
        val.x = fmaf(rw[3], d.x, fmaf(rw[2], c.x, fmaf(rw[1], bb.x, rw[0] * a.x)));
        val.y = fmaf(rw[3], d.y, fmaf(rw[2], c.y, fmaf(rw[1], bb.y, rw[0] * a.y)));
        val.z = fmaf(rw[3], d.z, fmaf(rw[2], c.z, fmaf(rw[1], bb.z, rw[0] * a.z)));
        val.w = fmaf(rw[3], d.w, fmaf(rw[2], c.w, fmaf(rw[1], bb.w, rw[0] * a.w)));
      }
      o4[((int64_t)m * G + g) * P + rp] = val;
    }
    __syncthreads();  // buffer b free for tile k + 2 gridDim
    k = kn;
    b ^= 1;
    rec = nrec;
    box = nbox;
    m = nm;
    staged = nstaged;
  }
}

}  // namespace

bool gather_tile32(const float* feats, int M, int Hf, int Wf, int C, const DevCam* cams_dev,
                   const DevRayCam& rc, const float* depth, int L, int H, int W, float* deltas,
                   cudaStream_t st) {
  if (C != 32 || (int64_t)M * Hf * Wf * 8 >= (int64_t(1) << 31) ||
      (int64_t)L * H * W >= (int64_t(1) << 31) ||
      (reinterpret_cast<uintptr_t>(feats) & 15) != 0)
    return false;
  static bool attr = [] {
    cudaFuncSetAttribute(gather_tile32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTileCap * 128);
    return true;
  }();
  (void)attr;
  static const int pipe = [] {  // LVSG_GATHER=tile1: the single-window (unpipelined) kernel
    const char* e = getenv("LVSG_GATHER");
    return !(e && e[0] == 't' && e[4] == '1');
  }();
  if (pipe) {
    static bool attr2 = [] {
      cudaFuncSetAttribute(gather_pipe32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           2 * kPipeCap * 128);
      return true;
    }();
    (void)attr2;
    const int tx = (W + kTileW - 1) / kTileW, ty = (H + kTileH - 1) / kTileH;
    const int ntiles = tx * ty * L * M;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = std::min(ntiles, 2 * sms);
    launch_k(gather_pipe32_kernel, grid, 256, 2 * kPipeCap * 128, st, feats, M, Hf, Wf, cams_dev, rc,
             depth, L, H, W, deltas, tx, ty, ntiles);
    return true;
  }
  const dim3 grid((W + kTileW - 1) / kTileW, L * ((H + kTileH - 1) / kTileH), M);
  launch_k(gather_tile32_kernel, grid, 256, kTileCap * 128, st, feats, M, Hf, Wf, cams_dev, rc,
           depth, L, H, W, deltas);
  return true;
}

}  // namespace lvsg
