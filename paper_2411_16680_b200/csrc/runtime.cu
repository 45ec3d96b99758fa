// liblvsg runtime: context (device weights, stream, scratch arena), the
// per-frame orchestration of forward() + render_target() on the device, and
// the C ABI of include/lvsg.h.
//
// Orchestration mirrors lvs::forward (network.hpp:562-603):
//   encode_inputs            network.hpp:368-417
//   initialize               network.hpp:459-493
//   layer_collapse           network.hpp:440-455
//   update_block             network.hpp:500-535
//   fusion_block             attention.hpp:275-281
//   decode_blend_logits      network.hpp:539-549
//   upsample_activate        ldm.hpp:249-271      (fused into the render)
//   render_target            ldm.hpp:193-199
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "host.h"
#include "kernels.h"

namespace lvsg {


namespace {

#define CUDA_OK(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                  \
  } while (0)

// ---- camera conversions (host, f64, reference operation order) -------------

DevCam dev_cam(const lvsg_camera& c) {
  DevCam d;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) d.R[i * 3 + j] = c.cam_from_world[i * 4 + j];
    d.t[i] = c.cam_from_world[i * 4 + 3];
  }
  d.fx = c.fx;
  d.fy = c.fy;
  d.cx = c.cx;
  d.cy = c.cy;
  d.W = int(c.width);
  d.H = int(c.height);
  d.wm = double(d.W) - 0.5;  // IEEE binary64 like the device's __dsub_rn / __dadd_rn
  d.hm = double(d.H) - 0.5;
  d.hu = d.wm + 1e-4;
  d.hv = d.hm + 1e-4;
  return d;
}

void center_of(const lvsg_camera& c, double o[3]) {
  const double* m = c.cam_from_world;
  for (int r = 0; r < 3; ++r) {
    double acc = (-m[0 * 4 + r]) * m[0 * 4 + 3];
    acc += (-m[1 * 4 + r]) * m[1 * 4 + 3];
    acc += (-m[2 * 4 + r]) * m[2 * 4 + 3];
    o[r] = acc;
  }
}

// world_points camera: the frustum camera re-digitised to (W, H).
DevRayCam ray_cam(const lvsg_camera& c0, int64_t W, int64_t H) {
  lvsg_camera c = camera_scaled(c0, W, H);
  DevRayCam r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.Rwc[i * 3 + j] = c.cam_from_world[j * 4 + i];
  center_of(c, r.c);
  r.fx = c.fx;
  r.fy = c.fy;
  r.cx = c.cx;
  r.cy = c.cy;
  return r;
}

DepthAct depth_act(int64_t L, const lvsg_frustum& fr) {
  DepthAct a;
  a.L = int(L);
  a.s_half_over_L = float(0.5 / double(L));
  a.s_span = float(1.0 / fr.near_depth - 1.0 / fr.far_depth);
  a.s_inv_far = float(1.0 / fr.far_depth);
  return a;
}

// ---- device arena ----------------------------------------------------------

struct Buf {
  float* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CUDA_OK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(float)));
    n = count;
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
};

struct ConvPairW {
  const float *w1, *b1, *w2, *b2;
};
struct MlpW {
  const float *gain, *w1, *b1, *w2, *b2;
};
struct FusionW {
  int heads;
  const float *wq, *wo, *gain;
  std::vector<MlpW> mlps;
};
struct StepW {
  std::vector<ConvPairW> collapse;  // w1 b1 w2 b2 of each Lc
  const float *stem_w = nullptr, *stem_b = nullptr;
  int64_t stem_cin = 0;
  ConvPairW r1{}, r2{};
  std::vector<FusionW> fusions;
};
struct NetW {
  const float* init_feature;
  const float *stem_w, *stem_b;
  std::vector<ConvPairW> lvl_r1, lvl_r2;
  std::vector<const float*> ray_proj;
  const float *w_sigma, *w_depth, *w_appear, *blend_w, *blend_gain;
  std::vector<StepW> steps;
};

}  // namespace
}  // namespace lvsg

namespace lvsg {
// One in-flight pipelined host frame: its device copies of the inputs and
// the output, the events that order them, its own depth-range flag.
struct FrameSlot {
  Buf enc_in, ren_in, rgb;
  std::vector<cudaEvent_t> ev_enc;
  cudaEvent_t ev_ren = nullptr, ev_free = nullptr, ev_done = nullptr;
  cudaEvent_t ev_band[4] = {};
  int* bad = nullptr;
  int64_t ticket = -1;  // frame owning the slot, -1 = free
};
}  // namespace lvsg

struct lvsg_ctx {
  lvsg::Config cfg;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  std::vector<lvsg::ParamSpec> layout;
  int64_t total_params = 0;
  lvsg::Buf weights;
  bool have_weights = false;
  lvsg::NetW W;

  // per-resolution plan
  int64_t He = 0, We = 0;
  lvsg::Plan plan;

  // arena
  lvsg::Buf enc_in, ren_in, rgb, enc_x, enc_t, ray_base;
  std::vector<lvsg::Buf> feats, rays;
  lvsg::Buf splat_scratch;  // deterministic splat: counts, runs, keys, footprints (ints)
  lvsg::Buf V0, V1, deltas, t1, rinv, uh, ut, uu, payload, depth_in, points, depth_out, fb,
      fbr, pre_d, pre_s, logits, anchors, ldm_d, ldm_s, ldm_b;
  lvsg::Buf cams_dev;  // DevCam / RayBaseCam tables
  int* bad_flag = nullptr;
  // where the forward's kernels report (atomicOr): bit 1 a depth outside the
  // frustum (render), bit 2 an fp16-split overflow (tensor-core operands) --
  // bad_flag, or the pipelined frame slot's flag while its frame is enqueued
  int* flag = nullptr;
  void* pinned = nullptr;  // camera staging
  size_t pinned_bytes = 0;
  cudaEvent_t staging_done = nullptr;
  // host-ABI transfers: a copy stream overlapping the render-view upload with
  // the forward pass and the output read-back with the banded render
  cudaStream_t xfer = nullptr;
  cudaEvent_t ev_main = nullptr, ev_ren = nullptr;
  cudaEvent_t ev_band[4] = {};
  std::vector<cudaEvent_t> ev_enc;  // per-view encoder upload landed
  // pipelined host frames (lvsg_submit_frame): two slots, a download stream
  lvsg::FrameSlot slots[2];
  cudaStream_t down = nullptr;
  int64_t next_ticket = 0;

  // resident forward result (for lvsg_render)
  bool have_ldm = false;
  int64_t L = 0, H = 0, Wd = 0, M = 0;
  lvsg_frustum target{};
  float* V = nullptr;
  int64_t launches = 0;      // kernels the last forward / render call launched
  int64_t launch_total = 0;  // every launch on this context (mark())

  // optional per-stage device timing (lvsg_profile_*): one event after each
  // group of launches; consecutive events bound that group's device time
  bool prof = false;
  int tl_next = -1;  // conv timeline (LVSG_TIMELINE debug builds): next slot, -1 off
  std::vector<cudaEvent_t> prof_pool;
  std::vector<const char*> prof_labels;
  std::vector<int> prof_counts;
  std::map<std::string, std::pair<double, int64_t>> prof_acc;

  // tensor-core conv weight images (conv3x3_tc_prepare), keyed by weight
  // tensor and input-channel slice; rebuilt whenever weights are (re)bound
  // (settled: made by an earlier forward call and synchronised since, so a
  // kernel may bulk-load it before its griddepcontrol.wait, under the
  // previous kernel's tail)
  struct WImg {
    lvsg::Buf buf;
    bool settled = false;
  };
  std::map<std::tuple<const float*, int, int>, std::unique_ptr<WImg>> wimg;
  bool wimg_fresh = false;  // an image was made during the current call
  lvsg::Buf wimg_tmp;  // uncached image for the stage entry points
  lvsg::Buf stage_a, stage_b, stage_c, stage_cams;  // scratch of the per-stage entry points
  lvsg::Buf attn_scratch;  // generic attention kernel rows (shapes without a tensor-core kernel)
  std::vector<float> stem_host;  // encoder stem weights [32*27] + bias [32] (host copy)
  std::vector<std::vector<float>> rayproj_host;  // per-level ray_proj [32, C] (host copies)
  std::vector<float> blendw_host;                // blend_w [C, C] (host copy)
  std::vector<float> decw_host;                  // decode heads [C][C+4] (host copy)
  int64_t pyr_He = -1, pyr_We = -1;  // encoder resolution of the resident feature pyramid
  // fused pyramid exchange: every peer's level buffers (CUDA IPC mappings)
  std::vector<std::vector<float*>> peer_feats;
  std::vector<void*> peer_maps;
};

namespace lvsg {
namespace {

thread_local std::string g_create_err;

// Counts `n` kernel launches under `label`; when profiling, records an event
// that closes the group on the context stream.
void mark(lvsg_ctx* c, const char* label, int n) {
  c->launch_total += n;  // per context: no shared counter across contexts / threads
  if (!c->prof) return;
  const size_t i = c->prof_labels.size();
  if (i >= c->prof_pool.size()) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreate(&e));
    c->prof_pool.push_back(e);
  }
  CUDA_OK(cudaEventRecord(c->prof_pool[i], c->stream));
  c->prof_labels.push_back(label);
  c->prof_counts.push_back(n);
}

// Folds the recorded events of the last frame into the accumulators.
void prof_collect(lvsg_ctx* c) {
  if (!c->prof || c->prof_labels.size() < 2) return;
  CUDA_OK(cudaEventSynchronize(c->prof_pool[c->prof_labels.size() - 1]));
  for (size_t i = 1; i < c->prof_labels.size(); ++i) {
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, c->prof_pool[i - 1], c->prof_pool[i]));
    auto& a = c->prof_acc[c->prof_labels[i]];
    a.first += ms;
    a.second += c->prof_counts[i];
  }
  c->prof_labels.clear();
  c->prof_counts.clear();
}

void bind_weights(lvsg_ctx* c) {
  c->wimg.clear();
  c->rayproj_host.clear();
  const Config& cfg = c->cfg;
  const int64_t C = cfg.channels, Ca = cfg.appear_channels();
  const float* cur = c->weights.p;
  auto take = [&](int64_t n) {
    const float* p = cur;
    cur += n;
    return p;
  };
  auto pair = [&] {
    ConvPairW p;
    p.w1 = take(C * C * 9);
    p.b1 = take(C);
    p.w2 = take(C * C * 9);
    p.b2 = take(C);
    return p;
  };
  NetW& W = c->W;
  W = NetW{};
  W.init_feature = take(C);
  W.stem_w = take(C * 27);
  W.stem_b = take(C);
  c->stem_host.assign(size_t(C * 27 + C), 0.f);
  CUDA_OK(cudaMemcpy(c->stem_host.data(), W.stem_w, size_t(C * 27) * sizeof(float), cudaMemcpyDeviceToHost));
  CUDA_OK(cudaMemcpy(c->stem_host.data() + C * 27, W.stem_b, size_t(C) * sizeof(float),
                     cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < cfg.pyramid_levels; ++k) {
    W.lvl_r1.push_back(pair());
    W.lvl_r2.push_back(pair());
    W.ray_proj.push_back(take(32 * C));
    c->rayproj_host.emplace_back(size_t(32 * C));
    CUDA_OK(cudaMemcpy(c->rayproj_host.back().data(), W.ray_proj.back(), size_t(32 * C) * sizeof(float),
                       cudaMemcpyDeviceToHost));
  }
  W.w_sigma = take(C);
  W.w_depth = take(C);
  W.w_appear = take(C * Ca);
  if (Ca == C) {  // the decode heads as [k][C+4] for the parameter-space kernel
    std::vector<float> wa(static_cast<size_t>(C * Ca)), ws(static_cast<size_t>(C)),
        wd(static_cast<size_t>(C));
    CUDA_OK(cudaMemcpy(wa.data(), W.w_appear, wa.size() * sizeof(float), cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(ws.data(), W.w_sigma, ws.size() * sizeof(float), cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(wd.data(), W.w_depth, wd.size() * sizeof(float), cudaMemcpyDeviceToHost));
    c->decw_host.assign(size_t(C * (C + 4)), 0.f);
    for (int64_t k = 0; k < C; ++k) {
      for (int64_t j = 0; j < C; ++j) c->decw_host[size_t(k * (C + 4) + j)] = wa[size_t(k * C + j)];
      c->decw_host[size_t(k * (C + 4) + C)] = ws[size_t(k)];
      c->decw_host[size_t(k * (C + 4) + C + 1)] = wd[size_t(k)];
    }
  } else {
    c->decw_host.clear();
  }
  W.blend_w = take(C * C);
  c->blendw_host.assign(size_t(C * C), 0.f);
  CUDA_OK(cudaMemcpy(c->blendw_host.data(), W.blend_w, size_t(C * C) * sizeof(float),
                     cudaMemcpyDeviceToHost));
  W.blend_gain = take(C);
  for (const Step& st : cfg.steps) {
    StepW sw;
    for (const Token& t : parse_blocks(st.blocks)) {
      switch (t.kind) {
        case Tok::collapse: {
          ConvPairW p;
          p.w1 = take(4 * C * C);
          p.b1 = take(2 * C);
          p.w2 = take(2 * C * C);
          p.b2 = take(C);
          sw.collapse.push_back(p);
          break;
        }
        case Tok::backproject:
        case Tok::update: {
          sw.stem_cin = t.kind == Tok::update ? 2 * C + Ca + 1 : 2 * C;
          sw.stem_w = take(C * sw.stem_cin * 9);
          sw.stem_b = take(C);
          sw.r1 = pair();
          sw.r2 = pair();
          break;
        }
        case Tok::attend: {
          FusionW f;
          f.heads = int(t.heads);
          f.wq = take(t.heads * C * C);
          f.wo = take(t.heads * C * C);
          f.gain = take(C);
          sw.fusions.push_back(f);
          break;
        }
        case Tok::conv: {
          MlpW m;
          m.gain = take(C);
          m.w1 = take(C * C * 9);
          m.b1 = take(C);
          m.w2 = take(C * C * 9);
          m.b2 = take(C);
          sw.fusions.back().mlps.push_back(m);
          break;
        }
      }
    }
    W.steps.push_back(std::move(sw));
  }
}

// Sizes every arena buffer for encoder input (He, We); no allocation after.
void ensure_plan(lvsg_ctx* c, int64_t He, int64_t We) {
  if (c->He == He && c->We == We) return;
  c->pyr_He = c->pyr_We = -1;  // buffers re-sized: no resident pyramid
  if (!c->peer_feats.empty())
    throw DimError("pyramid exchange: encoder resolution changed after lvsg_pyramid_import");
  const Config& cfg = c->cfg;
  Plan plan = plan_forward(cfg, He, We);
  const int64_t M = cfg.views, C = cfg.channels, Ca = cfg.appear_channels(), K = cfg.pyramid_levels;
  c->enc_x.ensure(size_t(M * He * We * C));
  c->enc_t.ensure(size_t(M * He * We * C));
  c->feats.resize(size_t(K));
  c->rays.resize(size_t(K));
  for (int64_t k = 0; k < K; ++k) {
    size_t n = size_t(M * plan.pyramid[size_t(k)].first * plan.pyramid[size_t(k)].second * C);
    c->feats[size_t(k)].ensure(n);
    c->rays[size_t(k)].ensure(n);
  }
  c->ray_base.ensure(size_t(M * plan.pyramid.back().first * plan.pyramid.back().second * 32));
  size_t maxV = 0, maxD = 0, maxU = 0, maxFb = 0, maxIn = 0, maxSplat = 0;
  for (const StepPlan& sp : plan.steps) {
    maxV = std::max({maxV, size_t(sp.in_layers * sp.in_height * sp.in_width),
                     size_t(sp.layers * sp.height * sp.width)});
    maxIn = std::max(maxIn, size_t(sp.layers * sp.in_height * sp.in_width));
    // Δ texel-major per view [M][P][C]
    maxD = std::max(maxD, size_t(sp.layers * sp.height * sp.width * M * C));
    maxU = std::max(maxU, size_t(M * sp.feat_h * sp.feat_w));
    // deterministic splat over the volume entering the step (at most
    // max(in_layers, layers) x in_height x in_width texels, all views):
    // bins = views x layers x render pixels
    const int64_t Ls = std::max(sp.in_layers, sp.layers);
    maxSplat = std::max(maxSplat, splat_det_scratch_ints(M * Ls * sp.in_height * sp.in_width,
                                                         M * Ls * sp.render_h * sp.render_w));
    maxFb = std::max(maxFb, size_t(M * sp.render_h * sp.render_w * pay_stride(int(Ca) + 1)));
  }
  c->V0.ensure(maxV * C);
  c->V1.ensure(maxV * C);
  c->deltas.ensure(maxD + 128);  // slack: attention's Δ boxes may read a partial row past the end
  c->t1.ensure(maxV * C);
  c->rinv.ensure(maxV);
  c->uh.ensure(maxU * C);
  c->ut.ensure(maxU * C);
  c->uu.ensure(maxU * C);
  c->payload.ensure(maxIn * payload_stride(int(Ca) + 1));
  c->depth_in.ensure(maxIn);
  c->points.ensure(maxIn * 3);
  c->depth_out.ensure(maxV);
  c->splat_scratch.ensure(maxSplat);
  c->fb.ensure(maxFb);
  c->fbr.ensure(maxU * pay_stride(int(Ca) + 1));
  const StepPlan& last = plan.steps.back();
  const size_t Pf = size_t(last.layers * last.height * last.width);
  c->pre_d.ensure(Pf);
  c->pre_s.ensure(Pf);
  c->logits.ensure(Pf * M);
  int64_t maxL = 0;
  for (const Step& s : cfg.steps) maxL = std::max(maxL, s.layers);
  c->anchors.ensure(size_t(maxL));
  // camera tables: per step (update cams + render cams) + ray base cams
  size_t cam_bytes = (plan.steps.size() * 2 + 2) * size_t(M) * sizeof(DevCam) + size_t(M) * sizeof(RayBaseCam);
  c->cams_dev.ensure((cam_bytes + sizeof(float) - 1) / sizeof(float));
  if (c->pinned_bytes < cam_bytes) {
    if (c->pinned) cudaFreeHost(c->pinned);
    CUDA_OK(cudaMallocHost(&c->pinned, cam_bytes));
    c->pinned_bytes = cam_bytes;
  }
  c->plan = std::move(plan);
  c->He = He;
  c->We = We;
}

ConvArgs conv_args(int B, int H, int W, int Cin, int Cout, const float* w, const float* b,
                   float* out) {
  ConvArgs a;
  std::memset(&a, 0, sizeof(a));
  a.B = B;
  a.H = H;
  a.W = W;
  a.Cin = Cin;
  a.Cout = Cout;
  a.w = w;
  a.bias = b;
  a.out = out;
  a.out_pstride = Cout;
  a.out_bstride = (long long)H * W * Cout;
  return a;
}

// LVSG_COLLAPSE=simt keeps the per-texel MLPs (layer collapse, ray
// projection) on the fp32 SIMT kernels (A/B and parity comparisons).
bool collapse_simt() {
  static const bool on = [] {
    const char* e = getenv("LVSG_COLLAPSE");
    return e && e[0] == 's';
  }();
  return on;
}

// Weight images made during this call become "settled" once the stream has
// drained them (one synchronisation, on the first frame after a weight
// binding): from then on kernels may bulk-load them before
// griddepcontrol.wait, overlapping the previous kernel.
void settle_images(lvsg_ctx* c) {
  if (!c->wimg_fresh) return;
  CUDA_OK(cudaStreamSynchronize(c->stream));
  for (auto& kv : c->wimg) kv.second->settled = true;
  c->wimg_fresh = false;
}

// conv3x3 through the dispatcher; a tensor-core launch gets its weight image
// from the context cache (cached = true: weights bound to the context) or a
// fresh one in scratch (stage entry points: arbitrary caller weights).
void run_conv(lvsg_ctx* c, ConvArgs a, cudaStream_t st, int impl = 0, bool cached = true) {
  a.ovf = c->flag;
  if (c->tl_next >= 0) a.tl_slot = ++c->tl_next;
  const int path = conv3x3_path(a, impl);
  if (path >= 2) {
    const size_t nf = kConvTcWeightBytes / sizeof(float);
    auto prepare = [&](void* dst) { conv3x3_tc_prepare(a, dst, st); };
    if (cached) {
      auto key = std::make_tuple(a.w, w_cin_of(a), a.w_ci0);
      auto it = c->wimg.find(key);
      a.pdl = 1;
      if (it == c->wimg.end()) {
        auto img = std::make_unique<lvsg_ctx::WImg>();
        img->buf.ensure(nf);
        prepare(img->buf.p);
        it = c->wimg.emplace(key, std::move(img)).first;
        c->wimg_fresh = true;
      }
      a.wsplit = it->second->buf.p;
      a.w_early = it->second->settled ? 1 : 0;
    } else {
      c->wimg_tmp.ensure(nf);
      prepare(c->wimg_tmp.p);
      a.wsplit = c->wimg_tmp.p;
    }
  }
  conv3x3(a, st, impl);
}

void add_src(ConvArgs& a, const float* p, int C, int H, int W) {
  a.src[a.nsrc] = ConvSrc{p, C, C, (long long)H * W * C};
  a.nsrc++;
}

// x = x + conv(gelu(conv(x))) on [B,H,W,C] (network.hpp:150-153); with
// `out` != x the sum lands in out (x untouched).
// pool_out (optional): also the 2x2 mean pool of the result ([B,H/2,W/2,C]),
// fused into the second conv's epilogue on the tensor-core path.
void conv_residual(lvsg_ctx* c, const float* x, float* out, float* tmp, int B, int H, int W,
                   const ConvPairW& p, float* pool_out = nullptr,
                   const std::vector<float*>* pool_peers = nullptr) {
  const int C = int(c->cfg.channels);
  ConvArgs a = conv_args(B, H, W, C, C, p.w1, p.b1, tmp);
  add_src(a, x, C, H, W);
  a.gelu = 1;
  run_conv(c, a, c->stream);
  ConvArgs b2 = conv_args(B, H, W, C, C, p.w2, p.b2, out);
  add_src(b2, tmp, C, H, W);
  b2.resid = x;
  b2.res_pstride = C;
  b2.res_bstride = (long long)H * W * C;
  const bool fuse_pool = pool_out && conv3x3_path(b2) == 2;
  if (pool_peers && !pool_peers->empty() && !fuse_pool)
    throw CudaError("pyramid exchange: needs the fused-pool tensor-core conv");
  if (fuse_pool) {
    b2.pool_out = pool_out;
    b2.pool_bstride = (long long)(H / 2) * (W / 2) * C;
    if (pool_peers) {
      b2.npool_peer = int(pool_peers->size());
      for (size_t q = 0; q < pool_peers->size(); ++q) b2.pool_peer[q] = (*pool_peers)[q];
    }
  }
  run_conv(c, b2, c->stream);
  mark(c, "conv", 2);
  if (pool_out && !fuse_pool) {
    mean_pool2(out, pool_out, B, H, W, C, c->stream);
    mark(c, "misc", 1);
  }
}

// run_update_cnn (network.hpp:155-160) on concatenated sources, all views.
void update_cnn(lvsg_ctx* c, const StepW& sw, const ConvArgs& stem_in, int M, int Hf, int Wf) {
  const int C = int(c->cfg.channels);
  ConvArgs a = stem_in;
  a.w = sw.stem_w;
  a.bias = sw.stem_b;
  a.Cin = int(sw.stem_cin);
  a.Cout = C;
  a.B = M;
  a.H = Hf;
  a.W = Wf;
  a.out = c->uh.p;
  a.out_pstride = C;
  a.out_bstride = (long long)Hf * Wf * C;
  a.w_cin = a.Cin;
  a.w_ci0 = 0;
  // By linearity the stem over concat(sources) is the sum of one conv per
  // source over its weight slice: each 32-channel source runs on the tensor
  // core, leftovers (the feedback's alpha channel) on the SIMT kernel, all
  // accumulating into uh (the first one adds the bias).
  bool split = C == 32;
  std::vector<ConvArgs> parts;
  if (split) {
    int ci0 = 0;
    for (int s = 0; s < a.nsrc && split; ++s) {
      const ConvSrc& S = a.src[s];
      for (int c0 = 0; c0 < S.C; c0 += 32) {
        const int cn = std::min(32, S.C - c0);
        if (cn == 1 && !parts.empty() && parts.back().src[0].ptr == S.ptr + c0 - 32 &&
            conv3x3_path(parts.back()) == 2) {
          // a trailing single channel (the feedback's alpha) folds into the
          // previous tensor-core part's epilogue instead of its own launch
          ConvArgs& q = parts.back();
          q.alpha = S.ptr + c0;
          q.alpha_pstride = int(S.pstride);
          q.alpha_bstride = S.bstride;
          q.alpha_ci = ci0 + c0;
          continue;
        }
        ConvArgs p = conv_args(M, Hf, Wf, cn, C, sw.stem_w, parts.empty() ? sw.stem_b : nullptr, c->uh.p);
        p.src[0] = ConvSrc{S.ptr + c0, cn, S.pstride, S.bstride};
        p.nsrc = 1;
        p.w_cin = a.Cin;
        p.w_ci0 = ci0 + c0;
        if (!parts.empty()) {
          p.resid = c->uh.p;
          p.res_pstride = C;
          p.res_bstride = (long long)Hf * Wf * C;
        }
        if (cn == 32 && !conv3x3_uses_tc(p)) split = false;
        parts.push_back(p);
      }
      ci0 += S.C;
    }
  }
  if (split) {
    for (const ConvArgs& p : parts) run_conv(c, p, c->stream);
    mark(c, "conv", int(parts.size()));
  } else {
    run_conv(c, a, c->stream);
    mark(c, "conv", 1);
  }
  conv_residual(c, c->uh.p, c->uh.p, c->ut.p, M, Hf, Wf, sw.r1);
  conv_residual(c, c->uh.p, c->uu.p, c->ut.p, M, Hf, Wf, sw.r2);
}

// fusion_block (attention.hpp:275-281): attention + conv MLPs, V in place.
void fusion(lvsg_ctx* c, float* V, int64_t L, int64_t H, int64_t W, const FusionW& f) {
  const int C = int(c->cfg.channels), M = int(c->cfg.views);
  const int64_t P = L * H * W;
  // the generic kernel's scratch (none for the tensor-core shapes) grows
  // the arena once, on the first frame of a plan
  c->attn_scratch.ensure(attend_scratch_floats(P, C, M, f.heads));
  // the tensor-core kernel's pre-split weight image, made once per binding
  const void* wimg = nullptr;
  bool wimg_early = false;
  if (const size_t nb = C == 32 ? attend_tc_weight_bytes(f.heads) : 0) {
    auto key = std::make_tuple(f.wq, -f.heads, 0);
    auto it = c->wimg.find(key);
    if (it == c->wimg.end()) {
      auto img = std::make_unique<lvsg_ctx::WImg>();
      img->buf.ensure((nb + 3) / 4);
      attend_tc_prepare(f.wq, f.wo, f.heads, img->buf.p, c->flag, c->stream);
      it = c->wimg.emplace(key, std::move(img)).first;
      c->wimg_fresh = true;
    }
    wimg = it->second->buf.p;
    wimg_early = it->second->settled;
  }
  attend(V, c->deltas.p, P, C, M, f.heads, f.wq, nullptr, f.wo, f.gain, c->cfg.ablate_attention,
         c->attn_scratch.p, wimg, wimg_early, c->flag, c->stream);
  mark(c, "attention", 1);
  for (const MlpW& m : f.mlps) {
    // conv_mlp_residual (attention.hpp:262-267), batched over layers
    ConvArgs a = conv_args(int(L), int(H), int(W), C, C, m.w1, m.b1, c->t1.p);
    add_src(a, V, C, int(H), int(W));
    a.rinv = c->rinv.p;
    a.gain = m.gain;
    a.gelu = 1;
    if (!conv3x3_uses_tc(a)) {  // the tcgen05 conv normalises its own halo
      rms_rinv(V, c->rinv.p, P, C, c->stream);
      mark(c, "misc", 1);
    }
    run_conv(c, a, c->stream);
    ConvArgs b = conv_args(int(L), int(H), int(W), C, C, m.w2, m.b2, V);
    add_src(b, c->t1.p, C, int(H), int(W));
    b.resid = V;
    b.res_pstride = C;
    b.res_bstride = (long long)H * W * C;
    run_conv(c, b, c->stream);
    mark(c, "conv", 2);
  }
}

struct CamTables {
  DevCam* upd[LVSG_MAX_STEPS];
  DevCam* rend[LVSG_MAX_STEPS];
  DevCam* final_cams;
  RayBaseCam* ray;
};

// Builds every per-frame camera table on the host and uploads them with one
// async copy from pinned staging.
CamTables upload_cams(lvsg_ctx* c, const lvsg_camera* enc_cams, const lvsg_frustum& target,
                      const lvsg_camera* render_cams) {
  const Plan& plan = c->plan;
  const int64_t M = c->cfg.views;
  const size_t S = plan.steps.size();
  CUDA_OK(cudaEventSynchronize(c->staging_done));  // previous frame's upload has landed
  char* host = static_cast<char*>(c->pinned);
  char* dev = reinterpret_cast<char*>(c->cams_dev.p);
  CamTables t;
  size_t off = 0;
  auto table = [&](auto fill) {
    DevCam* h = reinterpret_cast<DevCam*>(host + off);
    for (int64_t m = 0; m < M; ++m) h[m] = fill(m);
    DevCam* d = reinterpret_cast<DevCam*>(dev + off);
    off += size_t(M) * sizeof(DevCam);
    return d;
  };
  for (size_t s = 0; s < S; ++s) {
    const StepPlan& sp = plan.steps[s];
    t.upd[s] = table([&](int64_t m) { return dev_cam(camera_scaled(enc_cams[m], sp.feat_w, sp.feat_h)); });
    t.rend[s] = table([&](int64_t m) { return dev_cam(camera_scaled(enc_cams[m], sp.render_w, sp.render_h)); });
  }
  t.final_cams = render_cams ? table([&](int64_t m) { return dev_cam(render_cams[m]); }) : nullptr;
  // ray_plane_delta cameras (geometry.hpp:343-353)
  const int64_t hK = c->He >> c->cfg.pyramid_levels, wK = c->We >> c->cfg.pyramid_levels;
  RayBaseCam* rh = reinterpret_cast<RayBaseCam*>(host + off);
  const double* tm = target.camera.cam_from_world;
  for (int64_t m = 0; m < M; ++m) {
    lvsg_camera g = camera_scaled(enc_cams[m], wK, hK);
    RayBaseCam& r = rh[m];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.Rwc_in[i * 3 + j] = g.cam_from_world[j * 4 + i];
    double ow[3];
    center_of(g, ow);
    for (int i = 0; i < 3; ++i) {
      double acc = tm[i * 4 + 0] * ow[0];
      acc += tm[i * 4 + 1] * ow[1];
      acc += tm[i * 4 + 2] * ow[2];
      r.o[i] = acc + tm[i * 4 + 3];
    }
    r.fx = g.fx;
    r.fy = g.fy;
    r.cx = g.cx;
    r.cy = g.cy;
  }
  t.ray = reinterpret_cast<RayBaseCam*>(dev + off);
  off += size_t(M) * sizeof(RayBaseCam);
  // by a kernel, not a copy engine: on the compute stream a memcpy would
  // queue behind a bulk upload of the next frame's images (another stream)
  copy_from_pinned(dev, host, off, c->stream);
  mark(c, "misc", 1);
  CUDA_OK(cudaEventRecord(c->staging_done, c->stream));
  return t;
}

// encode_inputs' convolutional part (network.hpp:388-395) for views
// [m0, m1) of the device images [M, He, We, 3]: stem, per-level residual
// pairs and mean pools, written into those views' slices of the resident
// feature pyramid feats[k] ([M, H_k, W_k, C]). Target-independent: one
// encode serves every target of the frame (and, view-sharded, every GPU).
// enc_ready (optional, one event per view): view m's encoder image is only
// valid on the device once enc_ready[m] has fired (host-ABI uploads); level 0
// then runs view by view so each view's upload overlaps the previous view's
// convolutions.
void encode_views(lvsg_ctx* c, const float* enc, int64_t He, int64_t We, int m0, int m1,
                  const cudaEvent_t* enc_ready = nullptr) {
  const Config& cfg = c->cfg;
  const int C = int(cfg.channels), K = int(cfg.pyramid_levels), B = m1 - m0;
  cudaStream_t st = c->stream;
  const NetW& W = c->W;
  int h = int(He), w = int(We);
  const size_t per_in = size_t(h) * w * 3;
  auto fslice = [&](int k) {  // views [m0, m1) of pyramid level k
    const auto& e = c->plan.pyramid[size_t(k)];
    return c->feats[size_t(k)].p + size_t(m0) * e.first * e.second * C;
  };
  // fused exchange (lvsg_pyramid_import): the same slices of every peer
  const bool exch = !c->peer_feats.empty();
  std::vector<float*> peer_sl;
  auto peers = [&](int k, size_t extra) -> const std::vector<float*>* {
    if (!exch) return nullptr;
    const auto& e = c->plan.pyramid[size_t(k)];
    peer_sl.clear();
    for (auto& pf : c->peer_feats)
      peer_sl.push_back(pf[size_t(k)] + size_t(m0) * e.first * e.second * C + extra);
    return &peer_sl;
  };
  const float* x = c->enc_x.p;
  int k0 = 0;
  if (enc_ready) {
    const size_t per_x = size_t(h) * w * C;
    const size_t per_f = size_t(h / 2) * (w / 2) * C;
    for (int m = m0; m < m1; ++m) {
      CUDA_OK(cudaStreamWaitEvent(st, enc_ready[m], 0));
      float* xm = c->enc_x.p + per_x * (m - m0);
      ConvArgs a = conv_args(1, h, w, 3, C, W.stem_w, W.stem_b, xm);
      a.stem_host = c->stem_host.data();
      a.src[0] = ConvSrc{enc + per_in * m, 3, 3, (long long)per_in};
      a.nsrc = 1;
      run_conv(c, a, st);
      mark(c, "conv", 1);
      conv_residual(c, xm, xm, c->enc_t.p, 1, h, w, W.lvl_r1[0]);
      conv_residual(c, xm, xm, c->enc_t.p, 1, h, w, W.lvl_r2[0], fslice(0) + per_f * (m - m0),
                    peers(0, per_f * (m - m0)));
    }
    h /= 2;
    w /= 2;
    x = fslice(0);
    k0 = 1;
  } else {
    ConvArgs a = conv_args(B, h, w, 3, C, W.stem_w, W.stem_b, c->enc_x.p);
    a.stem_host = c->stem_host.data();
    a.src[0] = ConvSrc{enc + per_in * m0, 3, 3, (long long)per_in};
    a.nsrc = 1;
    run_conv(c, a, st);
    mark(c, "conv", 1);
  }
  for (int k = k0; k < K; ++k) {
    // level 0 reads the stem output in enc_x, level >= 1 feats[k-1]; both
    // write the level's residual pairs to enc_x and the pool to feats[k]
    float* xo = c->enc_x.p;
    conv_residual(c, x, xo, c->enc_t.p, B, h, w, W.lvl_r1[size_t(k)]);
    conv_residual(c, xo, xo, c->enc_t.p, B, h, w, W.lvl_r2[size_t(k)], fslice(k), peers(k, 0));
    h /= 2;
    w /= 2;
    x = fslice(k);
  }
  c->pyr_He = He;
  c->pyr_We = We;
}

// forward() on device images [M, He, We, 3]; leaves pre_d / pre_s / logits
// (volume resolution) and the final V resident. enc == nullptr: the encoder
// is skipped and the resident pyramid (lvsg_encode_device, all M views, at
// this He x We) is used. enc_ready: see encode_views.
void forward_device(lvsg_ctx* c, const float* enc, int64_t He, int64_t We,
                    const lvsg_camera* enc_cams, const lvsg_frustum& target,
                    const lvsg_camera* render_cams, CamTables* tables_out,
                    const cudaEvent_t* enc_ready = nullptr) {
  const Config& cfg = c->cfg;
  if (!c->have_weights) throw DimError("forward: no weights loaded (lvsg_load_weights / lvsg_init_weights)");
  frustum_validate(target);
  for (int64_t m = 0; m < cfg.views; ++m) camera_validate(enc_cams[m]);
  ensure_plan(c, He, We);
  if (!enc && (c->pyr_He != He || c->pyr_We != We))
    throw DimError("forward: no resident feature pyramid for " + std::to_string(He) + "x" +
                   std::to_string(We) + " inputs (lvsg_encode_device first)");
  const Plan& plan = c->plan;
  const int M = int(cfg.views), C = int(cfg.channels), Ca = int(cfg.appear_channels());
  const int K = int(cfg.pyramid_levels);
  cudaStream_t st = c->stream;
  const NetW& W = c->W;
  const int64_t launches0 = c->launch_total;
  if (c->prof) {
    prof_collect(c);
    mark(c, "start", 0);
  }
  CamTables cams = upload_cams(c, enc_cams, target, render_cams);
  if (tables_out) *tables_out = cams;

  // ---- encode_inputs --------------------------------------------------------
  {
    if (enc) encode_views(c, enc, He, We, 0, M, enc_ready);
    const int hK = int(plan.pyramid.back().first), wK = int(plan.pyramid.back().second);
    if (cfg.ablate_rays) {
      for (int k = 0; k < K; ++k)
        CUDA_OK(cudaMemsetAsync(c->rays[size_t(k)].p, 0,
                                size_t(M) * plan.pyramid[size_t(k)].first * plan.pyramid[size_t(k)].second * C * sizeof(float), st));
    } else {
      RayBaseArgs ra;
      const double* tm = target.camera.cam_from_world;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) ra.Rcw_t[i * 3 + j] = tm[i * 4 + j];
      ra.tfx = target.camera.fx;
      ra.tfy = target.camera.fy;
      ra.inv_span = 1.0 / target.far_depth - 1.0 / target.near_depth;
      ra.half_w = double(target.camera.width) / 2.0;
      ra.half_h = double(target.camera.height) / 2.0;
      ra.h = hK;
      ra.w = wK;
      ra.M = M;
      ray_base(cams.ray, ra, c->ray_base.p, st);
      mark(c, "misc", 1);
      for (int k = 0; k < K; ++k) {
        const int Hk = int(plan.pyramid[size_t(k)].first), Wk = int(plan.pyramid[size_t(k)].second);
        // C = 32: the 32 x 32 projection as a tcgen05 GEMM (collapse_tc.cu)
        const float* wimg = nullptr;
        if (C == 32 && !collapse_simt()) {
          auto key = std::make_tuple(W.ray_proj[size_t(k)], -2000, 0);
          auto it = c->wimg.find(key);
          if (it == c->wimg.end()) {
            auto img = std::make_unique<lvsg_ctx::WImg>();
            img->buf.ensure((ray_tc_weight_bytes() + 3) / 4);
            ray_tc_prepare(W.ray_proj[size_t(k)], img->buf.p, c->flag, st);
            it = c->wimg.emplace(key, std::move(img)).first;
            c->wimg_fresh = true;
          }
          wimg = it->second->buf.p;
        }
        if (!wimg || !ray_project_tc(c->ray_base.p, M, hK, wK, Hk, Wk, wimg, c->rays[size_t(k)].p,
                                     c->flag, st))
          ray_project(c->ray_base.p, M, hK, wK, Hk, Wk, W.ray_proj[size_t(k)], C,
                      c->rays[size_t(k)].p, st,
                      k < int(c->rayproj_host.size()) ? c->rayproj_host[size_t(k)].data() : nullptr);
        mark(c, "misc", 1);
      }
    }
  }

  // ---- initialize -----------------------------------------------------------
  float* V = c->V0.p;
  float* Vs = c->V1.p;
  int64_t L = plan.steps[0].layers, H = plan.steps[0].height, Wd = plan.steps[0].width;
  {
    const StepPlan& sp = plan.steps[0];
    fill_rows(V, W.init_feature, L * H * Wd, C, st);
    // flat band-centre depths (network.hpp:469-475)
    fill_anchor_depths(c->depth_out.p, int(L), H * Wd, 1.0 / target.near_depth - 1.0 / target.far_depth,
                       1.0 / target.far_depth, st);
    mark(c, "misc", 2);
    const int Hf = int(sp.feat_h), Wf = int(sp.feat_w);
    ConvArgs in{};
    in.nsrc = 0;
    add_src(in, c->feats[size_t(sp.level)].p, C, Hf, Wf);
    add_src(in, c->rays[size_t(sp.level)].p, C, Hf, Wf);
    update_cnn(c, W.steps[0], in, M, Hf, Wf);
    gather_stack(c->uu.p, M, Hf, Wf, C, cams.upd[0], ray_cam(target.camera, Wd, H),
                 c->depth_out.p, int(L), int(H), int(Wd), c->deltas.p, st);
    mark(c, "gather", 1);
    for (const FusionW& f : W.steps[0].fusions) fusion(c, V, L, H, Wd, f);
  }

  // ---- update steps -----------------------------------------------------------
  for (size_t s = 1; s < plan.steps.size(); ++s) {
    const StepPlan& sp = plan.steps[s];
    const StepW& sw = W.steps[s];
    for (const ConvPairW& cw : sw.collapse) {
      // the tensor-core MLP takes its split weight image from the context cache
      const float* wimg = nullptr;
      if (C == 32 && !collapse_simt()) {
        auto key = std::make_tuple(cw.w1, -1000, 0);
        auto it = c->wimg.find(key);
        if (it == c->wimg.end()) {
          auto img = std::make_unique<lvsg_ctx::WImg>();
          img->buf.ensure((collapse_tc_weight_bytes() + 3) / 4);
          collapse_tc_prepare(cw.w1, cw.w2, img->buf.p, c->flag, st);
          it = c->wimg.emplace(key, std::move(img)).first;
          c->wimg_fresh = true;
        }
        wimg = it->second->buf.p;
      }
      if (!wimg || !layer_collapse_tc(V, int(L), H * Wd, C, wimg, cw.b1, cw.b2, Vs, c->flag, st))
        layer_collapse(V, int(L), H * Wd, C, cw.w1, cw.b1, cw.w2, cw.b2, Vs, st);
      mark(c, "collapse", 1);
      std::swap(V, Vs);
      L /= 2;
    }
    const int Hf = int(sp.feat_h), Wf = int(sp.feat_w), Hv = int(sp.render_h), Wv = int(sp.render_w);
    const int Kp = Ca + 1, PS = pay_stride(Kp);
    const DepthAct act = depth_act(L, target);
    // update_block: render the volume into every view (ldm.hpp:223-244)
    decode_payload(V, int(L), int(H), int(Wd), C, W.w_appear, Ca, W.w_sigma, W.w_depth, act,
                   ray_cam(target.camera, Wd, H), c->payload.p, c->depth_in.p, c->points.p, st,
                   c->decw_host.empty() ? nullptr : c->decw_host.data());
    mark(c, "splat", 1);
    const float* feedback = c->fbr.p;
    if (cfg.ablate_render) {
      CUDA_OK(cudaMemsetAsync(c->fbr.p, 0, size_t(M) * Hf * Wf * PS * sizeof(float), st));
    } else {
      splat_det(c->payload.p, c->points.p, int(L), int(H * Wd), Kp, cams.rend[s], M, Hv, Wv,
                reinterpret_cast<int*>(c->splat_scratch.p), c->fb.p, st);
      mark(c, "splat", 6);
      if (sp.doubled) {
        resize_hwc(c->fb.p, c->fbr.p, M, Hv, Wv, PS, Hf, Wf, st);
        mark(c, "misc", 1);
      } else {
        feedback = c->fb.p;
      }
    }
    ConvArgs in{};
    in.nsrc = 0;
    add_src(in, feedback, Kp, Hf, Wf);
    in.src[0].pstride = PS;  // padded feedback rows
    in.src[0].bstride = (long long)Hf * Wf * PS;
    add_src(in, c->feats[size_t(sp.level)].p, C, Hf, Wf);
    add_src(in, c->rays[size_t(sp.level)].p, C, Hf, Wf);
    update_cnn(c, sw, in, M, Hf, Wf);
    // depth through the current volume, resized when the step doubles
    const float* dgather = c->depth_in.p;
    if (sp.doubled) {
      resize_hwc(c->depth_in.p, c->depth_out.p, int(L), int(H), int(Wd), 1, int(sp.height),
                 int(sp.width), st);
      mark(c, "misc", 1);
      dgather = c->depth_out.p;
    }
    gather_stack(c->uu.p, M, Hf, Wf, C, cams.upd[s], ray_cam(target.camera, sp.width, sp.height),
                 dgather, int(L), int(sp.height), int(sp.width), c->deltas.p, st);
    mark(c, "gather", 1);
    if (sp.doubled) {
      resize_hwc(V, Vs, int(L), int(H), int(Wd), C, int(sp.height), int(sp.width), st);
      mark(c, "misc", 1);
      std::swap(V, Vs);
    }
    H = sp.height;
    Wd = sp.width;
    for (const FusionW& f : sw.fusions) fusion(c, V, L, H, Wd, f);
  }

  // ---- decode_blend_logits + LDM pre-activation maps --------------------------
  const int64_t P = L * H * Wd;
  if (cfg.ablate_attention) {
    CUDA_OK(cudaMemsetAsync(c->logits.p, 0, size_t(P) * M * sizeof(float), st));
  } else {
    blend_logits(V, c->deltas.p, P, C, M, W.blend_w, W.blend_gain, c->logits.p, st,
                 c->blendw_host.data());
    mark(c, "attention", 1);
  }
  decode_scalar2(V, P, C, W.w_depth, c->pre_d.p, W.w_sigma, c->pre_s.p, st);
  mark(c, "misc", C == 32 ? 1 : 2);
  c->have_ldm = true;
  c->L = L;
  c->H = H;
  c->Wd = Wd;
  c->M = M;
  c->target = target;
  c->V = V;
  c->launches = c->launch_total - launches0;
  settle_images(c);
}

RenderArgs render_args(lvsg_ctx* c, const float* images, int64_t Hr, int64_t Wr,
                       const DevCam* cams_dev, float* rgb, int64_t row0, int64_t row1,
                       const lvsg_camera* host_cams = nullptr) {
  RenderArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pre_d = c->pre_d.p;
  a.pre_s = c->pre_s.p;
  a.logits = c->logits.p;
  a.L = int(c->L);
  a.H = int(c->H);
  a.W = int(c->Wd);
  a.M = int(c->M);
  a.Ho = int(c->plan.out_height);
  a.Wo = int(c->plan.out_width);
  a.row0 = int(row0);
  a.row1 = int(row1);
  a.act = depth_act(c->L, c->target);
  a.rc = ray_cam(c->target.camera, a.Wo, a.Ho);
  a.cams = cams_dev;
  // the same cameras by value in the kernel's parameter space (constant-bank
  // operands, no per-view shared-memory loads)
  if (host_cams && a.M <= kRenderParamViews) {
    for (int m = 0; m < a.M; ++m) {
      a.pc[m] = dev_cam(host_cams[m]);
      a.fc[m] = fast_cam(a.pc[m]);
    }
    a.pc_valid = 1;
  }
  a.images = images;
  a.Hr = int(Hr);
  a.Wr = int(Wr);
  a.rgb = rgb;
  a.bad_depth = c->bad_flag;
  const double slack = 1e-3 * (c->target.far_depth - c->target.near_depth);
  a.slack_lo = c->target.near_depth - slack;
  a.slack_hi = c->target.far_depth + slack;
  return a;
}

DevCam* upload_render_cams(lvsg_ctx* c, const lvsg_camera* cams) {
  // render-only path (lvsg_render): a dedicated slot after the frame tables
  const size_t M = size_t(c->M);
  const size_t S = c->plan.steps.size();
  const size_t off = (S * 2 + 1) * M * sizeof(DevCam) + M * sizeof(RayBaseCam);
  CUDA_OK(cudaEventSynchronize(c->staging_done));
  DevCam* h = reinterpret_cast<DevCam*>(static_cast<char*>(c->pinned) + off);
  for (size_t m = 0; m < M; ++m) h[m] = dev_cam(cams[m]);
  DevCam* d = reinterpret_cast<DevCam*>(reinterpret_cast<char*>(c->cams_dev.p) + off);
  copy_from_pinned(d, h, M * sizeof(DevCam), c->stream);
  mark(c, "misc", 1);
  CUDA_OK(cudaEventRecord(c->staging_done, c->stream));
  return d;
}

void check_render_inputs(lvsg_ctx* c, int64_t views, const lvsg_camera* cams) {
  if (!c->have_ldm) throw DimError("render_target: no LDM (call lvsg_forward first)");
  if (views != c->M)
    throw DimError("render_target: expected " + std::to_string(c->M) + " views, got " +
                   std::to_string(views) + " images / " + std::to_string(views) + " cameras");
  for (int64_t m = 0; m < views; ++m) camera_validate(cams[m]);
}

lvsg_status guard(lvsg_ctx* c, const auto& fn) {
  try {
    if (c) CUDA_OK(cudaSetDevice(c->device));
    fn();
    return LVSG_OK;
  } catch (const DimError& e) {
    if (c) c->err = e.what();
    return LVSG_ERR_DIM;
  } catch (const SchemaError& e) {
    if (c) c->err = e.what();
    return LVSG_ERR_DIM;
  } catch (const IoError& e) {
    if (c) c->err = e.what();
    return LVSG_ERR_IO;
  } catch (const NumericError& e) {
    if (c) c->err = e.what();
    return LVSG_ERR_NUMERIC;
  } catch (const CudaError& e) {
    if (c) c->err = e.what();
    return LVSG_ERR_CUDA;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return LVSG_ERR_INTERNAL;
  }
}

// The device flag's meaning: bit 2 an fp16-split overflow in a tensor-core
// operand (the result would be silently wrong: NumericError), bit 1 a depth
// outside the frustum (world_points, geometry.hpp:112-115: DimError).
[[noreturn]] void throw_flag(int bad) {
  if (bad & 2)
    throw NumericError(
        "fp16 split: a tensor-core operand (conv / attention activation or weight) has |x| >= "
        "65520, beyond the split's range");
  throw DimError("world_points: depth outside [near, far]");
}

void sync_and_check(lvsg_ctx* c) {
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaStreamSynchronize(c->stream));
  if (c->xfer) CUDA_OK(cudaStreamSynchronize(c->xfer));
  int bad = 0;
  CUDA_OK(cudaMemcpy(&bad, c->bad_flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) {
    CUDA_OK(cudaMemset(c->bad_flag, 0, sizeof(int)));
    throw_flag(bad);
  }
}

// Host wait for a pipelined frame: its read-back landed; its depth-range
// check (the reference's world_points DimError) is reported here.
void wait_slot(lvsg_ctx* c, FrameSlot& S) {
  S.ticket = -1;
  CUDA_OK(cudaEventSynchronize(S.ev_done));
  int bad = 0;
  CUDA_OK(cudaMemcpy(&bad, S.bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) {
    CUDA_OK(cudaMemset(S.bad, 0, sizeof(int)));
    throw_flag(bad);
  }
  (void)c;
}

void upload_images(lvsg_ctx* c, Buf& dst, int64_t views, const float* const* images, int64_t H,
                   int64_t W, cudaStream_t st) {
  if (!images) throw DimError("forward: null image list");
  const size_t per = size_t(H * W * 3);
  for (int64_t m = 0; m < views; ++m)
    if (!images[m]) throw DimError("forward: null image");
  dst.ensure(per * size_t(views));
  // host->device copies carry a large fixed cost per call on this link
  // (profiles/h2d_bw.py: 14 GB/s at 6 MB, 50 GB/s at 199 MB): views that are
  // adjacent in one host buffer go up as a single copy
  int64_t m = 0;
  while (m < views) {
    int64_t run = 1;
    while (m + run < views && images[m + run] == images[m] + per * size_t(run)) ++run;
    CUDA_OK(cudaMemcpyAsync(dst.p + per * size_t(m), images[m], per * size_t(run) * sizeof(float),
                            cudaMemcpyHostToDevice, st));
    m += run;
  }
}

void check_views(lvsg_ctx* c, int64_t views, int64_t H, int64_t W) {
  if (views != c->cfg.views)
    throw DimError("forward: expected " + std::to_string(c->cfg.views) + " views");
  if (H < 1 || W < 1) throw DimError("forward: images must be [H,W,3]");
}

}  // namespace
}  // namespace lvsg

using namespace lvsg;

extern "C" {

lvsg_status lvsg_validate_config(const lvsg_model_config* cfg, char* err, size_t err_len) {
  try {
    Config::from_c(cfg).validate();
    return LVSG_OK;
  } catch (const std::exception& e) {
    if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
    return LVSG_ERR_DIM;
  }
}

lvsg_status lvsg_plan_forward(const lvsg_model_config* cfg, int64_t image_h, int64_t image_w,
                              lvsg_plan* out, char* err, size_t err_len) {
  try {
    Plan p = plan_forward(Config::from_c(cfg), image_h, image_w);
    std::memset(out, 0, sizeof(*out));
    out->num_levels = int64_t(p.pyramid.size());
    for (size_t k = 0; k < p.pyramid.size(); ++k) {
      out->pyramid_h[k] = p.pyramid[k].first;
      out->pyramid_w[k] = p.pyramid[k].second;
    }
    out->num_steps = int64_t(p.steps.size());
    for (size_t s = 0; s < p.steps.size(); ++s) {
      const StepPlan& sp = p.steps[s];
      lvsg_step_plan& o = out->steps[s];
      o.in_layers = sp.in_layers;
      o.layers = sp.layers;
      o.in_height = sp.in_height;
      o.in_width = sp.in_width;
      o.height = sp.height;
      o.width = sp.width;
      o.doubled = sp.doubled;
      o.level = sp.level;
      o.feat_h = sp.feat_h;
      o.feat_w = sp.feat_w;
      o.render_h = sp.render_h;
      o.render_w = sp.render_w;
      o.collapse_count = sp.collapse_count;
      o.num_tokens = int64_t(sp.tokens.size());
    }
    out->out_height = p.out_height;
    out->out_width = p.out_width;
    return LVSG_OK;
  } catch (const std::exception& e) {
    if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
    return LVSG_ERR_DIM;
  }
}

lvsg_status lvsg_param_count(const lvsg_model_config* cfg, int64_t* count, int64_t* total_numel) {
  try {
    auto l = param_layout(Config::from_c(cfg));
    int64_t n = 0;
    for (auto& p : l) n += p.numel();
    if (count) *count = int64_t(l.size());
    if (total_numel) *total_numel = n;
    return LVSG_OK;
  } catch (const std::exception&) {
    return LVSG_ERR_DIM;
  }
}

lvsg_status lvsg_param_shape(const lvsg_model_config* cfg, int64_t index, int32_t* rank,
                             int64_t dims[4]) {
  try {
    auto l = param_layout(Config::from_c(cfg));
    if (index < 0 || index >= int64_t(l.size())) return LVSG_ERR_DIM;
    const auto& s = l[size_t(index)].shape;
    *rank = int32_t(s.size());
    for (int k = 0; k < 4; ++k) dims[k] = k < int(s.size()) ? s[size_t(k)] : 0;
    return LVSG_OK;
  } catch (const std::exception&) {
    return LVSG_ERR_DIM;
  }
}

lvsg_status lvsg_init_param_store(const lvsg_model_config* cfg, uint64_t seed, float* out) {
  try {
    init_param_store(Config::from_c(cfg), seed, out);
    return LVSG_OK;
  } catch (const std::exception&) {
    return LVSG_ERR_DIM;
  }
}

lvsg_status lvsg_create(const lvsg_model_config* cfg, int32_t device, lvsg_ctx** out) {
  g_create_err.clear();
  if (!out) return LVSG_ERR_DIM;
  *out = nullptr;
  std::unique_ptr<lvsg_ctx> c(new lvsg_ctx());
  try {
    c->cfg = Config::from_c(cfg);
    c->cfg.validate();
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return LVSG_ERR_DIM;
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    g_create_err = "lvsg_create: no CUDA device";
    return LVSG_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= n) {
    g_create_err = "lvsg_create: bad device ordinal";
    return LVSG_ERR_NO_DEVICE;
  }
  c->device = device;
  lvsg_status s = guard(c.get(), [&] {
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw CudaError("lvsg: built for sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                      std::to_string(prop.minor));
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->staging_done, cudaEventDisableTiming));
    CUDA_OK(cudaEventRecord(c->staging_done, c->stream));
    CUDA_OK(cudaStreamCreateWithFlags(&c->xfer, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->ev_ren, cudaEventDisableTiming));
    for (cudaEvent_t& e : c->ev_band) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_OK(cudaMalloc(&c->bad_flag, sizeof(int)));
    CUDA_OK(cudaMemset(c->bad_flag, 0, sizeof(int)));
    c->flag = c->bad_flag;
    c->layout = param_layout(c->cfg);
    c->total_params = 0;
    for (auto& p : c->layout) c->total_params += p.numel();
    c->weights.ensure(size_t(c->total_params));
  });
  if (s != LVSG_OK) {
    g_create_err = c->err;
    return s;
  }
  *out = c.release();
  return LVSG_OK;
}

void lvsg_destroy(lvsg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->bad_flag) cudaFree(c->bad_flag);
  if (c->xfer) cudaStreamSynchronize(c->xfer);
  if (c->staging_done) cudaEventDestroy(c->staging_done);
  for (cudaEvent_t e : {c->ev_main, c->ev_ren, c->ev_band[0], c->ev_band[1], c->ev_band[2],
                        c->ev_band[3]})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_enc) cudaEventDestroy(e);
  if (c->down) cudaStreamSynchronize(c->down);
  for (void* p : c->peer_maps) cudaIpcCloseMemHandle(p);
  for (FrameSlot& S : c->slots) {
    for (cudaEvent_t e : {S.ev_ren, S.ev_free, S.ev_done, S.ev_band[0], S.ev_band[1],
                          S.ev_band[2], S.ev_band[3]})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : S.ev_enc) cudaEventDestroy(e);
    if (S.bad) cudaFree(S.bad);
  }
  if (c->down) cudaStreamDestroy(c->down);
  if (c->xfer) cudaStreamDestroy(c->xfer);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* lvsg_last_error(const lvsg_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

lvsg_status lvsg_load_weights(lvsg_ctx* c, int64_t count, const float* const* tensors,
                              const int32_t* ranks, const int64_t* dims) {
  return guard(c, [&] {
    if (count < int64_t(c->layout.size())) throw DimError("bind_params: store has too few tensors");
    if (count > int64_t(c->layout.size())) throw DimError("bind_params: store has extra tensors");
    std::vector<float> flat(size_t(c->total_params));
    int64_t off = 0, doff = 0;
    for (size_t i = 0; i < c->layout.size(); ++i) {
      const auto& want = c->layout[i].shape;
      std::vector<int64_t> got(dims + doff, dims + doff + ranks[i]);
      doff += ranks[i];
      if (got != want) {
        auto str = [](const std::vector<int64_t>& s) {
          std::string o = "[";
          for (size_t k = 0; k < s.size(); ++k) o += (k ? "," : "") + std::to_string(s[k]);
          return o + "]";
        };
        throw DimError("bind_params tensor: expected shape " + str(want) + ", got " + str(got));
      }
      const int64_t n = c->layout[i].numel();
      std::memcpy(flat.data() + off, tensors[i], size_t(n) * sizeof(float));
      off += n;
    }
    CUDA_OK(cudaMemcpy(c->weights.p, flat.data(), flat.size() * sizeof(float), cudaMemcpyHostToDevice));
    bind_weights(c);
    c->have_weights = true;
  });
}

lvsg_status lvsg_load_weights_qntc(lvsg_ctx* c, const void* bytes, size_t len) {
  std::vector<std::vector<float>> store;
  std::vector<const float*> ptrs;
  std::vector<int32_t> ranks;
  std::vector<int64_t> dims;
  const lvsg_status s = guard(c, [&] {
    if (!bytes && len) throw IoError("tensor container: null buffer");
    const auto entries = qntc_unpack(static_cast<const uint8_t*>(bytes), len);
    for (const QntcEntry& e : entries) {
      // NamedTensor::as_f32 (io.cpp:86-90): a float model binds f32 entries
      if (e.dtype != 0)
        throw SchemaError("tensor container: entry \"" + e.name + "\" holds f64, expected f32");
      store.emplace_back(size_t(e.numel()));
      std::memcpy(store.back().data(), e.payload, store.back().size() * sizeof(float));
      ranks.push_back(int32_t(e.dims.size()));
      dims.insert(dims.end(), e.dims.begin(), e.dims.end());
    }
    for (const auto& t : store) ptrs.push_back(t.data());
  });
  if (s != LVSG_OK) return s;
  return lvsg_load_weights(c, int64_t(ptrs.size()), ptrs.data(), ranks.data(), dims.data());
}

lvsg_status lvsg_init_weights(lvsg_ctx* c, uint64_t seed) {
  return guard(c, [&] {
    std::vector<float> flat(size_t(c->total_params));
    init_param_store(c->cfg, seed, flat.data());
    CUDA_OK(cudaMemcpy(c->weights.p, flat.data(), flat.size() * sizeof(float), cudaMemcpyHostToDevice));
    bind_weights(c);
    c->have_weights = true;
  });
}

lvsg_status lvsg_forward(lvsg_ctx* c, int64_t views, const float* const* images, int64_t height,
                         int64_t width, const lvsg_camera* cams, const lvsg_frustum* target,
                         const lvsg_ldm_out* out) {
  return guard(c, [&] {
    check_views(c, views, height, width);
    upload_images(c, c->enc_in, views, images, height, width, c->stream);
    forward_device(c, c->enc_in.p, height, width, cams, *target, nullptr, nullptr);
    if (out) {
      const int64_t P = c->L * c->H * c->Wd, M = c->M, C = c->cfg.channels;
      const int64_t Po = c->L * c->plan.out_height * c->plan.out_width;
      if (out->depth || out->density || out->blend) {
        c->ldm_d.ensure(size_t(Po));
        c->ldm_s.ensure(size_t(Po));
        c->ldm_b.ensure(size_t(Po * M));
        RenderArgs a = render_args(c, nullptr, 0, 0, nullptr, nullptr, 0, c->plan.out_height);
        upsample_activate(a, c->ldm_d.p, c->ldm_s.p, c->ldm_b.p, c->stream);
      }
      sync_and_check(c);
      auto d2h = [&](float* dst, const float* src, int64_t n) {
        if (dst) CUDA_OK(cudaMemcpy(dst, src, size_t(n) * sizeof(float), cudaMemcpyDeviceToHost));
      };
      d2h(out->depth, c->ldm_d.p, Po);
      d2h(out->density, c->ldm_s.p, Po);
      d2h(out->blend, c->ldm_b.p, Po * M);
      d2h(out->blend_logits, c->logits.p, P * M);
      d2h(out->volume, c->V, P * C);
      if (out->deltas) {
        // device layout: texel-major per view [M][P][C] -> [L,H,W,M,C]
        std::vector<float> dev(size_t(P * M * C));
        d2h(dev.data(), c->deltas.p, P * M * C);
        for (int64_t m = 0; m < M; ++m)
          for (int64_t p = 0; p < P; ++p)
            std::memcpy(out->deltas + (p * M + m) * C, dev.data() + (m * P + p) * C,
                        size_t(C) * sizeof(float));
      }
      if (out->rgb && c->cfg.direct_rgb) {
        const int64_t Ho = c->plan.out_height, Wo = c->plan.out_width;
        c->ldm_d.ensure(size_t(P * 3));  // pre_a, then the composite
        c->rgb.ensure(size_t(Ho * Wo * 3));
        decode_linear(c->V, P, int(C), c->W.w_appear, 3, c->ldm_d.p, c->stream);
        RenderArgs a = render_args(c, nullptr, 0, 0, nullptr, nullptr, 0, Ho);
        direct_rgb(a, c->ldm_d.p, c->rgb.p, c->stream);
        sync_and_check(c);
        d2h(out->rgb, c->rgb.p, Ho * Wo * 3);
      }
    } else {
      sync_and_check(c);
    }
  });
}

lvsg_status lvsg_render(lvsg_ctx* c, int64_t views, const float* const* images, int64_t height,
                        int64_t width, const lvsg_camera* cams, float* rgb_out) {
  return guard(c, [&] {
    check_render_inputs(c, views, cams);
    if (height < 1 || width < 1) throw DimError("render_target: images must be [H,W,3]");
    upload_images(c, c->ren_in, views, images, height, width, c->stream);
    DevCam* dc = upload_render_cams(c, cams);
    const int64_t Ho = c->plan.out_height, Wo = c->plan.out_width;
    c->rgb.ensure(size_t(Ho * Wo * 3));
    RenderArgs a = render_args(c, c->ren_in.p, height, width, dc, c->rgb.p, 0, Ho, cams);
    render_fused(a, c->stream);
    CUDA_OK(cudaMemcpyAsync(rgb_out, c->rgb.p, size_t(Ho * Wo * 3) * sizeof(float),
                            cudaMemcpyDeviceToHost, c->stream));
    sync_and_check(c);
  });
}

// ---- pipelined host-buffer frames (lvsg_submit_frame / lvsg_wait_frame) ----
//
// The same work as the synchronous host call, split at the host wait: two
// frame slots (their own upload / output buffers and events) so frame k+1's
// uploads run on the copy stream under frame k's compute, and frame k's
// banded read-back runs on a separate download stream. lvsg_forward_render
// is submit + wait.
namespace lvsg {
namespace {
// decimate: no encoder images; the encoder input is resize_bilinear of the
// uploaded render views to (enc_h, enc_w) on the device (tape.hpp:858-917
// per channel), with the render cameras .scaled(enc_w, enc_h)
// (camera.cpp:67-77) as encoder cameras.
lvsg_status submit_impl(lvsg_ctx* c, int64_t views, const float* const* enc_images,
                        int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                        const float* const* render_images, int64_t render_h, int64_t render_w,
                        const lvsg_camera* render_cams, const lvsg_frustum* target,
                        float* rgb_out, int64_t* ticket, bool decimate) {
  std::unique_ptr<lvsg_camera[]> dec_cams;
  if (decimate && render_cams && views > 0 && views <= 4096 && enc_h > 0 && enc_w > 0) {
    dec_cams.reset(new lvsg_camera[size_t(views)]);
    for (int64_t m = 0; m < views; ++m) dec_cams[m] = camera_scaled(render_cams[m], enc_w, enc_h);
  }
  const lvsg_camera* enc_cams_used = decimate ? dec_cams.get() : enc_cams;
  return guard(c, [&] {
    if (decimate && !dec_cams) throw DimError("forward: bad decimation extents or cameras");
    check_views(c, views, enc_h, enc_w);
    check_views(c, views, render_h, render_w);
    for (int64_t m = 0; m < views; ++m) camera_validate(render_cams[m]);
    if (!rgb_out) throw DimError("forward: null output");
    if (enc_images)
      for (int64_t m = 0; m < views; ++m)
        if (!enc_images[m]) throw DimError("forward: null image");
    const int64_t k = c->next_ticket;
    FrameSlot& S = c->slots[k & 1];
    if (S.ticket >= 0) wait_slot(c, S);  // frame k-2 still owns the slot's buffers
    if (!S.ev_ren) {
      CUDA_OK(cudaEventCreateWithFlags(&S.ev_ren, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&S.ev_free, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&S.ev_done, cudaEventDisableTiming));
      for (cudaEvent_t& e : S.ev_band) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CUDA_OK(cudaMalloc(&S.bad, sizeof(int)));
      CUDA_OK(cudaMemset(S.bad, 0, sizeof(int)));
      CUDA_OK(cudaEventRecord(S.ev_free, c->stream));
    }
    if (!c->down) CUDA_OK(cudaStreamCreateWithFlags(&c->down, cudaStreamNonBlocking));
    // uploads (copy stream), once the slot's previous frame stopped reading
    // its buffers: the encoder views one by one, each with an event the
    // encoder's per-view level 0 waits on, then the render views, needed
    // only by the final render, under the rest of the forward pass
    CUDA_OK(cudaStreamWaitEvent(c->xfer, S.ev_free, 0));
    const size_t per = size_t(enc_h * enc_w * 3);
    if (enc_images) {
      S.enc_in.ensure(per * size_t(views));
      while (S.ev_enc.size() < size_t(views)) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        S.ev_enc.push_back(e);
      }
      for (int64_t m = 0; m < views; ++m) {
        CUDA_OK(cudaMemcpyAsync(S.enc_in.p + per * size_t(m), enc_images[m], per * sizeof(float),
                                cudaMemcpyHostToDevice, c->xfer));
        CUDA_OK(cudaEventRecord(S.ev_enc[size_t(m)], c->xfer));
      }
    }
    upload_images(c, S.ren_in, views, render_images, render_h, render_w, c->xfer);
    CUDA_OK(cudaEventRecord(S.ev_ren, c->xfer));
    if (decimate) {
      S.enc_in.ensure(per * size_t(views));
      if (S.ev_enc.empty()) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        S.ev_enc.push_back(e);
      }
      // on the compute stream behind the upload: a kernel on the copy
      // stream would interleave with the previous frame's persistent kernels
      CUDA_OK(cudaStreamWaitEvent(c->stream, S.ev_ren, 0));
      resize_hwc(S.ren_in.p, S.enc_in.p, int(views), int(render_h), int(render_w), 3, int(enc_h),
                 int(enc_w), c->stream);
      c->launches += 1;
    }
    // enc_images == NULL: the resident pyramid (lvsg_encode_device, complete
    // on the context's stream) is used. With the previous frame still in
    // flight the uploads finish under its compute, so the encoder runs
    // batched over the views behind the last upload; otherwise its level 0
    // runs view by view behind each view's upload.
    const bool behind = c->slots[(k + 1) & 1].ticket >= 0;
    if (enc_images && behind)
      CUDA_OK(cudaStreamWaitEvent(c->stream, S.ev_enc[size_t(views - 1)], 0));
    CamTables t;
    c->flag = S.bad;  // this frame's kernels report into its slot (read by wait_slot)
    try {
      forward_device(c, enc_images || decimate ? S.enc_in.p : nullptr, enc_h, enc_w,
                     enc_cams_used, *target, render_cams, &t,
                     enc_images && !behind ? S.ev_enc.data() : nullptr);
    } catch (...) {
      c->flag = c->bad_flag;
      throw;
    }
    c->flag = c->bad_flag;
    const int64_t Ho = c->plan.out_height, Wo = c->plan.out_width;
    S.rgb.ensure(size_t(Ho * Wo * 3));
    CUDA_OK(cudaStreamWaitEvent(c->stream, S.ev_ren, 0));
    // banded render; each band's read-back (download stream) overlaps the
    // next band's render
    constexpr int NB = 4;
    RenderArgs a0 = render_args(c, S.ren_in.p, render_h, render_w, t.final_cams, S.rgb.p, 0, Ho,
                                render_cams);
    for (int b = 0; b < NB; ++b) {
      const int64_t r0 = Ho * b / NB, r1 = Ho * (b + 1) / NB;
      if (r1 == r0) continue;
      RenderArgs a = a0;
      a.rgb = S.rgb.p + r0 * Wo * 3;
      a.row0 = int(r0);
      a.row1 = int(r1);
      a.bad_depth = S.bad;
      render_fused(a, c->stream);
      c->launches += 1;
      CUDA_OK(cudaEventRecord(S.ev_band[b], c->stream));
      CUDA_OK(cudaStreamWaitEvent(c->down, S.ev_band[b], 0));
      CUDA_OK(cudaMemcpyAsync(rgb_out + r0 * Wo * 3, S.rgb.p + r0 * Wo * 3,
                              size_t((r1 - r0) * Wo * 3) * sizeof(float), cudaMemcpyDeviceToHost,
                              c->down));
    }
    mark(c, "render", NB);
    CUDA_OK(cudaEventRecord(S.ev_free, c->stream));
    CUDA_OK(cudaEventRecord(S.ev_done, c->down));
    CUDA_OK(cudaGetLastError());
    S.ticket = k;
    c->next_ticket = k + 1;
    if (ticket) *ticket = k;
  });
}
}  // namespace
}  // namespace lvsg

lvsg_status lvsg_submit_frame(lvsg_ctx* c, int64_t views, const float* const* enc_images,
                              int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                              const float* const* render_images, int64_t render_h,
                              int64_t render_w, const lvsg_camera* render_cams,
                              const lvsg_frustum* target, float* rgb_out, int64_t* ticket) {
  return submit_impl(c, views, enc_images, enc_h, enc_w, enc_cams, render_images, render_h,
                     render_w, render_cams, target, rgb_out, ticket, false);
}

lvsg_status lvsg_submit_frame_decimated(lvsg_ctx* c, int64_t views,
                                        const float* const* render_images, int64_t render_h,
                                        int64_t render_w, const lvsg_camera* render_cams,
                                        int64_t enc_h, int64_t enc_w, const lvsg_frustum* target,
                                        float* rgb_out, int64_t* ticket) {
  return submit_impl(c, views, nullptr, enc_h, enc_w, nullptr, render_images, render_h, render_w,
                     render_cams, target, rgb_out, ticket, true);
}

lvsg_status lvsg_forward_render_decimated(lvsg_ctx* c, int64_t views,
                                          const float* const* render_images, int64_t render_h,
                                          int64_t render_w, const lvsg_camera* render_cams,
                                          int64_t enc_h, int64_t enc_w,
                                          const lvsg_frustum* target, float* rgb_out) {
  int64_t ticket = -1;
  const lvsg_status s = lvsg_submit_frame_decimated(c, views, render_images, render_h, render_w,
                                                    render_cams, enc_h, enc_w, target, rgb_out,
                                                    &ticket);
  if (s != LVSG_OK) return s;
  return lvsg_wait_frame(c, ticket);
}

lvsg_status lvsg_decimate_views_device(lvsg_ctx* c, int64_t views, const float* src, int64_t h,
                                       int64_t w, float* dst, int64_t out_h, int64_t out_w,
                                       void* stream) {
  return guard(c, [&] {
    if (views < 1 || h < 1 || w < 1 || out_h < 1 || out_w < 1 || !src || !dst)
      throw DimError("decimate: bad extents or null buffer");
    resize_hwc(src, dst, int(views), int(h), int(w), 3, int(out_h), int(out_w),
               stream ? static_cast<cudaStream_t>(stream) : c->stream);
    c->launches += 1;
    CUDA_OK(cudaGetLastError());
  });
}

lvsg_status lvsg_wait_frame(lvsg_ctx* c, int64_t ticket) {
  return guard(c, [&] {
    if (ticket < 0 || ticket >= c->next_ticket) throw DimError("wait_frame: no such frame");
    FrameSlot& S = c->slots[ticket & 1];
    if (S.ticket == ticket) wait_slot(c, S);  // else already retired (waited, or by a later submit)
  });
}

lvsg_status lvsg_forward_render(lvsg_ctx* c, int64_t views, const float* const* enc_images,
                                int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                                const float* const* render_images, int64_t render_h,
                                int64_t render_w, const lvsg_camera* render_cams,
                                const lvsg_frustum* target, float* rgb_out) {
  int64_t ticket = -1;
  const lvsg_status s = lvsg_submit_frame(c, views, enc_images, enc_h, enc_w, enc_cams,
                                          render_images, render_h, render_w, render_cams, target,
                                          rgb_out, &ticket);
  if (s != LVSG_OK) return s;
  return lvsg_wait_frame(c, ticket);
}

lvsg_status lvsg_forward_render_rows_device(lvsg_ctx* c, int64_t views, const float* enc_images,
                                            int64_t enc_h, int64_t enc_w,
                                            const lvsg_camera* enc_cams, const float* render_images,
                                            int64_t render_h, int64_t render_w,
                                            const lvsg_camera* render_cams,
                                            const lvsg_frustum* target, int64_t row0, int64_t row1,
                                            float* rgb_out, void* stream) {
  // enc_images == NULL: the encoder is skipped and the resident pyramid of
  // lvsg_encode_device is used (one encode, many targets / GPUs)
  return guard(c, [&] {
    check_views(c, views, enc_h, enc_w);
    check_views(c, views, render_h, render_w);
    for (int64_t m = 0; m < views; ++m) camera_validate(render_cams[m]);
    const Plan plan = plan_forward(c->cfg, enc_h, enc_w);
    if (row0 < 0 || row0 > row1 || row1 > plan.out_height)
      throw DimError("render_rows: bad row band");
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaStream_t own = c->stream;
    if (user) c->stream = user;
    try {
      CamTables t;
      forward_device(c, enc_images, enc_h, enc_w, enc_cams, *target, render_cams, &t);
      RenderArgs a = render_args(c, render_images, render_h, render_w, t.final_cams, rgb_out, row0,
                                 row1, render_cams);
      render_fused(a, c->stream);
      mark(c, "render", 1);
      c->launches += 1;
      CUDA_OK(cudaGetLastError());
    } catch (...) {
      c->stream = own;
      throw;
    }
    c->stream = own;
  });
}

lvsg_status lvsg_forward_render_device(lvsg_ctx* c, int64_t views, const float* enc_images,
                                       int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                                       const float* render_images, int64_t render_h,
                                       int64_t render_w, const lvsg_camera* render_cams,
                                       const lvsg_frustum* target, float* rgb_out, void* stream) {
  int64_t Ho = 0;
  try {
    if (c) Ho = lvsg::plan_forward(c->cfg, enc_h, enc_w).out_height;
  } catch (...) {
    Ho = 0;  // the rows call reports the DimError
  }
  return lvsg_forward_render_rows_device(c, views, enc_images, enc_h, enc_w, enc_cams,
                                         render_images, render_h, render_w, render_cams, target,
                                         0, Ho, rgb_out, stream);
}

lvsg_status lvsg_encode_device(lvsg_ctx* c, int64_t views, const float* enc_images, int64_t enc_h,
                               int64_t enc_w, int64_t view0, int64_t view1, void* stream) {
  return guard(c, [&] {
    check_views(c, views, enc_h, enc_w);
    if (view0 < 0 || view1 > views || view0 > view1) throw DimError("encode_inputs: bad view range");
    if (!c->have_weights)
      throw DimError("forward: no weights loaded (lvsg_load_weights / lvsg_init_weights)");
    plan_forward(c->cfg, enc_h, enc_w);  // DimError on a bad extent, before any launch
    ensure_plan(c, enc_h, enc_w);
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaStream_t own = c->stream;
    if (user) c->stream = user;
    const int64_t launches0 = c->launch_total;
    try {
      if (view1 > view0) encode_views(c, enc_images, enc_h, enc_w, int(view0), int(view1));
      c->pyr_He = enc_h;
      c->pyr_We = enc_w;
      CUDA_OK(cudaGetLastError());
    } catch (...) {
      c->stream = own;
      throw;
    }
    c->stream = own;
    c->launches = c->launch_total - launches0;
    settle_images(c);
  });
}

lvsg_status lvsg_pyramid_level(lvsg_ctx* c, int64_t level, float** data, int64_t dims[4]) {
  return guard(c, [&] {
    if (c->He <= 0)
      throw DimError("pyramid: no pyramid buffers yet (lvsg_encode_device / lvsg_pyramid_export)");
    if (level < 0 || level >= c->cfg.pyramid_levels) throw DimError("pyramid: bad level");
    const auto& e = c->plan.pyramid[size_t(level)];
    *data = c->feats[size_t(level)].p;
    dims[0] = c->cfg.views;
    dims[1] = e.first;
    dims[2] = e.second;
    dims[3] = c->cfg.channels;
  });
}

lvsg_status lvsg_pyramid_export(lvsg_ctx* c, int64_t enc_h, int64_t enc_w, uint8_t* handles) {
  return guard(c, [&] {
    plan_forward(c->cfg, enc_h, enc_w);
    ensure_plan(c, enc_h, enc_w);
    for (int64_t k = 0; k < c->cfg.pyramid_levels; ++k) {
      cudaIpcMemHandle_t h;
      CUDA_OK(cudaIpcGetMemHandle(&h, c->feats[size_t(k)].p));
      std::memcpy(handles + k * 64, &h, 64);
    }
  });
}

lvsg_status lvsg_pyramid_import(lvsg_ctx* c, int64_t npeers, const uint8_t* handles) {
  return guard(c, [&] {
    if (npeers < 0 || npeers > 7) throw DimError("pyramid exchange: 0..7 peers");
    if (npeers == 0) {  // back to a private pyramid (mappings stay open until destroy)
      c->peer_feats.clear();
      return;
    }
    if (c->He <= 0) throw DimError("pyramid exchange: lvsg_pyramid_export first");
    const int64_t K = c->cfg.pyramid_levels;
    int me = 0;
    CUDA_OK(cudaGetDevice(&me));
    std::vector<std::vector<float*>> feats;
    for (int64_t q = 0; q < npeers; ++q) {
      std::vector<float*> lv;
      for (int64_t k = 0; k < K; ++k) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + (q * K + k) * 64, 64);
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          cudaGetLastError();
          throw CudaError(std::string("pyramid exchange: peer pyramid not mappable (") +
                          cudaGetErrorString(e) + "); use the NCCL all-gather");
        }
        c->peer_maps.push_back(p);
        // the epilogue stores into this buffer directly: its device must be
        // this one or a peer this device can write over NVLink
        cudaPointerAttributes pa{};
        CUDA_OK(cudaPointerGetAttributes(&pa, p));
        int ok = 1;
        if (pa.device != me) CUDA_OK(cudaDeviceCanAccessPeer(&ok, me, pa.device));
        if (!ok)
          throw CudaError("pyramid exchange: device " + std::to_string(me) +
                          " has no peer access to device " + std::to_string(pa.device) +
                          "; use the NCCL all-gather");
        lv.push_back(static_cast<float*>(p));
      }
      feats.push_back(std::move(lv));
    }
    c->peer_feats = std::move(feats);
  });
}

lvsg_status lvsg_render_rows_device(lvsg_ctx* c, int64_t views, const float* render_images,
                                    int64_t render_h, int64_t render_w,
                                    const lvsg_camera* render_cams, int64_t row0, int64_t row1,
                                    float* rgb_out, void* stream) {
  return guard(c, [&] {
    check_render_inputs(c, views, render_cams);
    if (row0 < 0 || row1 > c->plan.out_height || row0 > row1)
      throw DimError("render_rows: bad row band");
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaStream_t own = c->stream;
    if (user) c->stream = user;
    DevCam* dc = upload_render_cams(c, render_cams);
    RenderArgs a = render_args(c, render_images, render_h, render_w, dc, rgb_out, row0, row1,
                               render_cams);
    render_fused(a, c->stream);
    c->stream = own;
    CUDA_OK(cudaGetLastError());
  });
}

lvsg_status lvsg_synchronize(lvsg_ctx* c) {
  return guard(c, [&] { sync_and_check(c); });
}

int64_t lvsg_last_launch_count(const lvsg_ctx* c) { return c ? c->launches : 0; }

// Debug hook (not in the public header): cmd 0 resets and starts the conv
// timeline, 1 copies `n` slots [entry, ready, exit, CTAs] (globaltimer ns)
// into buf and returns the slot count through *n, 2 stops it. Builds without
// LVSG_TIMELINE report *n = -1.
extern "C" lvsg_status lvsg_debug_conv_timeline(lvsg_ctx* c, int32_t cmd, unsigned long long* buf,
                                                int32_t* n) {
  return guard(c, [&] {
    if (cmd == 0) {
      CUDA_OK(cudaStreamSynchronize(c->stream));
      lvsg::conv_timeline_reset();
      c->tl_next = 0;
    } else if (cmd == 1) {
      CUDA_OK(cudaDeviceSynchronize());
      const int got = lvsg::conv_timeline_read(buf, std::min(*n, c->tl_next));
      *n = got < 0 ? -1 : got;
    } else {
      c->tl_next = -1;
    }
  });
}

lvsg_status lvsg_profile_enable(lvsg_ctx* c, int32_t on) {
  return guard(c, [&] {
    prof_collect(c);
    c->prof = on != 0;
    c->prof_labels.clear();
    c->prof_counts.clear();
    c->prof_acc.clear();
  });
}

lvsg_status lvsg_profile_read(lvsg_ctx* c, char* buf, size_t len) {
  return guard(c, [&] {
    prof_collect(c);
    std::string out;
    for (const auto& kv : c->prof_acc) {
      char line[160];
      std::snprintf(line, sizeof(line), "%s %.6f %lld\n", kv.first.c_str(), kv.second.first,
                    (long long)kv.second.second);
      out += line;
    }
    c->prof_acc.clear();
    if (buf && len) std::snprintf(buf, len, "%s", out.c_str());
  });
}

void* lvsg_stream(lvsg_ctx* c) { return c ? c->stream : nullptr; }

lvsg_status lvsg_stage_world_points(lvsg_ctx* c, const lvsg_frustum* fr, const float* depth,
                                    int64_t L, int64_t H, int64_t W, float* points) {
  return guard(c, [&] {
    frustum_validate(*fr);
    if (L < 1 || H < 1 || W < 1) throw DimError("world_points: depth must be [L,H,W]");
    const double slack = 1e-3 * (fr->far_depth - fr->near_depth);
    stage_world_points(ray_cam(fr->camera, W, H), depth, int(L), int(H), int(W), points,
                       fr->near_depth - slack, fr->far_depth + slack, c->bad_flag, c->stream);
    sync_and_check(c);
  });
}

lvsg_status lvsg_stage_footprints(lvsg_ctx* c, const lvsg_camera* cam, const float* points,
                                  int64_t P, int32_t* taps, uint8_t* valid, double* fracs) {
  return guard(c, [&] {
    stage_footprints(dev_cam(*cam), points, P, taps, valid, fracs, c->stream);
    sync_and_check(c);
  });
}

lvsg_status lvsg_stage_conv3x3(lvsg_ctx* c, const float* x, const float* w, const float* b,
                               float* y, int64_t B, int64_t Cin, int64_t Cout, int64_t H,
                               int64_t W, int32_t impl) {
  return guard(c, [&] {
    if (B < 1 || Cin < 1 || Cout < 1 || H < 1 || W < 1) throw DimError("conv3x3: bad shapes");
    ConvArgs a = conv_args(int(B), int(H), int(W), int(Cin), int(Cout), w, b, y);
    add_src(a, x, int(Cin), int(H), int(W));
    run_conv(c, a, c->stream, impl, false);
    sync_and_check(c);
  });
}

lvsg_status lvsg_stage_conv3x3_fused(lvsg_ctx* c, const float* x, int64_t x_pstride,
                                     const float* w, int64_t w_cin, int64_t w_ci0, const float* b,
                                     const float* norm_gain, int32_t gelu, const float* resid,
                                     float* y, int64_t B, int64_t Cin, int64_t Cout, int64_t H,
                                     int64_t W, int32_t impl) {
  return guard(c, [&] {
    if (B < 1 || Cin < 1 || Cout < 1 || H < 1 || W < 1 || x_pstride < Cin || w_ci0 < 0 ||
        w_ci0 + Cin > w_cin)
      throw DimError("conv3x3: bad shapes");
    ConvArgs a = conv_args(int(B), int(H), int(W), int(Cin), int(Cout), w, b, y);
    a.src[0] = ConvSrc{x, int(Cin), int(x_pstride), (long long)H * W * x_pstride};
    a.nsrc = 1;
    a.w_cin = int(w_cin);
    a.w_ci0 = int(w_ci0);
    a.gelu = gelu;
    if (resid) {
      a.resid = resid;
      a.res_pstride = int(Cout);
      a.res_bstride = (long long)H * W * Cout;
    }
    if (norm_gain) {  // conv_mlp_residual's rms_norm on the input
      if (x_pstride != Cin) throw DimError("conv3x3: rms-norm input must be dense");
      c->rinv.ensure(size_t(B * H * W));
      a.rinv = c->rinv.p;
      a.gain = norm_gain;
      if (!conv3x3_uses_tc(a, impl)) rms_rinv(x, c->rinv.p, B * H * W, int(Cin), c->stream);
    }
    run_conv(c, a, c->stream, impl, false);
    sync_and_check(c);
  });
}

lvsg_status lvsg_stage_gather(lvsg_ctx* c, const lvsg_camera* cam, const float* image,
                              int64_t Hi, int64_t Wi, int64_t C, const float* points, int64_t P,
                              float* values, float* mask) {
  return guard(c, [&] {
    stage_gather(dev_cam(*cam), image, int(Hi), int(Wi), int(C), points, P, values, mask, c->stream);
    sync_and_check(c);
  });
}

// ---- per-stage entry points on caller-supplied (oracle) inputs --------------

lvsg_status lvsg_stage_attend(lvsg_ctx* c, float* V, const float* deltas, int64_t P, int64_t M,
                              int64_t heads, const float* wq, const float* wo, const float* gain,
                              int32_t zero_scores) {
  return guard(c, [&] {
    const int C = int(c->cfg.channels);
    if (P < 1 || M < 1 || heads < 1 || heads > 8) throw DimError("attend_residual: bad shapes");
    // Δ from the reference layout [P, M, C] into the kernels' [M][P][C]
    const size_t n = size_t(P) * M * C;
    c->stage_a.ensure(n + 128);
    deltas_to_view_major(deltas, c->stage_a.p, P, int(M), C, c->stream);
    c->attn_scratch.ensure(attend_scratch_floats(P, C, int(M), int(heads)));
    attend(V, c->stage_a.p, P, C, int(M), int(heads), wq, nullptr, wo, gain, zero_scores,
           c->attn_scratch.p, nullptr, false, c->flag, c->stream);
    sync_and_check(c);
  });
}

lvsg_status lvsg_stage_upsample_render(lvsg_ctx* c, const lvsg_frustum* target, const float* V,
                                       const float* logits, int64_t L, int64_t H, int64_t W,
                                       int64_t M, const float* w_depth, const float* w_sigma,
                                       const float* images, int64_t Hr, int64_t Wr,
                                       const lvsg_camera* cams, int64_t Ho, int64_t Wo,
                                       float* rgb) {
  return guard(c, [&] {
    frustum_validate(*target);
    const int C = int(c->cfg.channels);
    if (L < 1 || H < 1 || W < 1 || M < 1 || M > 32 || Ho < 1 || Wo < 1 || Hr < 1 || Wr < 1)
      throw DimError("render_target: bad shapes");
    for (int64_t m = 0; m < M; ++m) camera_validate(cams[m]);
    const int64_t P = L * H * W;
    c->stage_b.ensure(size_t(2 * P));
    decode_scalar2(V, P, C, w_depth, c->stage_b.p, w_sigma, c->stage_b.p + P, c->stream);
    std::vector<DevCam> hc(static_cast<size_t>(M));
    for (int64_t m = 0; m < M; ++m) hc[size_t(m)] = dev_cam(cams[m]);
    c->stage_cams.ensure((hc.size() * sizeof(DevCam) + 3) / 4);
    CUDA_OK(cudaMemcpyAsync(c->stage_cams.p, hc.data(), hc.size() * sizeof(DevCam),
                            cudaMemcpyHostToDevice, c->stream));
    RenderArgs a;
    std::memset(&a, 0, sizeof(a));
    a.pre_d = c->stage_b.p;
    a.pre_s = c->stage_b.p + P;
    a.logits = logits;
    a.L = int(L);
    a.H = int(H);
    a.W = int(W);
    a.M = int(M);
    a.Ho = int(Ho);
    a.Wo = int(Wo);
    a.row0 = 0;
    a.row1 = int(Ho);
    a.act = depth_act(L, *target);
    a.rc = ray_cam(target->camera, Wo, Ho);
    a.cams = reinterpret_cast<const DevCam*>(c->stage_cams.p);
    if (M <= kRenderParamViews) {
      for (int64_t m = 0; m < M; ++m) {
        a.pc[m] = hc[size_t(m)];
        a.fc[m] = fast_cam(hc[size_t(m)]);
      }
      a.pc_valid = 1;
    }
    a.images = images;
    a.Hr = int(Hr);
    a.Wr = int(Wr);
    a.rgb = rgb;
    a.bad_depth = c->bad_flag;
    const double slack = 1e-3 * (target->far_depth - target->near_depth);
    a.slack_lo = target->near_depth - slack;
    a.slack_hi = target->far_depth + slack;
    render_fused(a, c->stream);
    sync_and_check(c);
  });
}

lvsg_status lvsg_stage_render_to_view(lvsg_ctx* c, const lvsg_frustum* target, const float* V,
                                      int64_t L, int64_t H, int64_t W, const float* w_appear,
                                      int64_t Ca, const float* w_sigma, const float* w_depth,
                                      const lvsg_camera* cam, float* out) {
  return guard(c, [&] {
    frustum_validate(*target);
    camera_validate(*cam);
    const int C = int(c->cfg.channels);
    if (L < 1 || H < 1 || W < 1 || Ca < 1) throw DimError("render_to_input_view: bad shapes");
    const int64_t P = L * H * W, Hv = cam->height, Wv = cam->width;
    const int K = int(Ca) + 1, PS = pay_stride(K);
    c->stage_a.ensure(size_t(P) * payload_stride(K));  // payload
    c->stage_b.ensure(size_t(P) * 4);       // depth + points
    c->stage_c.ensure(size_t(Hv * Wv) * PS + splat_det_scratch_ints(P, L * Hv * Wv));
    float* depth = c->stage_b.p;
    float* points = c->stage_b.p + P;
    decode_payload(V, int(L), int(H), int(W), C, w_appear, int(Ca), w_sigma, w_depth,
                   depth_act(L, *target), ray_cam(target->camera, W, H), c->stage_a.p, depth,
                   points, c->stream);
    const DevCam hc = dev_cam(*cam);
    c->stage_cams.ensure((sizeof(DevCam) + 3) / 4);
    CUDA_OK(cudaMemcpyAsync(c->stage_cams.p, &hc, sizeof(DevCam), cudaMemcpyHostToDevice,
                            c->stream));
    float* fb = c->stage_c.p;
    splat_det(c->stage_a.p, points, int(L), int(H * W), K,
              reinterpret_cast<const DevCam*>(c->stage_cams.p), 1, int(Hv), int(Wv),
              reinterpret_cast<int*>(fb + size_t(Hv * Wv) * PS), fb, c->stream);
    // padded feedback rows [Hv*Wv][PS] -> [Hv*Wv][K]
    CUDA_OK(cudaMemcpy2DAsync(out, size_t(K) * sizeof(float), fb, size_t(PS) * sizeof(float),
                              size_t(K) * sizeof(float), size_t(Hv * Wv),
                              cudaMemcpyDeviceToDevice, c->stream));
    sync_and_check(c);
  });
}

}  // extern "C"
