// Reference-side drop-in adapter (header only). A maintainer of the `lvs`
// C++ library includes this next to "lvs/network.hpp" and links liblvsg.so to
// run the per-frame path on a B200 with the reference's own types:
//
//   lvs::gpu::Model m(cfg);               // ModelConfig  (network.hpp:46-59)
//   m.bind(store);                        // bind_params  (network.hpp:330-339)
//   lvs::gpu::Ldm ldm = m.forward(images, cams, target);   // forward (network.hpp:562-603)
//   lvs::Tensor<float> rgb = m.render_target(images_hd, cams_hd);  // ldm.hpp:193-199
//
// Errors come back as the reference's exception classes (DimError,
// NumericError) so call sites keep their handling (main.cpp:670-693).
#pragma once

#include <string>
#include <vector>

#include "lvs/camera.hpp"
#include "lvs/network.hpp"
#include "lvs/tensor.hpp"
#include "lvsg.h"

namespace lvs::gpu {

inline lvsg_camera to_c(const Camera& c) {
  lvsg_camera o;
  o.fx = c.fx;
  o.fy = c.fy;
  o.cx = c.cx;
  o.cy = c.cy;
  o.width = c.width;
  o.height = c.height;
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) o.cam_from_world[r * 4 + k] = c.cam_from_world(r, k);
  return o;
}

inline lvsg_frustum to_c(const Frustum& f) {
  lvsg_frustum o;
  o.camera = to_c(f.camera);
  o.near_depth = f.near;
  o.far_depth = f.far;
  return o;
}

// ForwardResult (network.hpp:551-558) without the tape: the LDM, the
// pre-softmax blend logits, the final volume and deltas, and (direct_rgb
// configs only, else empty) the decoded-colour composite rgb.
struct Ldm {
  Tensor<float> depth, density, blend, blend_logits, volume, deltas, rgb;
};

class Model {
 public:
  explicit Model(const ModelConfig& cfg, int device = 0) : cfg_(cfg) {
    for (const StepConfig& s : cfg.steps)
      steps_.push_back({s.in_layers, s.layers, s.height, s.width, s.pyramid_level, s.blocks.c_str()});
    c_.steps = steps_.data();
    c_.num_steps = int64_t(steps_.size());
    c_.channels = cfg.channels;
    c_.views = cfg.views;
    c_.pyramid_levels = cfg.pyramid_levels;
    c_.upsample = cfg.upsample;
    c_.near_depth = cfg.near;
    c_.far_depth = cfg.far;
    c_.ablate_render = cfg.ablate_render;
    c_.ablate_attention = cfg.ablate_attention;
    c_.ablate_rays = cfg.ablate_rays;
    c_.direct_rgb = cfg.direct_rgb;
    const lvsg_status s = lvsg_create(&c_, device, &ctx_);
    check(s, lvsg_last_error(nullptr));
  }
  ~Model() { lvsg_destroy(ctx_); }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;

  // bind_params(cfg, store): the flat tensor list in build_params order.
  void bind(const std::vector<Tensor<float>>& store) {
    std::vector<const float*> ptrs;
    std::vector<int32_t> ranks;
    std::vector<int64_t> dims;
    for (const auto& t : store) {
      ptrs.push_back(t.data());
      ranks.push_back(t.rank());
      for (int64_t d : t.shape()) dims.push_back(d);
    }
    check(lvsg_load_weights(ctx_, int64_t(store.size()), ptrs.data(), ranks.data(), dims.data()));
  }

  Ldm forward(const std::vector<Tensor<float>>& images, const std::vector<Camera>& cams,
              const Frustum& target) {
    if (images.empty()) throw DimError("forward: expected " + std::to_string(cfg_.views) + " views");
    std::vector<const float*> ptrs;
    for (const auto& im : images) ptrs.push_back(im.data());
    std::vector<lvsg_camera> cc;
    for (const auto& c : cams) cc.push_back(to_c(c));
    if (cc.size() != images.size()) throw DimError("encode_inputs: need one camera per image");
    const int64_t H = images[0].dim(0), W = images[0].dim(1);
    ForwardPlan plan = plan_forward(cfg_, H, W);
    const auto& last = plan.steps.back();
    const int64_t L = last.layers, Ho = plan.out_height, Wo = plan.out_width, M = cfg_.views;
    Ldm out{Tensor<float>({L, Ho, Wo}), Tensor<float>({L, Ho, Wo}), Tensor<float>({L, Ho, Wo, M}),
            Tensor<float>({L, last.height, last.width, M}),
            Tensor<float>({L, last.height, last.width, cfg_.channels}),
            Tensor<float>({L, last.height, last.width, M, cfg_.channels}),
            cfg_.direct_rgb ? Tensor<float>({Ho, Wo, 3}) : Tensor<float>()};
    lvsg_ldm_out o{out.depth.data(), out.density.data(), out.blend.data(), out.blend_logits.data(),
                   out.volume.data(), out.deltas.data(),
                   cfg_.direct_rgb ? out.rgb.data() : nullptr};
    lvsg_frustum t = to_c(target);
    check(lvsg_forward(ctx_, int64_t(images.size()), ptrs.data(), H, W, cc.data(), &t, &o));
    out_hw_ = {Ho, Wo};
    return out;
  }

  Tensor<float> render_target(const std::vector<Tensor<float>>& images,
                              const std::vector<Camera>& cams) {
    std::vector<const float*> ptrs;
    for (const auto& im : images) ptrs.push_back(im.data());
    std::vector<lvsg_camera> cc;
    for (const auto& c : cams) cc.push_back(to_c(c));
    Tensor<float> rgb({out_hw_.first, out_hw_.second, 3});
    check(lvsg_render(ctx_, int64_t(images.size()), ptrs.data(), images.at(0).dim(0),
                      images.at(0).dim(1), cc.data(), rgb.data()));
    return rgb;
  }

 private:
  void check(lvsg_status s, const char* msg = nullptr) {
    if (s == LVSG_OK) return;
    std::string m = msg ? msg : lvsg_last_error(ctx_);
    if (s == LVSG_ERR_DIM) throw DimError(m);
    if (s == LVSG_ERR_NUMERIC) throw NumericError(m);
    throw std::runtime_error("lvsg: " + m);
  }

  ModelConfig cfg_;
  std::vector<lvsg_step_config> steps_;
  lvsg_model_config c_{};
  lvsg_ctx* ctx_ = nullptr;
  std::pair<int64_t, int64_t> out_hw_{0, 0};
};

}  // namespace lvs::gpu
