// C-ABI driver over the REAL reference library (TEST INFRASTRUCTURE ONLY).
//
// Compiled against the unmodified headers/sources under /root/reference/proj
// (see oracle/Makefile) into oracle/_ref/libref.so. Used by tests/ to pin the
// C restatement (oracle/lvs_oracle.c) and to make golden fixtures, and by
// bench.py's reference arm as the CPU baseline. Never part of the product.
//
// Every entry point runs the reference's own T=float path:
//   init_param_store  network.hpp:354-362
//   forward           network.hpp:562-603
//   render_target     ldm.hpp:193-199
//   RigSpec/make_scene/oracle_render  scenes.cpp:40-171

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../include/lvsg.h"
#include "lvs/io.hpp"
#include "lvs/network.hpp"
#include "lvs/scenes.hpp"

using namespace lvs;

namespace {

void set_err(char* err, size_t len, const std::string& msg) {
  if (err && len) {
    std::snprintf(err, len, "%s", msg.c_str());
  }
}

ModelConfig to_cfg(const lvsg_model_config* c) {
  ModelConfig m;
  for (int64_t s = 0; s < c->num_steps; ++s) {
    const lvsg_step_config& st = c->steps[s];
    m.steps.push_back({st.in_layers, st.layers, st.height, st.width, st.pyramid_level,
                       std::string(st.blocks ? st.blocks : "")});
  }
  m.channels = c->channels;
  m.views = c->views;
  m.pyramid_levels = c->pyramid_levels;
  m.upsample = c->upsample;
  m.near = c->near_depth;
  m.far = c->far_depth;
  m.ablate_render = c->ablate_render != 0;
  m.ablate_attention = c->ablate_attention != 0;
  m.ablate_rays = c->ablate_rays != 0;
  m.direct_rgb = c->direct_rgb != 0;
  return m;
}

Camera to_cam(const lvsg_camera& c) {
  Eigen::Matrix4d m;
  for (int r = 0; r < 4; ++r)
    for (int k = 0; k < 4; ++k) m(r, k) = c.cam_from_world[r * 4 + k];
  Camera cam;
  cam.fx = c.fx;
  cam.fy = c.fy;
  cam.cx = c.cx;
  cam.cy = c.cy;
  cam.width = c.width;
  cam.height = c.height;
  cam.cam_from_world = m;
  return cam;
}

lvsg_camera from_cam(const Camera& c) {
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

Frustum to_fr(const lvsg_frustum& f) { return Frustum{to_cam(f.camera), f.near_depth, f.far_depth}; }

template <typename Fn>
int guarded(char* err, size_t len, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const DimError& e) {
    set_err(err, len, e.what());
    return 1;
  } catch (const NumericError& e) {
    set_err(err, len, e.what());
    return 2;
  } catch (const SchemaError& e) {
    set_err(err, len, e.what());
    return 1;
  } catch (const IoError& e) {
    set_err(err, len, e.what());
    return 3;
  } catch (const std::exception& e) {
    set_err(err, len, e.what());
    return 13;
  }
}

void copy_out(const Tensor<float>& t, float* dst) {
  if (dst) std::memcpy(dst, t.data(), size_t(t.numel()) * sizeof(float));
}

}  // namespace

extern "C" {

int ref_param_count(const lvsg_model_config* c, int64_t* count, int64_t* numel, char* err,
                    size_t len) {
  return guarded(err, len, [&] {
    std::vector<Tensor<float>> s = init_param_store<float>(to_cfg(c), 0);
    int64_t n = 0;
    for (auto& t : s) n += t.numel();
    *count = int64_t(s.size());
    *numel = n;
  });
}

int ref_init_param_store(const lvsg_model_config* c, uint64_t seed, float* out, int32_t* ranks,
                         int64_t* dims, char* err, size_t len) {
  return guarded(err, len, [&] {
    std::vector<Tensor<float>> s = init_param_store<float>(to_cfg(c), seed);
    int64_t off = 0;
    for (size_t i = 0; i < s.size(); ++i) {
      std::memcpy(out + off, s[i].data(), size_t(s[i].numel()) * sizeof(float));
      off += s[i].numel();
      if (ranks) ranks[i] = s[i].rank();
      if (dims)
        for (int k = 0; k < 4; ++k) dims[i * 4 + k] = k < s[i].rank() ? s[i].dim(k) : 0;
    }
  });
}

int ref_plan_forward(const lvsg_model_config* c, int64_t h, int64_t w, lvsg_plan* out, char* err,
                     size_t len) {
  return guarded(err, len, [&] {
    ForwardPlan p = plan_forward(to_cfg(c), h, w);
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
  });
}

// RigSpec::cameras / ::target (scenes.cpp:40-60).
int ref_rig(int64_t rows, int64_t cols, double baseline, int64_t width, int64_t height,
            double focal, lvsg_camera* cams, lvsg_camera* target, char* err, size_t len) {
  return guarded(err, len, [&] {
    RigSpec r{rows, cols, baseline, width, height, focal};
    std::vector<Camera> cs = r.cameras();
    for (size_t i = 0; i < cs.size(); ++i) cams[i] = from_cam(cs[i]);
    if (target) *target = from_cam(r.target());
  });
}

// make_scene(seed, planes, scene_frustum) then oracle_render per camera,
// f64 -> f32 (scenes.cpp:62-171). images: [M,H,W,3] contiguous.
int ref_scene_images_shifted(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr,
                             double shift_x, int64_t M, const lvsg_camera* cams, float* images,
                             char* err, size_t len);

int ref_scene_images(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr, int64_t M,
                     const lvsg_camera* cams, float* images, char* err, size_t len) {
  return ref_scene_images_shifted(seed, planes, scene_fr, 0.0, M, cams, images, err, len);
}

// The same with every plane but the last moved by shift_x along x, then
// PlaneScene::validate (config 4's moving content).
int ref_scene_images_shifted(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr,
                             double shift_x, int64_t M, const lvsg_camera* cams, float* images,
                             char* err, size_t len) {
  return guarded(err, len, [&] {
    PlaneScene sc = make_scene(seed, planes, to_fr(*scene_fr));
    if (shift_x != 0.0) {
      for (size_t i = 0; i + 1 < sc.planes.size(); ++i) {
        sc.planes[i].x0 += shift_x;
        sc.planes[i].x1 += shift_x;
      }
      sc.validate();
    }
    int64_t off = 0;
    for (int64_t m = 0; m < M; ++m) {
      Camera cam = to_cam(cams[m]);
      auto img = oracle_render(sc, cam).first;
      for (int64_t i = 0; i < img.numel(); ++i) images[off + i] = float(img[i]);
      off += img.numel();
    }
  });
}

// forward<float> + render_target<float> with weights bound from a flat store
// in build_params order. Any output pointer may be NULL. Images are
// contiguous [M,H,W,3].
int ref_forward_render_ex(const lvsg_model_config* c, int64_t M, const float* enc_images,
                          int64_t He, int64_t We, const lvsg_camera* enc_cams,
                          const float* render_images, int64_t Hr, int64_t Wr,
                          const lvsg_camera* render_cams, const lvsg_frustum* target,
                          const float* weights, float* rgb, float* depth, float* density,
                          float* blend, float* blend_logits, float* volume, float* deltas,
                          float* rgb_direct, double* seconds, char* err, size_t len);

int ref_forward_render(const lvsg_model_config* c, int64_t M, const float* enc_images,
                       int64_t He, int64_t We, const lvsg_camera* enc_cams,
                       const float* render_images, int64_t Hr, int64_t Wr,
                       const lvsg_camera* render_cams, const lvsg_frustum* target,
                       const float* weights, float* rgb, float* depth, float* density,
                       float* blend, float* blend_logits, float* volume, double* seconds,
                       char* err, size_t len) {
  return ref_forward_render_ex(c, M, enc_images, He, We, enc_cams, render_images, Hr, Wr,
                               render_cams, target, weights, rgb, depth, density, blend,
                               blend_logits, volume, nullptr, nullptr, seconds, err, len);
}

// ... plus ForwardResult.deltas ([L,H,W,M,C]) and ForwardResult.rgb (set
// only under direct_rgb, [Ho,Wo,3]).
int ref_forward_render_ex(const lvsg_model_config* c, int64_t M, const float* enc_images,
                          int64_t He, int64_t We, const lvsg_camera* enc_cams,
                          const float* render_images, int64_t Hr, int64_t Wr,
                          const lvsg_camera* render_cams, const lvsg_frustum* target,
                          const float* weights, float* rgb, float* depth, float* density,
                          float* blend, float* blend_logits, float* volume, float* deltas,
                          float* rgb_direct, double* seconds, char* err, size_t len) {
  return guarded(err, len, [&] {
    ModelConfig cfg = to_cfg(c);
    std::vector<Tensor<float>> shapes = init_param_store<float>(cfg, 0);
    std::vector<Tensor<float>> store;
    int64_t off = 0;
    for (auto& t : shapes) {
      Tensor<float> w(t.shape());
      std::memcpy(w.data(), weights + off, size_t(w.numel()) * sizeof(float));
      off += w.numel();
      store.push_back(std::move(w));
    }
    auto t0 = std::chrono::steady_clock::now();
    Tape<float> tape;
    NetParams p = bind_params(tape, cfg, store);
    std::vector<Var> enc, ren;
    std::vector<Camera> ecams, rcams;
    for (int64_t m = 0; m < M; ++m) {
      Tensor<float> im({He, We, 3});
      std::memcpy(im.data(), enc_images + m * He * We * 3, size_t(He * We * 3) * sizeof(float));
      enc.push_back(tape.constant(std::move(im)));
      ecams.push_back(to_cam(enc_cams[m]));
    }
    ForwardResult<float> r = forward(tape, enc, ecams, to_fr(*target), cfg, p);
    auto t1 = std::chrono::steady_clock::now();
    if (render_images) {
      for (int64_t m = 0; m < M; ++m) {
        Tensor<float> im({Hr, Wr, 3});
        std::memcpy(im.data(), render_images + m * Hr * Wr * 3, size_t(Hr * Wr * 3) * sizeof(float));
        ren.push_back(tape.constant(std::move(im)));
        rcams.push_back(to_cam(render_cams[m]));
      }
      Var out = render_target(tape, r.ldm, ren, rcams);
      copy_out(tape.value(out), rgb);
    }
    auto t2 = std::chrono::steady_clock::now();
    copy_out(tape.value(r.ldm.depth), depth);
    copy_out(tape.value(r.ldm.density), density);
    copy_out(tape.value(r.ldm.blend), blend);
    copy_out(tape.value(r.blend_logits), blend_logits);
    copy_out(tape.value(r.volume.V), volume);
    copy_out(tape.value(r.deltas), deltas);
    if (cfg.direct_rgb) copy_out(tape.value(r.rgb), rgb_direct);
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      seconds[1] = std::chrono::duration<double>(t2 - t1).count();
    }
  });
}

// geo::world_points (geometry.hpp:84-129).
int ref_world_points(const lvsg_frustum* fr, const float* depth, int64_t L, int64_t H, int64_t W,
                     float* points, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    Tensor<float> d({L, H, W});
    std::memcpy(d.data(), depth, size_t(L * H * W) * sizeof(float));
    Var pts = geo::world_points(tape, to_fr(*fr), tape.constant(std::move(d)));
    copy_out(tape.value(pts), points);
  });
}

// geo::gather_backproject (geometry.hpp:138-224). points [P,3].
int ref_gather(const lvsg_camera* cam, const float* image, int64_t Hi, int64_t Wi, int64_t C,
               const float* points, int64_t P, float* values, float* mask, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    Tensor<float> im({Hi, Wi, C});
    std::memcpy(im.data(), image, size_t(Hi * Wi * C) * sizeof(float));
    Tensor<float> pts({1, 1, P, 3});
    std::memcpy(pts.data(), points, size_t(P * 3) * sizeof(float));
    geo::Gather<float> g =
        geo::gather_backproject(tape, tape.constant(std::move(im)), to_cam(*cam),
                                tape.constant(std::move(pts)));
    copy_out(tape.value(g.values), values);
    copy_out(g.mask, mask);
  });
}

// Footprint rule over points (geometry.hpp:34-79, :152-160).
int ref_footprints(const lvsg_camera* cam, const float* points, int64_t P, int32_t* taps,
                   uint8_t* valid, double* fracs, char* err, size_t len) {
  return guarded(err, len, [&] {
    geo::CamPod cp = geo::CamPod::from(to_cam(*cam));
    for (int64_t p = 0; p < P; ++p) {
      double pw[3] = {double(points[p * 3]), double(points[p * 3 + 1]), double(points[p * 3 + 2])};
      double q[3];
      cp.to_cam(pw, q);
      geo::Footprint f{0, 0, 0, 0, 0, 0, false};
      if (q[2] > geo::kZMin) {
        double u = cp.fx * q[0] / q[2] + cp.cx;
        double v = cp.fy * q[1] / q[2] + cp.cy;
        f = geo::footprint(u, v, cp.W, cp.H);
      }
      taps[p * 4 + 0] = int32_t(f.x0);
      taps[p * 4 + 1] = int32_t(f.x1);
      taps[p * 4 + 2] = int32_t(f.y0);
      taps[p * 4 + 3] = int32_t(f.y1);
      valid[p] = f.valid ? 1 : 0;
      fracs[p * 2] = f.fx;
      fracs[p * 2 + 1] = f.fy;
    }
  });
}

// upsample_activate (ldm.hpp:249-271) from a given volume, heads and logits.
int ref_upsample_activate(const lvsg_frustum* fr, const float* V, int64_t L, int64_t H, int64_t W,
                          int64_t C, const float* w_depth, const float* w_sigma,
                          const float* logits, int64_t M, int64_t Ho, int64_t Wo, float* depth,
                          float* density, float* blend, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    auto mk = [&](const float* src, Shape s) {
      Tensor<float> t(s);
      std::memcpy(t.data(), src, size_t(t.numel()) * sizeof(float));
      return tape.constant(std::move(t));
    };
    FeatureVolume<float> fv{mk(V, {L, H, W, C}), 0, to_fr(*fr)};
    DecodeHeads heads{mk(w_sigma, {C, 1}), mk(w_depth, {C, 1}), mk(w_depth, {C, 1})};
    Ldm<float> ldm = upsample_activate(tape, fv, heads, mk(logits, {L, H, W, M}), Ho, Wo);
    copy_out(tape.value(ldm.depth), depth);
    copy_out(tape.value(ldm.density), density);
    copy_out(tape.value(ldm.blend), blend);
  });
}

// attend_residual (attention.hpp:248-252) on V [P,C] in place; deltas
// [P,M,C]; wq: heads x [C,C] contiguous; wo [heads*C, C]; gain [C].
int ref_attend_residual(float* V, const float* deltas, int64_t P, int64_t C, int64_t M,
                        int64_t heads, const float* wq, const float* wo, const float* gain,
                        int zero_scores, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    auto mk = [&](const float* src, Shape s) {
      Tensor<float> t(s);
      std::memcpy(t.data(), src, size_t(t.numel()) * sizeof(float));
      return tape.constant(std::move(t));
    };
    AttendParams ap;
    for (int64_t h = 0; h < heads; ++h) ap.attn.w_q.push_back(mk(wq + h * C * C, {C, C}));
    ap.attn.w_o = mk(wo, {heads * C, C});
    ap.norm_gain = mk(gain, {C});
    ap.zero_scores = zero_scores != 0;
    Var out = attend_residual(tape, mk(V, {P, C}), mk(deltas, {P, M, C}), ap);
    copy_out(tape.value(out), V);
  });
}

// render_to_input_view (ldm.hpp:223-244) of V [L,H,W,C] in the frustum fr
// into camera cam: out [cam.height, cam.width, Ca+1].
int ref_render_to_input_view(const lvsg_frustum* fr, const float* V, int64_t L, int64_t H,
                             int64_t W, int64_t C, int64_t Ca, const float* w_appear,
                             const float* w_sigma, const float* w_depth, const lvsg_camera* cam,
                             float* out, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    auto mk = [&](const float* src, Shape s) {
      Tensor<float> t(s);
      std::memcpy(t.data(), src, size_t(t.numel()) * sizeof(float));
      return tape.constant(std::move(t));
    };
    FeatureVolume<float> fv{mk(V, {L, H, W, C}), 0, to_fr(*fr)};
    DecodeHeads heads{mk(w_sigma, {C, 1}), mk(w_depth, {C, 1}), mk(w_appear, {C, Ca})};
    copy_out(tape.value(render_to_input_view(tape, fv, heads, to_cam(*cam))), out);
  });
}

// render_target (ldm.hpp:193-199) of a given activated LDM. images [M,Hr,Wr,3].
int ref_render_target(const lvsg_frustum* fr, const float* depth, const float* density,
                      const float* blend, int64_t L, int64_t Ho, int64_t Wo, int64_t M,
                      const float* images, int64_t Hr, int64_t Wr, const lvsg_camera* cams,
                      float* rgb, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    auto mk = [&](const float* src, Shape s) {
      Tensor<float> t(s);
      std::memcpy(t.data(), src, size_t(t.numel()) * sizeof(float));
      return tape.constant(std::move(t));
    };
    Ldm<float> ldm;
    ldm.depth = mk(depth, {L, Ho, Wo});
    ldm.density = mk(density, {L, Ho, Wo});
    ldm.blend = mk(blend, {L, Ho, Wo, M});
    ldm.frustum = to_fr(*fr);
    ldm.views = M;
    std::vector<Var> ims;
    std::vector<Camera> cs;
    for (int64_t m = 0; m < M; ++m) {
      ims.push_back(mk(images + m * Hr * Wr * 3, {Hr, Wr, 3}));
      cs.push_back(to_cam(cams[m]));
    }
    copy_out(tape.value(render_target(tape, ldm, ims, cs)), rgb);
  });
}

// model_config_to_json (io.cpp:571-596) into out (NUL-terminated).
int ref_model_config_to_json(const lvsg_model_config* c, char* out, size_t out_len, char* err,
                             size_t len) {
  return guarded(err, len, [&] {
    const std::string j = model_config_to_json(to_cfg(c));
    if (j.size() + 1 > out_len) throw std::runtime_error("ref_model_config_to_json: buffer too small");
    std::memcpy(out, j.c_str(), j.size() + 1);
  });
}

// model_config_from_json (io.cpp:598-633), re-serialised by
// model_config_to_json into out (the parsed config, as text); SchemaError
// and DimError keep their messages in err.
int ref_model_config_roundtrip(const char* text, char* out, size_t out_len, char* err,
                               size_t len) {
  return guarded(err, len, [&] {
    const std::string j = model_config_to_json(model_config_from_json(text));
    if (j.size() + 1 > out_len) throw std::runtime_error("ref_model_config_roundtrip: buffer too small");
    std::memcpy(out, j.c_str(), j.size() + 1);
  });
}

// chw_to_hwc(resize_bilinear(hwc_to_chw(x))) (tape.hpp:629-917) of a
// [B,H,W,C] batch: the input-side decimation of 1080p views.
int ref_resize_hwc(const float* in, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Ho,
                   int64_t Wo, float* out, char* err, size_t len) {
  return guarded(err, len, [&] {
    Tape<float> tape;
    std::vector<float> v(in, in + B * H * W * C);
    Var x = tape.constant(Tensor<float>({B, H, W, C}, std::move(v)));
    copy_out(tape.value(tape.chw_to_hwc(tape.resize_bilinear(tape.hwc_to_chw(x), Ho, Wo))), out);
  });
}

// pack_tensors (io.cpp:100-124) of init_param_store(cfg, seed), entry i
// named by line i of `names` ('\n'-separated). *outlen = bytes needed.
int ref_pack_param_store(const lvsg_model_config* c, uint64_t seed, const char* names, char* out,
                         size_t cap, size_t* outlen, char* err, size_t len) {
  return guarded(err, len, [&] {
    std::vector<Tensor<float>> s = init_param_store<float>(to_cfg(c), seed);
    std::vector<NamedTensor> entries;
    std::string all(names), cur;
    size_t at = 0;
    for (size_t i = 0; i < s.size(); ++i) {
      const size_t nl = all.find('\n', at);
      entries.push_back(NamedTensor::wrap(all.substr(at, nl - at), s[i]));
      at = nl == std::string::npos ? all.size() : nl + 1;
    }
    const std::string b = pack_tensors(entries);
    *outlen = b.size();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  });
}

// pack_tensors(unpack_tensors(in)) (io.cpp:100-171): the reference's
// IoError / SchemaError messages for malformed input.
int ref_qntc_roundtrip(const char* in, size_t n, char* out, size_t cap, size_t* outlen, char* err,
                       size_t len) {
  return guarded(err, len, [&] {
    const std::string b = pack_tensors(unpack_tensors(std::string_view(in, n)));
    *outlen = b.size();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  });
}

}  // extern "C"
