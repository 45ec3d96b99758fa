// Drop-in check (TEST INFRASTRUCTURE): the reference's own forward +
// render_target next to the same call sequence through include/lvsg_lvs.hpp
// (the adapter a reference maintainer adds), on the nano config with the
// reference's RigSpec / make_scene / init_param_store. Built by
// `make -C oracle ref` into oracle/_ref/adapter_check; run on a B200:
//   oracle/_ref/adapter_check   -> prints max-abs and exits 0 when <= 1e-3
#include <cmath>
#include <cstdio>

#include "../include/lvsg_lvs.hpp"
#include "lvs/scenes.hpp"

using namespace lvs;

int main() {
  ModelConfig cfg = nano_config();
  RigSpec rig{2, 2, 0.05, 64, 64, 64.0};
  std::vector<Camera> cams = rig.cameras();
  Frustum target{Camera::make(64, 64, 32, 32, 64, 64, Eigen::Matrix4d::Identity()), 1.0, 6.0};
  PlaneScene scene = make_scene(21, 3, target);
  std::vector<Tensor<float>> images;
  for (const Camera& c : cams) images.push_back(oracle_render(scene, c).first.cast<float>());
  std::vector<Tensor<float>> store = init_param_store<float>(cfg, 3);

  // reference
  Tape<float> tape;
  NetParams p = bind_params(tape, cfg, store);
  std::vector<Var> iv;
  for (const auto& im : images) iv.push_back(tape.constant(im));
  ForwardResult<float> r = forward(tape, iv, cams, target, cfg, p);
  Tensor<float> want = tape.value(render_target(tape, r.ldm, iv, cams));

  // the same calls through the B200 adapter
  try {
    gpu::Model m(cfg, 0);
    m.bind(store);
    gpu::Ldm ldm = m.forward(images, cams, target);
    Tensor<float> got = m.render_target(images, cams);
    double err = 0, derr = 0;
    for (int64_t i = 0; i < got.numel(); ++i) err = std::max(err, double(std::fabs(got[i] - want[i])));
    const Tensor<float>& wd = tape.value(r.ldm.depth);
    for (int64_t i = 0; i < wd.numel(); ++i)
      derr = std::max(derr, double(std::fabs(ldm.depth[i] - wd[i]) / wd[i]));
    std::printf("adapter_check: rgb max-abs %.3e, LDM depth max-rel %.3e\n", err, derr);
    bool bad_caught = false;
    try {
      m.forward(std::vector<Tensor<float>>(images.begin(), images.begin() + 3),
                std::vector<Camera>(cams.begin(), cams.begin() + 3), target);
    } catch (const DimError&) {
      bad_caught = true;
    }
    std::printf("adapter_check: wrong view count -> DimError: %s\n", bad_caught ? "yes" : "no");
    return (err <= 1e-3 && bad_caught) ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("adapter_check: %s\n", e.what());
    return 2;
  }
}
