// Host-side runtime pieces of liblvsg: config grammar + validation, forward
// planning, the build_params weight layout, the bit-exact init RNG, and the
// synthetic scene generator. Pure C++ (no CUDA).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lvsg.h"

namespace lvsg {

struct DimError : std::runtime_error {
  explicit DimError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericError : std::runtime_error {
  explicit NumericError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

enum class Tok { backproject, update, collapse, attend, conv };
struct Token {
  Tok kind;
  int64_t heads;
};

struct Step {
  int64_t in_layers, layers, height, width, pyramid_level;
  std::string blocks;
};

struct Config {
  std::vector<Step> steps;
  int64_t channels = 0, views = 0, pyramid_levels = 0;
  double upsample = 1.0, near_depth = 0, far_depth = 0;
  bool ablate_render = false, ablate_attention = false, ablate_rays = false, direct_rgb = false;

  static Config from_c(const lvsg_model_config* c);
  void validate() const;
  int64_t appear_channels() const { return direct_rgb ? 3 : channels; }
};

std::vector<Token> parse_blocks(const std::string& spec);

struct StepPlan {
  int64_t in_layers, layers, in_height, in_width, height, width;
  bool doubled;
  int64_t level, feat_h, feat_w, render_h, render_w;
  std::vector<Token> tokens;
  int64_t collapse_count;
};

struct Plan {
  std::vector<std::pair<int64_t, int64_t>> pyramid;
  std::vector<StepPlan> steps;
  int64_t out_height = 0, out_width = 0;
};

Plan plan_forward(const Config& cfg, int64_t image_h, int64_t image_w);

// One learnable tensor of build_params (network.hpp:244-317).
enum class Init { normal, zeros, ones };
struct ParamSpec {
  std::vector<int64_t> shape;
  Init init;
  double scale;
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
};
std::vector<ParamSpec> param_layout(const Config& cfg);

// init_param_store<float> (network.hpp:354-362), bit-exact.
void init_param_store(const Config& cfg, uint64_t seed, float* out);

// Camera helpers (camera.cpp) on the POD type.
lvsg_camera camera_scaled(const lvsg_camera& c, int64_t w, int64_t h);
void camera_validate(const lvsg_camera& c);
void frustum_validate(const lvsg_frustum& f);

}  // namespace lvsg
