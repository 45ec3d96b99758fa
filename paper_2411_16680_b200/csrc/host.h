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
// io.hpp:20-31: corrupt / truncated containers (exit 3) and content that
// does not fit the expected schema (exit 1, like DimError).
struct IoError : std::runtime_error {
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct SchemaError : std::runtime_error {
  explicit SchemaError(const std::string& m) : std::runtime_error(m) {}
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
  // NetParams member path, e.g. "encoder.levels.0.res1.w1" (network.hpp:95-132)
  std::string name;
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
};
std::vector<ParamSpec> param_layout(const Config& cfg);

// QNTC named-tensor container (io.hpp:33-60, io.cpp:100-171): "QNTC", u32
// version 1, u32 count, then per entry u32 name length, name, u8 dtype
// (0 f32, 1 f64), u32 rank, u64 dims, little-endian payload.
struct QntcEntry {
  std::string name;
  uint8_t dtype = 0;  // 0 f32, 1 f64
  std::vector<int64_t> dims;
  const uint8_t* payload = nullptr;  // points into the parsed buffer
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : dims) n *= d;
    return n;
  }
};
// Throws IoError with the reference's messages on a malformed container.
std::vector<QntcEntry> qntc_unpack(const uint8_t* bytes, size_t len);
// Appends one f32 entry.
void qntc_put_f32(std::string& out, const std::string& name, const std::vector<int64_t>& dims,
                  const float* data);
std::string qntc_header(uint32_t count);

// init_param_store<float> (network.hpp:354-362), bit-exact.
void init_param_store(const Config& cfg, uint64_t seed, float* out);

// Camera helpers (camera.cpp) on the POD type.
lvsg_camera camera_scaled(const lvsg_camera& c, int64_t w, int64_t h);
void camera_validate(const lvsg_camera& c);
void frustum_validate(const lvsg_frustum& f);

}  // namespace lvsg
