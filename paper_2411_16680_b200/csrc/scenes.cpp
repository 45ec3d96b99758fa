// Synthetic inputs for every BASELINE config: the
// reference's plane-scene generator and exact ray caster, restated on the
// host (not a hot path). Same RNG stream and libm calls as the reference, so
// images are bit-identical to its make_scene + oracle_render:
//   RigSpec::cameras/target   scenes.cpp:40-60
//   make_scene                scenes.cpp:62-120
//   oracle_render             scenes.cpp:122-171
#include <algorithm>
#include <cstdio>
#include <array>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "host.h"

namespace lvsg {
namespace {

uint64_t seed_for(uint64_t seed, const std::string& name) {
  uint64_t h = 14695981039346656037ull;
  for (unsigned char c : name) {
    h ^= c;
    h *= 1099511628211ull;
  }
  uint64_t z = h ^ (seed + 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Rng {
  std::mt19937_64 gen;
  explicit Rng(uint64_t s) : gen(s) {}
  double uniform() { return double(gen() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int64_t index(int64_t n) { return static_cast<int64_t>(gen() % static_cast<uint64_t>(n)); }
};

struct Wave {
  double fu = 0, fv = 0, phase = 0;
  std::array<double, 3> amp{};
};
struct Plane {
  double z = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0, opacity = 1;
  std::array<double, 3> base{};
  std::vector<Wave> waves;
};
struct Scene {
  std::vector<Plane> planes;
  std::array<double, 3> background{};
  double background_depth = 0;
};

std::array<double, 3> tex_eval(const Plane& p, double u, double v) {
  std::array<double, 3> c = p.base;
  for (const Wave& w : p.waves) {
    double s = std::sin(2.0 * M_PI * (w.fu * u + w.fv * v) + w.phase);
    for (int k = 0; k < 3; ++k) c[k] += w.amp[k] * s;
  }
  return c;
}

Scene make_scene(uint64_t seed, int64_t num_planes, const lvsg_frustum& fr) {
  if (num_planes < 1) throw DimError("make_scene: need at least one plane");
  frustum_validate(fr);
  Rng rng(seed_for(seed, "plane-scene"));
  Scene sc;
  double lo = fr.near_depth * 1.1, hi = fr.far_depth * 0.88;
  std::vector<double> zs(static_cast<size_t>(num_planes));
  for (int64_t i = 0; i < num_planes; ++i) {
    double f = (double(i) + 0.5 + 0.3 * rng.uniform(-1.0, 1.0)) / double(num_planes);
    zs[size_t(i)] = 1.0 / (1.0 / hi + f * (1.0 / lo - 1.0 / hi));
  }
  std::sort(zs.begin(), zs.end());
  double minsep = (fr.far_depth - fr.near_depth) * 0.02;
  for (size_t i = 1; i < zs.size(); ++i) zs[i] = std::max(zs[i], zs[i - 1] + minsep);
  const lvsg_camera& cam = fr.camera;
  auto half_w = [&](double z) { return z * (double(cam.width) / 2.0) / cam.fx; };
  auto half_h = [&](double z) { return z * (double(cam.height) / 2.0) / cam.fy; };
  for (int64_t i = 0; i < num_planes; ++i) {
    bool last = i + 1 == num_planes;
    Plane p;
    p.z = zs[size_t(i)];
    double scale = last ? 1.6 : rng.uniform(0.75, 1.35);
    double cxw = last ? 0.0 : rng.uniform(-0.15, 0.15) * half_w(p.z);
    double cyw = last ? 0.0 : rng.uniform(-0.15, 0.15) * half_h(p.z);
    p.x0 = cxw - scale * half_w(p.z);
    p.x1 = cxw + scale * half_w(p.z);
    p.y0 = cyw - scale * half_h(p.z);
    p.y1 = cyw + scale * half_h(p.z);
    p.opacity = last ? 1.0 : rng.uniform(0.5, 1.0);
    for (int k = 0; k < 3; ++k) p.base[size_t(k)] = rng.uniform(0.3, 0.7);
    for (int w = 0; w < 3; ++w) {
      Wave wave;
      wave.fu = double(rng.index(4));
      wave.fv = double(rng.index(4));
      if (wave.fu == 0 && wave.fv == 0) wave.fu = 1;
      wave.phase = rng.uniform(0.0, 2.0 * M_PI);
      for (int k = 0; k < 3; ++k) wave.amp[size_t(k)] = rng.uniform(0.02, 0.25 / 3.0);
      p.waves.push_back(wave);
    }
    sc.planes.push_back(std::move(p));
  }
  for (int k = 0; k < 3; ++k) sc.background[size_t(k)] = rng.uniform(0.25, 0.75);
  sc.background_depth = std::max(zs.back() + minsep, fr.far_depth * 0.93);
  double prev = fr.near_depth;
  for (const Plane& p : sc.planes) {
    if (!(p.z > prev) || !(p.z < fr.far_depth)) throw DimError("PlaneScene: bad plane depths");
    prev = p.z;
  }
  if (!(sc.background_depth > prev && sc.background_depth < fr.far_depth))
    throw DimError("PlaneScene: backdrop must sit behind every plane inside the frustum");
  return sc;
}

// -R^T t and R^T d with k-ascending products (camera.cpp:40-53).
void center_of(const lvsg_camera& c, double o[3]) {
  const double* m = c.cam_from_world;
  for (int r = 0; r < 3; ++r) {
    double acc = (-m[0 * 4 + r]) * m[0 * 4 + 3];
    acc += (-m[1 * 4 + r]) * m[1 * 4 + 3];
    acc += (-m[2 * 4 + r]) * m[2 * 4 + 3];
    o[r] = acc;
  }
}

void render(const Scene& sc, const lvsg_camera& cam, float* img) {
  camera_validate(cam);
  double o[3];
  center_of(cam, o);
  if (o[2] >= sc.planes.front().z)
    throw DimError("oracle_render: camera must sit in front of the nearest plane");
  const double* m = cam.cam_from_world;
  const int64_t H = cam.height, W = cam.width;
  for (int64_t i = 0; i < H; ++i)
    for (int64_t j = 0; j < W; ++j) {
      double dc[3] = {((double(j) + 0.5) - cam.cx) / cam.fx, ((double(i) + 0.5) - cam.cy) / cam.fy, 1.0};
      double d[3];
      for (int r = 0; r < 3; ++r) {
        double acc = m[0 * 4 + r] * dc[0];
        acc += m[1 * 4 + r] * dc[1];
        acc += m[2 * 4 + r] * dc[2];
        d[r] = acc;
      }
      double trans = 1.0, rgb[3] = {0, 0, 0};
      bool opaque = false;
      auto blend = [&](const std::array<double, 3>& c, double a) {
        for (int k = 0; k < 3; ++k) rgb[k] += trans * a * c[size_t(k)];
        if (!opaque && a >= 0.999) opaque = true;
        trans *= 1.0 - a;
      };
      if (std::abs(d[2]) > 1e-12) {
        for (const Plane& p : sc.planes) {
          double t = (p.z - o[2]) / d[2];
          if (t <= 1e-9) continue;
          double x = o[0] + t * d[0], y = o[1] + t * d[1];
          if (!(x >= p.x0 && x <= p.x1 && y >= p.y0 && y <= p.y1)) continue;
          blend(tex_eval(p, (x - p.x0) / (p.x1 - p.x0), (y - p.y0) / (p.y1 - p.y0)), p.opacity);
          if (trans < 1e-12) break;
        }
        if (trans > 0) {
          double t = (sc.background_depth - o[2]) / d[2];
          if (t > 0) blend(sc.background, 1.0);
        }
      }
      for (int k = 0; k < 3; ++k) img[(i * W + j) * 3 + k] = float(rgb[k]);
    }
}

lvsg_status guard(char* err, size_t len, const auto& fn) {
  try {
    fn();
    return LVSG_OK;
  } catch (const DimError& e) {
    if (err && len) std::snprintf(err, len, "%s", e.what());
    return LVSG_ERR_DIM;
  } catch (const std::exception& e) {
    if (err && len) std::snprintf(err, len, "%s", e.what());
    return LVSG_ERR_INTERNAL;
  }
}

}  // namespace
}  // namespace lvsg

extern "C" {

lvsg_status lvsg_rig_cameras(int64_t rows, int64_t cols, double baseline, int64_t width,
                             int64_t height, double focal, lvsg_camera* cams,
                             lvsg_camera* target) {
  return lvsg::guard(nullptr, 0, [&] {
    if (rows < 1 || cols < 1) throw lvsg::DimError("RigSpec: camera grid must be at least 1x1");
    if (!(baseline > 0)) throw lvsg::DimError("RigSpec: baseline must be positive");
    if (width < 1 || height < 1 || !(focal > 0)) throw lvsg::DimError("RigSpec: bad image spec");
    auto make = [&](double x, double y) {
      lvsg_camera c;
      c.fx = c.fy = focal;
      c.cx = double(width) / 2.0;
      c.cy = double(height) / 2.0;
      c.width = width;
      c.height = height;
      std::memset(c.cam_from_world, 0, sizeof(c.cam_from_world));
      for (int k = 0; k < 4; ++k) c.cam_from_world[k * 5] = 1.0;
      // pose_cam_from_world(I, (x, y, 0)): t = -I^T c, k-ascending
      double ctr[3] = {x, y, 0.0};
      for (int r = 0; r < 3; ++r) {
        double acc = (-(r == 0 ? 1.0 : 0.0)) * ctr[0];
        acc += (-(r == 1 ? 1.0 : 0.0)) * ctr[1];
        acc += (-(r == 2 ? 1.0 : 0.0)) * ctr[2];
        c.cam_from_world[r * 4 + 3] = acc;
      }
      return c;
    };
    int64_t n = 0;
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t c = 0; c < cols; ++c) {
        double x = (double(c) - double(cols - 1) / 2.0) * baseline;
        double y = (double(r) - double(rows - 1) / 2.0) * baseline;
        cams[n++] = make(x, y);
      }
    if (target) {
      *target = make(0.0, 0.0);
      for (int r = 0; r < 3; ++r) target->cam_from_world[r * 4 + 3] = 0.0;
    }
  });
}

lvsg_status lvsg_scene_images(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr,
                              int64_t views, const lvsg_camera* cams, float* images, char* err,
                              size_t err_len) {
  return lvsg_scene_images_shifted(seed, planes, scene_fr, 0.0, views, cams, images, err,
                                   err_len);
}

lvsg_status lvsg_scene_images_shifted(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr,
                                      double shift_x, int64_t views, const lvsg_camera* cams,
                                      float* images, char* err, size_t err_len) {
  return lvsg::guard(err, err_len, [&] {
    lvsg::Scene sc = lvsg::make_scene(seed, planes, *scene_fr);
    // Config 4's dynamic content: every plane but the last
    // (the opaque full-coverage wall, scenes.cpp:91-93) moves by shift_x
    // along x; the shifted scene is re-validated (PlaneScene::validate,
    // scenes.cpp:19-32: only depths / extents, which a shift keeps).
    if (shift_x != 0.0)
      for (size_t i = 0; i + 1 < sc.planes.size(); ++i) {
        sc.planes[i].x0 += shift_x;
        sc.planes[i].x1 += shift_x;
        if (!(sc.planes[i].x1 > sc.planes[i].x0))
          throw lvsg::DimError("PlaneScene: empty plane extent");
      }
    int64_t off = 0;
    for (int64_t m = 0; m < views; ++m) {
      lvsg::render(sc, cams[m], images + off);
      off += cams[m].width * cams[m].height * 3;
    }
  });
}

}  // extern "C"
