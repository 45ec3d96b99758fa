// QNTC named-tensor container codec (the reference's pack_tensors /
// unpack_tensors, io.cpp:100-171) and its weight hand-off entry points:
// a parameter store written by the reference side (NamedTensor::wrap of every
// leaf in build_params order, network.hpp:244-317) loads through
// lvsg_load_weights_qntc exactly as bind_params (network.hpp:330-339) binds a
// store: by position, shapes checked, names carried but not used for binding.
#include <cstring>
#include <string>
#include <vector>

#include "host.h"

namespace lvsg {
namespace {

constexpr uint32_t kVersion = 1;  // kTensorContainerVersion (io.hpp:44)

// Bounds-checked little-endian cursor; every short read names what it was
// reading ("tensor container: truncated <what>").
class Cursor {
 public:
  Cursor(const uint8_t* p, size_t n) : p_(p), n_(n) {}
  const uint8_t* span(size_t k, const std::string& what) {
    if (k > n_ - at_) throw IoError("tensor container: truncated " + what);
    const uint8_t* s = p_ + at_;
    at_ += k;
    return s;
  }
  template <typename T>
  T get(const std::string& what) {
    T v;
    std::memcpy(&v, span(sizeof(T), what), sizeof(T));
    return v;
  }
  size_t left() const { return n_ - at_; }

 private:
  const uint8_t* p_;
  size_t n_, at_ = 0;
};

template <typename T>
void put(std::string& o, T v) {
  o.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

}  // namespace

std::vector<QntcEntry> qntc_unpack(const uint8_t* bytes, size_t len) {
  Cursor c(bytes, len);
  const uint8_t* m = c.span(4, "magic");
  const std::string magic(reinterpret_cast<const char*>(m), 4);
  if (magic != "QNTC") throw IoError("tensor container: bad magic \"" + magic + "\"");
  const uint32_t version = c.get<uint32_t>("version");
  if (version != kVersion)
    throw IoError("tensor container: unsupported version " + std::to_string(version));
  const uint32_t count = c.get<uint32_t>("entry count");
  if (count > (1u << 20)) throw IoError("tensor container: implausible entry count");
  std::vector<QntcEntry> out(count);
  for (uint32_t i = 0; i < count; ++i) {
    QntcEntry& e = out[i];
    const std::string at = "entry " + std::to_string(i);
    const uint32_t nl = c.get<uint32_t>(at + " name length");
    if (nl > (1u << 16)) throw IoError("tensor container: " + at + ": implausible name length");
    e.name.assign(reinterpret_cast<const char*>(c.span(nl, at + " name")), nl);
    e.dtype = c.get<uint8_t>(at + " dtype");
    if (e.dtype > 1)
      throw IoError("tensor container: " + at + " (\"" + e.name + "\"): unknown dtype tag " +
                    std::to_string(int(e.dtype)));
    const uint32_t rank = c.get<uint32_t>(at + " rank");
    if (rank > 16) throw IoError("tensor container: " + at + ": implausible rank");
    int64_t n = 1;
    for (uint32_t d = 0; d < rank; ++d) {
      const uint64_t ext = c.get<uint64_t>(at + " dims");
      if (ext > (uint64_t(1) << 32)) throw IoError("tensor container: " + at + ": implausible extent");
      e.dims.push_back(int64_t(ext));
      n *= int64_t(ext);
      if (n > (int64_t(1) << 33))
        throw IoError("tensor container: " + at + ": implausible element count");
    }
    e.payload = c.span(size_t(n) * (e.dtype ? 8 : 4), at + " (\"" + e.name + "\") payload");
  }
  if (c.left())
    throw IoError("tensor container: " + std::to_string(c.left()) +
                  " trailing bytes after the last entry");
  return out;
}

std::string qntc_header(uint32_t count) {
  std::string o = "QNTC";
  put<uint32_t>(o, kVersion);
  put<uint32_t>(o, count);
  return o;
}

void qntc_put_f32(std::string& o, const std::string& name, const std::vector<int64_t>& dims,
                  const float* data) {
  put<uint32_t>(o, uint32_t(name.size()));
  o += name;
  put<uint8_t>(o, 0);
  put<uint32_t>(o, uint32_t(dims.size()));
  int64_t n = 1;
  for (int64_t d : dims) {
    put<uint64_t>(o, uint64_t(d));
    n *= d;
  }
  o.append(reinterpret_cast<const char*>(data), size_t(n) * sizeof(float));
}

}  // namespace lvsg

using namespace lvsg;

extern "C" {

lvsg_status lvsg_param_name(const lvsg_model_config* cfg, int64_t index, char* out, size_t len) {
  try {
    const auto lay = param_layout(Config::from_c(cfg));
    if (index < 0 || index >= int64_t(lay.size()) || !out || lay[index].name.size() + 1 > len)
      return LVSG_ERR_DIM;
    std::memcpy(out, lay[index].name.c_str(), lay[index].name.size() + 1);
    return LVSG_OK;
  } catch (const std::exception&) {
    return LVSG_ERR_DIM;
  }
}

lvsg_status lvsg_pack_param_store_qntc(const lvsg_model_config* cfg, uint64_t seed, void* out,
                                       size_t cap, size_t* len) {
  try {
    const Config c = Config::from_c(cfg);
    const auto lay = param_layout(c);
    int64_t total = 0;
    for (const auto& p : lay) total += p.numel();
    std::vector<float> flat(static_cast<size_t>(total));
    init_param_store(c, seed, flat.data());
    std::string o = qntc_header(uint32_t(lay.size()));
    int64_t off = 0;
    for (const auto& p : lay) {
      qntc_put_f32(o, p.name, p.shape, flat.data() + off);
      off += p.numel();
    }
    if (len) *len = o.size();
    if (!out) return LVSG_OK;
    if (cap < o.size()) return LVSG_ERR_DIM;
    std::memcpy(out, o.data(), o.size());
    return LVSG_OK;
  } catch (const std::exception&) {
    return LVSG_ERR_DIM;
  }
}

}  // extern "C"
