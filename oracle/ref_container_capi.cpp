// TEST INFRASTRUCTURE (oracle): C entry points over the reference's OWN
// container.cpp (serialize_ocw / deserialize_ocw, src/container.cpp:123-199,
// 278-373), compiled unmodified by oracle/build_ref.sh against the
// nlohmann/json 3.11.3 header the image ships (the reference expects it in
// proj/vendor/, absent here).  Only tests/ may load this library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ocw/container.hpp"
#include "ocw/quant.hpp"

namespace {
std::string g_err;

ocw::QuantConfig cfg_of(int bits, int scheme, int gran, size_t group) {
  ocw::QuantConfig c;
  c.bits = bits;
  c.scheme = scheme == 1 ? ocw::Scheme::asymmetric : ocw::Scheme::symmetric;
  c.granularity = gran == 0   ? ocw::Granularity::per_tensor
                  : gran == 1 ? ocw::Granularity::per_channel
                              : ocw::Granularity::per_group;
  c.group_size = group;
  return c;
}

int put_out(const std::vector<uint8_t>& b, uint8_t* out, size_t cap, size_t* len) {
  *len = b.size();
  if (b.size() > cap) return 5;
  if (!b.empty()) std::memcpy(out, b.data(), b.size());
  return 0;
}
}  // namespace

extern "C" {
const char* ocwref_container_error() { return g_err.c_str(); }

// Records: kind 0 = f32 (from_f32), 1 = uniform (from_uniform) -- container.cpp:270-289.
int ocwref_serialize_ocw(int k, const char* const* names, const int* kind, const size_t* rows,
                         const size_t* cols, const int* bits, const int* scheme, const int* gran,
                         const size_t* group, const float* const* f32, const int16_t* const* codes,
                         const float* const* scales, const int32_t* const* zeros,
                         const char* meta_json, uint8_t* out, size_t cap, size_t* len) {
  try {
    ocw::OcwContainer c;
    c.meta = meta_json ? nlohmann::json::parse(meta_json) : nlohmann::json::object();
    for (int i = 0; i < k; ++i) {
      if (kind[i] == 0) {
        ocw::Matrix m(rows[i], cols[i]);
        std::memcpy(m.data.data(), f32[i], rows[i] * cols[i] * sizeof(float));
        c.tensors.push_back(ocw::TensorRecord::from_f32(names[i], m));
      } else {
        ocw::QuantizedMatrix q;
        q.rows = rows[i];
        q.cols = cols[i];
        q.config = cfg_of(bits[i], scheme[i], gran[i], group[i]);
        q.codes.assign(codes[i], codes[i] + rows[i] * cols[i]);
        const size_t ng = ocw::quant_group_count(q.config, rows[i], cols[i]);
        q.grids.resize(ng);
        for (size_t g = 0; g < ng; ++g) {
          q.grids[g].scale = scales[i][g];
          q.grids[g].zero_point = zeros[i][g];
          q.grids[g].qmin = ocw::scheme_qmin(q.config.bits, q.config.scheme);
          q.grids[g].qmax = ocw::scheme_qmax(q.config.bits, q.config.scheme);
        }
        c.tensors.push_back(ocw::TensorRecord::from_uniform(names[i], q));
      }
    }
    return put_out(ocw::serialize_ocw(c), out, cap, len);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// serialize_ocw(deserialize_ocw(bytes)): the reference's parser on a file.
int ocwref_roundtrip_ocw(const uint8_t* in, size_t n, uint8_t* out, size_t cap, size_t* len) {
  try {
    return put_out(ocw::serialize_ocw(ocw::deserialize_ocw(std::vector<uint8_t>(in, in + n))),
                   out, cap, len);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // extern "C"
