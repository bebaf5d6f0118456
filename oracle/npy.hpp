// Minimal .npy (format 1.0) writer/reader for golden fixtures. Test
// infrastructure only: used by oracle/ref_driver.cpp.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace npyio {

template <typename T> const char* descr();
template <> inline const char* descr<std::uint8_t>() { return "|u1"; }
template <> inline const char* descr<std::int32_t>() { return "<i4"; }
template <> inline const char* descr<std::uint16_t>() { return "<u2"; }
template <> inline const char* descr<std::uint32_t>() { return "<u4"; }
template <> inline const char* descr<std::int64_t>() { return "<i8"; }
template <> inline const char* descr<std::uint64_t>() { return "<u8"; }
template <> inline const char* descr<double>() { return "<f8"; }

template <typename T>
void save(const std::string& path, const T* data, const std::vector<std::size_t>& shape) {
  std::string dict = std::string("{'descr': '") + descr<T>() + "', 'fortran_order': False, 'shape': (";
  std::size_t count = 1;
  for (std::size_t d = 0; d < shape.size(); ++d) {
    dict += std::to_string(shape[d]);
    dict += (shape.size() == 1 || d + 1 < shape.size()) ? "," : "";
    if (d + 1 < shape.size()) dict += " ";
    count *= shape[d];
  }
  dict += "), }";
  const std::size_t preamble = 10;
  std::size_t total = preamble + dict.size() + 1;
  const std::size_t padded = (total + 63) / 64 * 64;
  dict.append(padded - total, ' ');
  dict.push_back('\n');
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open " + path);
  const unsigned char magic[8] = {0x93, 'N', 'U', 'M', 'P', 'Y', 1, 0};
  std::fwrite(magic, 1, 8, f);
  const std::uint16_t hlen = static_cast<std::uint16_t>(dict.size());
  std::fwrite(&hlen, 2, 1, f);
  std::fwrite(dict.data(), 1, dict.size(), f);
  if (count) std::fwrite(data, sizeof(T), count, f);
  std::fclose(f);
}

template <typename T>
void save(const std::string& path, const std::vector<T>& v) {
  save(path, v.data(), {v.size()});
}

}  // namespace npyio
