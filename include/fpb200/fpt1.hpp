// fpb200/fpt1.hpp — the reference's FPT1 tensor container (tensor.hpp:97-221), host side.
//
// Little-endian: magic "FPT1" | u32 version = 1 | u32 ndim (1..8) | ndim x u64 dims (each >= 1) |
// u32 dtype (0 f32, 1 i32) | row-major payload.  Loading rejects, like the reference: bad magic,
// version, ndim, zero dims, shape overflow, dtype mismatch, truncation and trailing bytes
// (FormatError); non-finite f32 payloads (ValidationError); unopenable paths (IoError).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <type_traits>
#include <vector>

#include "bsattn.hpp"

namespace fpb200 {

namespace fpt1 {

template <typename T>
constexpr std::uint32_t dtype_code() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, std::int32_t>, "f32 or i32");
  return std::is_same_v<T, float> ? 0u : 1u;
}

inline void put_u32(std::ostream& o, std::uint32_t v) {
  unsigned char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  o.write(reinterpret_cast<const char*>(b), 4);
}
inline void put_u64(std::ostream& o, std::uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  o.write(reinterpret_cast<const char*>(b), 8);
}
inline void get(std::istream& in, void* dst, std::size_t n, const char* what) {
  in.read(static_cast<char*>(dst), static_cast<std::streamsize>(n));
  if (static_cast<std::size_t>(in.gcount()) != n)
    throw FormatError(std::string("truncated container while reading ") + what);
}
inline std::uint32_t get_u32(std::istream& in, const char* what) {
  unsigned char b[4];
  get(in, b, 4, what);
  return std::uint32_t(b[0]) | std::uint32_t(b[1]) << 8 | std::uint32_t(b[2]) << 16 |
         std::uint32_t(b[3]) << 24;
}
inline std::uint64_t get_u64(std::istream& in, const char* what) {
  unsigned char b[8];
  get(in, b, 8, what);
  std::uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = v << 8 | b[i];
  return v;
}

}  // namespace fpt1

template <typename T>
void save_tensor(const Tensor<T>& t, const std::string& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open for writing: " + path);
  out.write("FPT1", 4);
  fpt1::put_u32(out, 1);
  fpt1::put_u32(out, static_cast<std::uint32_t>(t.ndim()));
  for (auto d : t.shape()) fpt1::put_u64(out, d);
  fpt1::put_u32(out, fpt1::dtype_code<T>());
  out.write(reinterpret_cast<const char*>(t.data()), static_cast<std::streamsize>(t.numel() * 4));
  out.flush();
  if (!out) throw IoError("write failed: " + path);
}

template <typename T>
Tensor<T> load_tensor(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open: " + path);
  char magic[4];
  fpt1::get(in, magic, 4, "magic");
  if (std::memcmp(magic, "FPT1", 4) != 0) throw FormatError("bad magic: " + path);
  if (fpt1::get_u32(in, "version") != 1) throw FormatError("unsupported container version: " + path);
  const std::uint32_t ndim = fpt1::get_u32(in, "ndim");
  if (ndim == 0 || ndim > 8) throw FormatError("malformed ndim: " + path);
  std::vector<std::uint64_t> shape(ndim);
  std::uint64_t numel = 1;
  for (auto& d : shape) {
    d = fpt1::get_u64(in, "dims");
    if (d == 0) throw FormatError("zero dimension: " + path);
    if (numel > std::numeric_limits<std::uint64_t>::max() / d)
      throw FormatError("shape overflow: " + path);
    numel *= d;
  }
  if (fpt1::get_u32(in, "dtype") != fpt1::dtype_code<T>()) throw FormatError("dtype mismatch: " + path);
  Tensor<T> t(std::move(shape));
  fpt1::get(in, t.data(), t.numel() * 4, "payload");
  if (in.peek() != std::ifstream::traits_type::eof())
    throw FormatError("trailing bytes after payload: " + path);
  if constexpr (std::is_same_v<T, float>)
    for (std::size_t i = 0; i < t.numel(); ++i)
      if (!std::isfinite(t.data()[i])) throw ValidationError("non-finite payload value: " + path);
  return t;
}

}  // namespace fpb200
