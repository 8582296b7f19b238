// mttkrp_b200/frostt.hpp — drop-in for the reference's FROSTT I/O
// (/root/reference/proj/core/include/mttkrp/frostt.hpp) on top of the multithreaded host
// ingest of the C ABI (mk_frostt_*, csrc/frostt.cpp), plus the binary tensor cache.
//
// Same names, options, results and error texts as the reference:
//   FrosttOptions, FrosttParseResult            frostt.hpp:22-35
//   parse_frostt(istream | string_view)         frostt.hpp:74-163
//   write_frostt / write_frostt_string          frostt.hpp:165-192
//   read_frostt_file / write_frostt_file        frostt.hpp:194-206
// Additions: save_tensor_cache / load_tensor_cache / load_tensor (binary cache "MKBT").
#pragma once

#include <filesystem>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "mttkrp_b200/mttkrp.hpp"

namespace mttkrp_b200 {

struct FrosttOptions {
  bool merge_duplicates = true;
  std::vector<index_t> dims_override;
};

template <typename T>
struct FrosttParseResult {
  SparseTensorCOO<T> tensor;
  std::size_t duplicates_merged = 0;
};

namespace detail {
constexpr int prec_of(float) { return 32; }
constexpr int prec_of(double) { return 64; }

template <typename T>
FrosttParseResult<T> take_host_tensor(mk_host_tensor* h) {
  struct Free {
    mk_host_tensor* h;
    ~Free() { mk_host_tensor_free(h); }
  } guard{h};
  uint32_t n = 0;
  uint64_t nnz = 0, dups = 0;
  int prec = 0;
  check(mk_host_tensor_info(h, &n, nullptr, 0, &nnz, &dups, &prec));
  if (prec != prec_of(T{})) throw error("frostt: value precision mismatch");
  std::vector<index_t> dims(n);
  std::vector<index_t> coords(static_cast<std::size_t>(nnz) * n);
  std::vector<T> vals(nnz);
  check(mk_host_tensor_info(h, nullptr, dims.data(), n, nullptr, nullptr, nullptr));
  check(mk_host_tensor_export(h, coords.data(), vals.data()));
  return {SparseTensorCOO<T>::from_parts(Shape(std::move(dims)), std::move(coords),
                                         std::move(vals)),
          static_cast<std::size_t>(dups)};
}
}  // namespace detail

template <typename T = float>
FrosttParseResult<T> parse_frostt(std::string_view text, const FrosttOptions& opt = {}) {
  mk_host_tensor* h = nullptr;
  detail::check(mk_frostt_parse(text.data(), text.size(), detail::prec_of(T{}),
                                opt.merge_duplicates ? 1 : 0, opt.dims_override.data(),
                                static_cast<uint32_t>(opt.dims_override.size()), 0, &h));
  return detail::take_host_tensor<T>(h);
}

template <typename T = float>
FrosttParseResult<T> parse_frostt(std::istream& in, const FrosttOptions& opt = {}) {
  const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
  return parse_frostt<T>(std::string_view(text), opt);
}

template <typename T = float>
FrosttParseResult<T> read_frostt_file(const std::filesystem::path& path,
                                      const FrosttOptions& opt = {}) {
  mk_host_tensor* h = nullptr;
  detail::check(mk_frostt_read_file(path.c_str(), detail::prec_of(T{}),
                                    opt.merge_duplicates ? 1 : 0, opt.dims_override.data(),
                                    static_cast<uint32_t>(opt.dims_override.size()), 0, &h));
  return detail::take_host_tensor<T>(h);
}

template <typename T>
std::string write_frostt_string(const SparseTensorCOO<T>& t) {
  uint64_t len = 0;
  const auto n = static_cast<uint32_t>(t.mode_count());
  detail::check(mk_frostt_format(n, t.nnz(), t.coord_data(), t.values().data(),
                                 detail::prec_of(T{}), 0, nullptr, 0, &len));
  std::string s(len, '\0');
  detail::check(mk_frostt_format(n, t.nnz(), t.coord_data(), t.values().data(),
                                 detail::prec_of(T{}), 0, s.data(), len, &len));
  return s;
}

template <typename T>
void write_frostt(const SparseTensorCOO<T>& t, std::ostream& out) {
  const std::string s = write_frostt_string(t);
  out.write(s.data(), static_cast<std::streamsize>(s.size()));
  if (!out) throw error("frostt: write failed");
}

template <typename T>
void write_frostt_file(const SparseTensorCOO<T>& t, const std::filesystem::path& path) {
  detail::check(mk_frostt_write_file(path.c_str(), static_cast<uint32_t>(t.mode_count()), t.nnz(),
                                     t.coord_data(), t.values().data(), detail::prec_of(T{}), 0));
}

// ---- binary tensor cache (no reference counterpart) -------------------------------------
template <typename T>
void save_tensor_cache(const SparseTensorCOO<T>& t, const std::filesystem::path& path) {
  detail::check(mk_tensor_cache_write(path.c_str(), static_cast<uint32_t>(t.mode_count()),
                                      t.shape().dims.data(), t.nnz(), t.coord_data(),
                                      t.values().data(), detail::prec_of(T{})));
}

template <typename T = float>
SparseTensorCOO<T> load_tensor_cache(const std::filesystem::path& path) {
  mk_host_tensor* h = nullptr;
  detail::check(mk_tensor_cache_read(path.c_str(), &h));
  return std::move(detail::take_host_tensor<T>(h).tensor);
}

// A FROSTT file through `<path>.mkbt`: used when newer than the text and of the same
// precision, else the text is parsed and the cache (re)written (best effort).
template <typename T = float>
FrosttParseResult<T> load_tensor(const std::filesystem::path& path) {
  namespace fs = std::filesystem;
  const fs::path cache = fs::path(path.string() + ".mkbt");
  std::error_code ec;
  if (fs::exists(cache, ec) && fs::last_write_time(cache, ec) >= fs::last_write_time(path, ec) &&
      !ec) {
    try {
      return {load_tensor_cache<T>(cache), 0};
    } catch (const error&) {
      // stale, corrupt or other-precision cache: parse below
    }
  }
  auto res = read_frostt_file<T>(path);
  try {
    save_tensor_cache(res.tensor, cache);
  } catch (const error&) {
  }
  return res;
}

}  // namespace mttkrp_b200
