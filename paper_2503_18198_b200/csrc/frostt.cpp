// Host-side tensor ingest: a multithreaded FROSTT `.tns` reader/writer and a
// binary tensor cache, behind the C ABI so the Python package and the C++ drop-in host share
// one implementation.
//
// Semantics follow the reference's sequential parser exactly (frostt.hpp:74-160): same
// tokenisation (whitespace-separated, `#` comment lines and blank lines skipped, 1-based
// indices, std::from_chars with chars_format::general for the value in the target precision),
// same error texts with the same line numbers, duplicates merged by summing in file order into
// the first occurrence (or rejected at the second occurrence's line), extents inferred as the
// largest index per mode unless overridden.  Only the execution differs:
//
//   1. the file is read whole and cut into per-thread chunks at newline boundaries;
//   2. every thread parses its chunk into chunk-local arrays and records its first error;
//   3. the earliest error (in file order) wins; elements before it are kept, because a
//      strict-mode duplicate earlier in the file must still be reported first;
//   4. duplicates are found per hash bucket: elements are scattered by (hash mod buckets) in
//      file order, and each thread owns whole buckets, so every tuple's occurrences are seen
//      by one thread in file order (summation order = the reference's);
//   5. survivors are compacted in file order.
//
// The writer prints the reference's format (frostt.hpp:165-186: 1-based indices, shortest
// round-trip decimal via std::to_chars) with chunks formatted in parallel and written in order.
//
// Binary cache ("MKBT" v1): header {magic, version, n_modes, value bits, nnz, dims[n]}, then the
// AoS coordinates (u32) and values, then a 64-bit checksum of the payload.  Loading it skips the
// text parse entirely (the 77M-nnz config's text is ~2 GB).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <string_view>
#include <system_error>
#include <thread>
#include <vector>

#include "mttkrp_b200.h"

namespace mkb {
std::string& last_error_ref();
}

struct mk_host_tensor {
  uint32_t n = 0;
  int prec = 32;
  std::vector<uint32_t> dims;
  std::vector<uint32_t> coords;  // AoS, nnz * n
  std::vector<float> v32;
  std::vector<double> v64;
  uint64_t duplicates = 0;
  uint64_t nnz() const { return prec == 64 ? v64.size() : v32.size(); }
};

namespace {

constexpr uint64_t kMaxExtent = std::numeric_limits<uint32_t>::max();  // types.hpp:16
constexpr uint32_t kMaxModes = 64;

struct IngestError {
  int status;
  std::string msg;
};

[[noreturn]] void fail(std::string msg, int status = MK_EINVAL) {
  throw IngestError{status, std::move(msg)};
}

template <typename F>
int run(F&& f) {
  try {
    f();
    return MK_OK;
  } catch (const IngestError& e) {
    mkb::last_error_ref() = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    mkb::last_error_ref() = "frostt: host allocation failed";
    return MK_ENOMEM;
  } catch (const std::exception& e) {
    mkb::last_error_ref() = e.what();
    return MK_EINVAL;
  }
}

// threads for `work` units: all hardware threads with at least per_thread_min units each, or
// exactly `requested` (bounded by the work) when the caller asks (tests force chunking this way)
unsigned thread_count(uint32_t requested, uint64_t work, uint64_t per_thread_min) {
  if (requested) return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(requested, work)));
  unsigned hw = std::thread::hardware_concurrency();
  if (!hw) hw = 1;
  const uint64_t cap = std::max<uint64_t>(1, work / std::max<uint64_t>(per_thread_min, 1));
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(hw, cap)));
}

template <typename F>
void parallel_for(unsigned threads, F&& f) {
  if (threads <= 1) {
    f(0u);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads - 1);
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back([&f, t] { f(t); });
  f(0u);
  for (auto& th : pool) th.join();
}

inline bool is_space(char c) {  // std::isspace in the "C" locale (split_tokens, frostt.hpp:41-49)
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// ------------------------------------------------------------------------------------- parse
struct ChunkOut {
  std::vector<uint32_t> coords;
  std::vector<double> vals;      // parsed in the target precision, widened exactly for storage
  std::vector<uint64_t> line;    // chunk-local 1-based line of each element
  std::vector<uint64_t> maxidx;  // 1-based max per mode
  uint64_t lines = 0;            // lines in the chunk
  bool err = false;
  uint64_t err_line = 0;         // chunk-local
  std::string err_msg;           // without the "frostt: line N: " prefix
};

template <typename T>
void parse_chunk(const char* p, const char* end, uint32_t n, ChunkOut& out) {
  out.maxidx.assign(n, 0);
  std::string_view toks[kMaxModes + 2];
  uint64_t line_no = 0;
  while (p < end) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', end - p));
    const char* le = nl ? nl : end;
    ++line_no;
    const char* q = p;
    p = nl ? nl + 1 : end;
    while (q < le && is_space(*q)) ++q;
    if (q == le || *q == '#') continue;
    size_t nt = 0;
    bool too_many = false;
    while (q < le) {
      const char* s = q;
      while (q < le && !is_space(*q)) ++q;
      if (nt < n + 2) toks[nt] = std::string_view(s, q - s);
      else too_many = true;
      ++nt;
      while (q < le && is_space(*q)) ++q;
    }
    (void)too_many;
    auto error = [&](std::string msg) {
      out.err = true;
      out.err_line = line_no;
      out.err_msg = std::move(msg);
    };
    if (nt != n + 1) {
      error("expected " + std::to_string(n + 1) + " tokens, got " + std::to_string(nt));
      break;
    }
    const size_t base = out.coords.size();
    bool bad = false;
    for (uint32_t h = 0; h < n; ++h) {
      const std::string_view tok = toks[h];
      uint64_t raw = 0;
      auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), raw);
      if (ec != std::errc{} || ptr != tok.data() + tok.size()) {
        error("non-numeric index token '" + std::string(tok) + "'");
        bad = true;
        break;
      }
      if (raw < 1) {
        error("index " + std::to_string(raw) + " < 1 (indices are 1-based)");
        bad = true;
        break;
      }
      if (raw > kMaxExtent) {
        error("index " + std::to_string(raw) + " exceeds the 32-bit coordinate range");
        bad = true;
        break;
      }
      out.maxidx[h] = std::max(out.maxidx[h], raw);
      out.coords.push_back(static_cast<uint32_t>(raw - 1));
    }
    if (bad) {
      out.coords.resize(base);
      break;
    }
    const std::string_view vt = toks[n];
    T v{};
    auto [ptr, ec] =
        std::from_chars(vt.data(), vt.data() + vt.size(), v, std::chars_format::general);
    if (ec != std::errc{} || ptr != vt.data() + vt.size()) {
      out.coords.resize(base);
      error("bad value token '" + std::string(vt) + "'");
      break;
    }
    if (!std::isfinite(static_cast<double>(v))) {
      out.coords.resize(base);
      error("non-finite value");
      break;
    }
    out.vals.push_back(static_cast<double>(v));
    out.line.push_back(line_no);
  }
  out.lines = line_no;
}

// first element line of the text: decides the mode count (frostt.hpp:96-103)
bool first_element_line(const char* p, const char* end, uint64_t& line_no, size_t& ntok) {
  line_no = 0;
  while (p < end) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', end - p));
    const char* le = nl ? nl : end;
    ++line_no;
    const char* q = p;
    p = nl ? nl + 1 : end;
    while (q < le && is_space(*q)) ++q;
    if (q == le || *q == '#') continue;
    ntok = 0;
    while (q < le) {
      while (q < le && !is_space(*q)) ++q;
      ++ntok;
      while (q < le && is_space(*q)) ++q;
    }
    return true;
  }
  return false;
}

inline uint64_t tuple_hash(const uint32_t* c, uint32_t n) {
  uint64_t h = 0x9e3779b97f4a7c15ull;
  for (uint32_t i = 0; i < n; ++i) {
    h ^= c[i];
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 32;
  }
  h ^= h >> 29;
  h *= 0xc4ceb9fe1a85ec53ull;
  return h ^ (h >> 32);
}

template <typename T>
mk_host_tensor* parse_text(const char* text, uint64_t len, bool merge, const uint32_t* dims_ovr,
                           uint32_t n_ovr, uint32_t threads_req) {
  const char* end = text + len;
  uint64_t first_line = 0;
  size_t ntok = 0;
  if (!first_element_line(text, end, first_line, ntok))
    fail("frostt: empty input (no element lines)");
  if (ntok < 2)
    fail("frostt: line " + std::to_string(first_line) + ": need at least one index and a value");
  if (ntok - 1 > kMaxModes)
    fail("frostt: line " + std::to_string(first_line) + ": more than " +
         std::to_string(kMaxModes) + " modes");
  const uint32_t n = static_cast<uint32_t>(ntok - 1);

  // chunks at newline boundaries
  const unsigned T_ = thread_count(threads_req, len, 1u << 20);
  std::vector<const char*> cut(T_ + 1);
  cut[0] = text;
  cut[T_] = end;
  for (unsigned t = 1; t < T_; ++t) {
    const char* c = text + len * t / T_;
    if (c < cut[t - 1]) c = cut[t - 1];
    const char* nl = c < end ? static_cast<const char*>(memchr(c, '\n', end - c)) : nullptr;
    cut[t] = nl ? nl + 1 : end;
  }
  std::vector<ChunkOut> ch(T_);
  parallel_for(T_, [&](unsigned t) { parse_chunk<T>(cut[t], cut[t + 1], n, ch[t]); });

  // line offsets; the earliest error in file order
  std::vector<uint64_t> line0(T_ + 1, 0);
  for (unsigned t = 0; t < T_; ++t) line0[t + 1] = line0[t] + ch[t].lines;
  int err_chunk = -1;
  for (unsigned t = 0; t < T_; ++t)
    if (ch[t].err) {
      err_chunk = static_cast<int>(t);
      break;
    }
  const unsigned used = err_chunk >= 0 ? static_cast<unsigned>(err_chunk) + 1 : T_;
  std::vector<uint64_t> eoff(used + 1, 0);
  for (unsigned t = 0; t < used; ++t) eoff[t + 1] = eoff[t] + ch[t].vals.size();
  const uint64_t M = eoff[used];

  auto ht = std::make_unique<mk_host_tensor>();
  ht->n = n;
  ht->prec = sizeof(T) == 8 ? 64 : 32;
  std::vector<uint32_t> coords(M * n);
  std::vector<T> vals(M);
  std::vector<uint64_t> maxidx(n, 0);
  parallel_for(used, [&](unsigned t) {
    std::memcpy(coords.data() + eoff[t] * n, ch[t].coords.data(),
                ch[t].coords.size() * sizeof(uint32_t));
    for (size_t i = 0; i < ch[t].vals.size(); ++i)
      vals[eoff[t] + i] = static_cast<T>(ch[t].vals[i]);
  });
  for (unsigned t = 0; t < used; ++t)
    for (uint32_t h = 0; h < n; ++h) maxidx[h] = std::max(maxidx[h], ch[t].maxidx[h]);

  // duplicates: bucket by hash (file order inside a bucket), one owner thread per bucket
  std::vector<uint8_t> dead(M, 0);
  uint64_t dup_count = 0;
  uint64_t strict_line = UINT64_MAX;  // earliest duplicate line (global), strict mode
  uint64_t strict_elem = 0;
  if (M > 1) {
    const unsigned TD = thread_count(threads_req, M, 1u << 16);
    const uint32_t NB = TD * 4;
    std::vector<uint64_t> hash(M);
    std::vector<uint64_t> cnt(static_cast<size_t>(TD) * NB, 0);
    auto erange = [&](unsigned t, uint64_t& a, uint64_t& b) {
      a = M * t / TD;
      b = M * (t + 1) / TD;
    };
    parallel_for(TD, [&](unsigned t) {
      uint64_t a, b;
      erange(t, a, b);
      uint64_t* c = cnt.data() + static_cast<size_t>(t) * NB;
      for (uint64_t e = a; e < b; ++e) {
        hash[e] = tuple_hash(coords.data() + e * n, n);
        ++c[hash[e] % NB];
      }
    });
    std::vector<uint64_t> boff(static_cast<size_t>(NB) + 1, 0), pos(cnt.size());
    {
      uint64_t run_ = 0;
      for (uint32_t bkt = 0; bkt < NB; ++bkt) {
        boff[bkt] = run_;
        for (unsigned t = 0; t < TD; ++t) {
          pos[static_cast<size_t>(t) * NB + bkt] = run_;
          run_ += cnt[static_cast<size_t>(t) * NB + bkt];
        }
      }
      boff[NB] = run_;
    }
    std::vector<uint64_t> order(M);
    parallel_for(TD, [&](unsigned t) {
      uint64_t a, b;
      erange(t, a, b);
      uint64_t* p = pos.data() + static_cast<size_t>(t) * NB;
      for (uint64_t e = a; e < b; ++e) order[p[hash[e] % NB]++] = e;
    });
    std::vector<uint64_t> dups(TD, 0), sline(TD, UINT64_MAX), selem(TD, 0);
    // global line of element e (for strict-mode errors)
    auto gline = [&](uint64_t e) {
      const unsigned t = static_cast<unsigned>(std::upper_bound(eoff.begin(), eoff.end(), e) -
                                               eoff.begin()) - 1;
      return line0[t] + ch[t].line[e - eoff[t]];
    };
    parallel_for(TD, [&](unsigned t) {
      std::vector<uint64_t> table;
      for (uint32_t bkt = t; bkt < NB; bkt += TD) {
        const uint64_t b0 = boff[bkt], b1 = boff[bkt + 1], cntb = b1 - b0;
        if (cntb < 2) continue;
        uint64_t cap = 16;
        while (cap < 2 * cntb) cap <<= 1;
        table.assign(cap, UINT64_MAX);
        for (uint64_t k = b0; k < b1; ++k) {
          const uint64_t e = order[k];
          uint64_t slot = (hash[e] >> 7) & (cap - 1);
          for (;;) {
            const uint64_t f = table[slot];
            if (f == UINT64_MAX) {
              table[slot] = e;
              break;
            }
            if (hash[f] == hash[e] &&
                std::memcmp(coords.data() + f * n, coords.data() + e * n, n * 4) == 0) {
              ++dups[t];
              dead[e] = 1;
              if (merge) {
                vals[f] += vals[e];
              } else {
                const uint64_t L = gline(e);
                if (L < sline[t]) {
                  sline[t] = L;
                  selem[t] = e;
                }
              }
              break;
            }
            slot = (slot + 1) & (cap - 1);
          }
        }
      }
    });
    for (unsigned t = 0; t < TD; ++t) {
      dup_count += dups[t];
      if (sline[t] < strict_line) {
        strict_line = sline[t];
        strict_elem = selem[t];
      }
    }
  }
  // strict duplicate vs parse error: whichever line comes first (frostt.hpp:135-142)
  const uint64_t perr_line =
      err_chunk >= 0 ? line0[err_chunk] + ch[err_chunk].err_line : UINT64_MAX;
  if (!merge && strict_line < perr_line) {
    std::string pos;
    for (uint32_t h = 0; h < n; ++h)
      pos += std::to_string(static_cast<uint64_t>(coords[strict_elem * n + h]) + 1) + " ";
    fail("frostt: line " + std::to_string(strict_line) + ": duplicate index tuple " + pos +
         "(merging disabled)");
  }
  if (err_chunk >= 0)
    fail("frostt: line " + std::to_string(perr_line) + ": " + ch[err_chunk].err_msg);

  // compaction in file order
  const uint64_t keep = M - dup_count;
  if (dup_count) {
    const unsigned TC = thread_count(threads_req, M, 1u << 16);
    std::vector<uint64_t> live(TC + 1, 0);
    parallel_for(TC, [&](unsigned t) {
      uint64_t c = 0;
      for (uint64_t e = M * t / TC; e < M * (t + 1) / TC; ++e) c += !dead[e];
      live[t + 1] = c;
    });
    for (unsigned t = 0; t < TC; ++t) live[t + 1] += live[t];
    std::vector<uint32_t> c2(keep * n);
    std::vector<T> v2(keep);
    parallel_for(TC, [&](unsigned t) {
      uint64_t o = live[t];
      for (uint64_t e = M * t / TC; e < M * (t + 1) / TC; ++e)
        if (!dead[e]) {
          std::memcpy(c2.data() + o * n, coords.data() + e * n, n * 4);
          v2[o++] = vals[e];
        }
    });
    coords.swap(c2);
    vals.swap(v2);
  }
  for (const T v : vals)
    if (!std::isfinite(static_cast<double>(v)))
      fail("frostt: merged duplicate values are non-finite");

  std::vector<uint32_t> dims(n);
  if (n_ovr) {
    if (n_ovr != n)
      fail("frostt: dims override has " + std::to_string(n_ovr) + " modes, file has " +
           std::to_string(n));
    for (uint32_t h = 0; h < n; ++h)
      if (dims_ovr[h] < maxidx[h])
        fail("frostt: dims override extent " + std::to_string(dims_ovr[h]) +
             " below largest index " + std::to_string(maxidx[h]) + " in mode " +
             std::to_string(h));
    dims.assign(dims_ovr, dims_ovr + n);
    for (uint32_t e : dims)
      if (e == 0) fail("shape: zero extent");  // Shape::validate (types.hpp:31-35)
  } else {
    for (uint32_t h = 0; h < n; ++h) dims[h] = static_cast<uint32_t>(maxidx[h]);
  }
  ht->dims = std::move(dims);
  ht->coords = std::move(coords);
  if constexpr (sizeof(T) == 8) ht->v64 = std::move(vals);
  else ht->v32 = std::move(vals);
  ht->duplicates = dup_count;
  return ht.release();
}

std::vector<char> slurp(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) fail(std::string("frostt: cannot open '") + path + "'");
  std::vector<char> buf;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long sz = std::ftell(f);
    if (sz > 0) {
      std::rewind(f);
      buf.resize(static_cast<size_t>(sz));
      const size_t got = std::fread(buf.data(), 1, buf.size(), f);
      buf.resize(got);
      std::fclose(f);
      return buf;
    }
    std::rewind(f);
  }
  char tmp[1 << 16];  // pipes / unsized streams
  size_t got;
  while ((got = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  std::fclose(f);
  return buf;
}

// ------------------------------------------------------------------------------------ write
template <typename T>
void format_range(const uint32_t* coords, const T* vals, uint32_t n, uint64_t a, uint64_t b,
                  std::string& s) {
  char buf[64];
  for (uint64_t i = a; i < b; ++i) {
    for (uint32_t h = 0; h < n; ++h) {
      auto [p, ec] = std::to_chars(buf, buf + sizeof buf,
                                   static_cast<uint64_t>(coords[i * n + h]) + 1);
      s.append(buf, p);
      s.push_back(' ');
    }
    auto [p, ec] = std::to_chars(buf, buf + sizeof buf, vals[i]);
    s.append(buf, p);
    s.push_back('\n');
  }
}

template <typename T>
std::vector<std::string> format_all(const uint32_t* coords, const T* vals, uint32_t n,
                                    uint64_t nnz, uint32_t threads_req) {
  const unsigned T_ = thread_count(threads_req, nnz, 1u << 15);
  std::vector<std::string> parts(T_);
  parallel_for(T_, [&](unsigned t) {
    format_range(coords, vals, n, nnz * t / T_, nnz * (t + 1) / T_, parts[t]);
  });
  return parts;
}

// ------------------------------------------------------------------------------------ cache
constexpr char kMagic[4] = {'M', 'K', 'B', 'T'};
constexpr uint32_t kVersion = 1;

uint64_t payload_checksum(const unsigned char* p, uint64_t len) {
  // per-1MiB FNV-1a-64 words folded in block order (parallel-friendly, deterministic)
  const uint64_t B = 1ull << 20, nb = (len + B - 1) / B;
  std::vector<uint64_t> hs(nb);
  const unsigned T_ = thread_count(0, nb, 4);
  parallel_for(T_, [&](unsigned t) {
    for (uint64_t k = nb * t / T_; k < nb * (t + 1) / T_; ++k) {
      uint64_t h = 0xcbf29ce484222325ull;
      const uint64_t a = k * B, b = std::min(len, a + B);
      uint64_t i = a;
      for (; i + 8 <= b; i += 8) {
        uint64_t w;
        std::memcpy(&w, p + i, 8);
        h = (h ^ w) * 0x100000001b3ull;
      }
      for (; i < b; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
      hs[k] = h;
    }
  });
  uint64_t h = 0x84222325cbf29ce4ull ^ len;
  for (uint64_t x : hs) h = (h ^ x) * 0x100000001b3ull;
  return h;
}

}  // namespace

extern "C" {

int mk_frostt_parse(const char* text, uint64_t len, int prec, int merge_duplicates,
                    const uint32_t* dims_override, uint32_t n_override, uint32_t threads,
                    mk_host_tensor** out) {
  return run([&] {
    if (!out || (!text && len)) fail("frostt: null argument");
    if (prec != 32 && prec != 64) fail("frostt: precision must be 32 or 64");
    if (n_override && !dims_override) fail("frostt: null dims override");
    *out = prec == 64 ? parse_text<double>(text, len, merge_duplicates != 0, dims_override,
                                           n_override, threads)
                      : parse_text<float>(text, len, merge_duplicates != 0, dims_override,
                                          n_override, threads);
  });
}

int mk_frostt_read_file(const char* path, int prec, int merge_duplicates,
                        const uint32_t* dims_override, uint32_t n_override, uint32_t threads,
                        mk_host_tensor** out) {
  return run([&] {
    if (!path || !out) fail("frostt: null argument");
    const std::vector<char> buf = slurp(path);
    if (prec != 32 && prec != 64) fail("frostt: precision must be 32 or 64");
    *out = prec == 64 ? parse_text<double>(buf.data(), buf.size(), merge_duplicates != 0,
                                           dims_override, n_override, threads)
                      : parse_text<float>(buf.data(), buf.size(), merge_duplicates != 0,
                                          dims_override, n_override, threads);
  });
}

int mk_host_tensor_info(const mk_host_tensor* t, uint32_t* n_modes, uint32_t* dims,
                        uint32_t dims_capacity, uint64_t* nnz, uint64_t* duplicates_merged,
                        int* prec) {
  return run([&] {
    if (!t) fail("host tensor: null handle");
    if (n_modes) *n_modes = t->n;
    if (dims) {
      if (dims_capacity < t->n) fail("host tensor: dims buffer too small");
      std::copy(t->dims.begin(), t->dims.end(), dims);
    }
    if (nnz) *nnz = t->nnz();
    if (duplicates_merged) *duplicates_merged = t->duplicates;
    if (prec) *prec = t->prec;
  });
}

int mk_host_tensor_export(const mk_host_tensor* t, uint32_t* coords_aos, void* values) {
  return run([&] {
    if (!t) fail("host tensor: null handle");
    if (coords_aos && !t->coords.empty())
      std::memcpy(coords_aos, t->coords.data(), t->coords.size() * sizeof(uint32_t));
    if (values) {
      if (t->prec == 64) std::memcpy(values, t->v64.data(), t->v64.size() * sizeof(double));
      else std::memcpy(values, t->v32.data(), t->v32.size() * sizeof(float));
    }
  });
}

int mk_host_tensor_free(mk_host_tensor* t) {
  delete t;
  return MK_OK;
}

int mk_frostt_format(uint32_t n_modes, uint64_t nnz, const uint32_t* coords_aos,
                     const void* values, int prec, uint32_t threads, char* buf, uint64_t cap,
                     uint64_t* len) {
  return run([&] {
    if (prec != 32 && prec != 64) fail("frostt: precision must be 32 or 64");
    if (nnz && (!coords_aos || !values)) fail("frostt: null argument");
    const auto parts =
        prec == 64 ? format_all(coords_aos, static_cast<const double*>(values), n_modes, nnz, threads)
                   : format_all(coords_aos, static_cast<const float*>(values), n_modes, nnz, threads);
    uint64_t total = 0;
    for (const auto& s : parts) total += s.size();
    if (len) *len = total;
    if (!buf) return;  // size query
    if (cap < total) fail("frostt: format buffer too small");
    for (const auto& s : parts) {
      std::memcpy(buf, s.data(), s.size());
      buf += s.size();
    }
  });
}

int mk_frostt_write_file(const char* path, uint32_t n_modes, uint64_t nnz,
                         const uint32_t* coords_aos, const void* values, int prec,
                         uint32_t threads) {
  return run([&] {
    if (!path) fail("frostt: null argument");
    if (prec != 32 && prec != 64) fail("frostt: precision must be 32 or 64");
    if (nnz && (!coords_aos || !values)) fail("frostt: null argument");
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(std::string("frostt: cannot create '") + path + "'");
    const auto parts =
        prec == 64 ? format_all(coords_aos, static_cast<const double*>(values), n_modes, nnz, threads)
                   : format_all(coords_aos, static_cast<const float*>(values), n_modes, nnz, threads);
    bool ok = true;
    for (const auto& s : parts) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) fail("frostt: write failed");
  });
}

int mk_tensor_cache_write(const char* path, uint32_t n_modes, const uint32_t* dims, uint64_t nnz,
                          const uint32_t* coords_aos, const void* values, int prec) {
  return run([&] {
    if (!path || !dims || (nnz && (!coords_aos || !values))) fail("cache: null argument");
    if (prec != 32 && prec != 64) fail("cache: precision must be 32 or 64");
    if (n_modes < 1 || n_modes > kMaxModes) fail("cache: bad mode count");
    const uint64_t cb = nnz * n_modes * 4, vb = nnz * (prec / 8);
    std::vector<unsigned char> payload(cb + vb);
    if (cb) std::memcpy(payload.data(), coords_aos, cb);
    if (vb) std::memcpy(payload.data() + cb, values, vb);
    const uint64_t sum = payload_checksum(payload.data(), payload.size());
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) fail(std::string("cache: cannot create '") + path + "'");
    const uint32_t hdr[4] = {0, kVersion, n_modes, static_cast<uint32_t>(prec)};
    bool ok = std::fwrite(kMagic, 1, 4, f) == 4 && std::fwrite(hdr + 1, 4, 3, f) == 3 &&
              std::fwrite(&nnz, 8, 1, f) == 1 && std::fwrite(dims, 4, n_modes, f) == n_modes &&
              std::fwrite(payload.data(), 1, payload.size(), f) == payload.size() &&
              std::fwrite(&sum, 8, 1, f) == 1;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok || std::rename(tmp.c_str(), path) != 0) {
      std::remove(tmp.c_str());
      fail("cache: write failed");
    }
  });
}

int mk_tensor_cache_read(const char* path, mk_host_tensor** out) {
  return run([&] {
    if (!path || !out) fail("cache: null argument");
    const std::vector<char> buf = slurp(path);
    const unsigned char* p = reinterpret_cast<const unsigned char*>(buf.data());
    uint64_t at = 0;
    auto need = [&](uint64_t k) {
      if (buf.size() < at + k) fail(std::string("cache: truncated file '") + path + "'");
    };
    need(4 + 12 + 8);
    if (std::memcmp(p, kMagic, 4) != 0) fail(std::string("cache: not a tensor cache '") + path + "'");
    uint32_t h[3];
    std::memcpy(h, p + 4, 12);
    uint64_t nnz;
    std::memcpy(&nnz, p + 16, 8);
    at = 24;
    if (h[0] != kVersion) fail("cache: unsupported version " + std::to_string(h[0]));
    const uint32_t n = h[1];
    const int prec = static_cast<int>(h[2]);
    if (n < 1 || n > kMaxModes || (prec != 32 && prec != 64)) fail("cache: corrupt header");
    need(4ull * n);
    auto t = std::make_unique<mk_host_tensor>();
    t->n = n;
    t->prec = prec;
    t->dims.resize(n);
    std::memcpy(t->dims.data(), p + at, 4ull * n);
    at += 4ull * n;
    const uint64_t cb = nnz * n * 4, vb = nnz * (prec / 8);
    if (nnz > (UINT64_MAX / 16) / n) fail("cache: corrupt header");
    need(cb + vb + 8);
    uint64_t sum;
    std::memcpy(&sum, p + at + cb + vb, 8);
    if (payload_checksum(p + at, cb + vb) != sum)
      fail(std::string("cache: checksum mismatch in '") + path + "'");
    t->coords.resize(nnz * n);
    if (cb) std::memcpy(t->coords.data(), p + at, cb);
    if (prec == 64) {
      t->v64.resize(nnz);
      if (vb) std::memcpy(t->v64.data(), p + at + cb, vb);
    } else {
      t->v32.resize(nnz);
      if (vb) std::memcpy(t->v32.data(), p + at + cb, vb);
    }
    *out = t.release();
  });
}

}  // extern "C"
