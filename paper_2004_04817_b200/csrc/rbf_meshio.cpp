// Multi-threaded MDK1 mesh / MDK1-DISP text codec (host code).
//
// Replaces the bulk of reference meshio.py:135-250 (`read_mesh`,
// `write_mesh`, `read_displacements`, `write_displacements`), whose
// per-token Python parsing dominates end-to-end time at Nv = 1e7-4e7
// (SURVEY.md §8(f) row 3). The native readers accept exactly the inputs the
// reference parses the same way and return RBF_EPARSE for anything else --
// malformed input, but also tokens outside the plain numeric grammar
// (underscores, "inf", non-ASCII whitespace, ...) -- so that the Python layer
// can re-parse those rare files with the reference's own semantics and
// report the reference's first error with its line number. Writers emit the
// reference's canonical text: "%.17g" coordinates, decimal integers, "\n".
//
// Parsing is two-pass over contiguous byte ranges (one per thread, cut at
// newlines): pass 1 counts physical and content lines per range, a prefix
// sum assigns every content line its section (header / nodes / boundary /
// cells), pass 2 parses each range in place. Numbers go through
// std::from_chars (correctly rounded, as Python's float()).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rbf_internal.h"

using rbf::set_error;

namespace {

inline bool is_ws(unsigned char c) {
  // str.split() whitespace restricted to ASCII: \t \n \v \f \r, \x1c-\x1f, space
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

struct Tok {
  const char* b;
  const char* e;
};

// content tokens of one physical line [b, e) (comment stripped); returns count (<= cap + 1)
inline int tokenize(const char* b, const char* e, Tok* out, int cap) {
  const char* hash = static_cast<const char*>(memchr(b, '#', (size_t)(e - b)));
  if (hash) e = hash;
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_ws((unsigned char)*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_ws((unsigned char)*p)) ++p;
    if (n < cap) out[n] = Tok{s, p};
    ++n;
    if (n > cap) return n;
  }
  return n;
}

// [+-]? digits — the subset of Python int() literals handled natively
inline bool parse_i64(Tok t, int64_t& v) {
  const char* b = t.b;
  bool neg = false;
  if (b < t.e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b >= t.e) return false;
  for (const char* p = b; p < t.e; ++p)
    if (*p < '0' || *p > '9') return false;
  uint64_t u = 0;
  auto r = std::from_chars(b, t.e, u);
  if (r.ec != std::errc() || r.ptr != t.e || u > (uint64_t)INT64_MAX) return false;
  v = neg ? -(int64_t)u : (int64_t)u;
  return true;
}

// [+-]? (d+ (. d*)? | . d+) ([eE] [+-]? d+)? — Python float() accepts these
// and rounds them correctly, as from_chars does; the value must be finite
inline bool parse_f64(Tok t, double& v) {
  const char* b = t.b;
  bool neg = false;
  if (b < t.e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  const char* p = b;
  int mant = 0;
  while (p < t.e && *p >= '0' && *p <= '9') ++p, ++mant;
  if (p < t.e && *p == '.') {
    ++p;
    while (p < t.e && *p >= '0' && *p <= '9') ++p, ++mant;
  }
  if (mant == 0) return false;
  if (p < t.e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < t.e && (*p == '+' || *p == '-')) ++p;
    int ed = 0;
    while (p < t.e && *p >= '0' && *p <= '9') ++p, ++ed;
    if (ed == 0) return false;
  }
  if (p != t.e) return false;
  double x = 0.0;
  auto r = std::from_chars(b, t.e, x, std::chars_format::general);
  if (r.ptr != t.e) return false;
  if (r.ec == std::errc::result_out_of_range) return false;  // overflow/underflow: leave to Python
  if (r.ec != std::errc() || !std::isfinite(x)) return false;
  v = neg ? -x : x;
  return true;
}

struct Range {
  const char* b;
  const char* e;
  int64_t content = 0;  // content lines in this range
  int64_t first = 0;    // content-line index of its first content line
};

std::vector<Range> split_ranges(const char* text, size_t len, int threads) {
  std::vector<Range> r;
  const char* end = text + len;
  const char* p = text;
  for (int t = 0; t < threads && p < end; ++t) {
    const char* q = t == threads - 1 ? end : text + (size_t)((double)len * (t + 1) / threads);
    if (q < p) q = p;
    if (q < end) {
      const char* nl = static_cast<const char*>(memchr(q, '\n', (size_t)(end - q)));
      q = nl ? nl + 1 : end;
    }
    r.push_back(Range{p, q});
    p = q;
  }
  if (r.empty()) r.push_back(Range{text, text});
  return r;
}

template <class F>
void for_lines(const char* b, const char* e, F&& f) {
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* le = nl ? nl : e;
    f(p, le);
    p = nl ? nl + 1 : e;
  }
}

inline bool has_content(const char* b, const char* e) {
  for (const char* p = b; p < e; ++p) {
    if (*p == '#') return false;
    if (!is_ws((unsigned char)*p)) return true;
  }
  return false;
}

template <class F>
void parallel(int n, F&& f) {
  if (n <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> pool;
  for (int i = 0; i < n; ++i) pool.emplace_back([&, i] { f(i); });
  for (auto& t : pool) t.join();
}

int clamp_threads(int threads, size_t len) {
  int hw = (int)std::thread::hardware_concurrency();
  if (threads <= 0) threads = hw > 0 ? hw : 1;
  const int by_size = (int)std::max<size_t>(1, len / (1u << 20));  // >= 1 MiB per thread
  return std::max(1, std::min({threads, by_size, 64}));
}

// content lines -> the ranges' prefix offsets; also returns the total
int64_t count_content(std::vector<Range>& rs) {
  parallel((int)rs.size(), [&](int i) {
    int64_t c = 0;
    for_lines(rs[i].b, rs[i].e, [&](const char* b, const char* e) { c += has_content(b, e); });
    rs[i].content = c;
  });
  int64_t acc = 0;
  for (auto& r : rs) {
    r.first = acc;
    acc += r.content;
  }
  return acc;
}

// pointer to the content line with index k (and its end), or nullptr
const char* seek_content(const std::vector<Range>& rs, int64_t k, const char** le_out) {
  for (const auto& r : rs) {
    if (k >= r.first + r.content) continue;
    int64_t idx = r.first;
    const char* found = nullptr;
    const char* p = r.b;
    while (p < r.e) {
      const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(r.e - p)));
      const char* le = nl ? nl : r.e;
      if (has_content(p, le)) {
        if (idx == k) {
          found = p;
          *le_out = le;
          break;
        }
        ++idx;
      }
      p = nl ? nl + 1 : r.e;
    }
    return found;
  }
  return nullptr;
}

bool parse_count_line(const std::vector<Range>& rs, int64_t k, const char* kw, int64_t& count) {
  const char* le = nullptr;
  const char* b = seek_content(rs, k, &le);
  if (!b) return false;
  Tok t[3];
  if (tokenize(b, le, t, 2) != 2) return false;
  const size_t kl = strlen(kw);
  if ((size_t)(t[0].e - t[0].b) != kl || memcmp(t[0].b, kw, kl) != 0) return false;
  return parse_i64(t[1], count) && count >= 0;
}

}  // namespace

// ------------------------------------------------------------------ reading
extern "C" int rbf_mdk1_counts(const char* text, size_t len, int64_t* counts, int threads) {
  // counts[0..2] = nodes, boundary nodes, cells (RBF_EPARSE: not natively parseable)
  if (!text || !counts) return set_error(RBF_EARG, "null pointer");
  auto rs = split_ranges(text, len, clamp_threads(threads, len));
  const int64_t total = count_content(rs);
  const char* le = nullptr;
  const char* b = seek_content(rs, 0, &le);
  Tok t[2];
  if (!b || tokenize(b, le, t, 1) != 1 || t[0].e - t[0].b != 4 || memcmp(t[0].b, "MDK1", 4) != 0)
    return set_error(RBF_EPARSE, "header");
  int64_t nv = 0, nb = 0, ne = 0;
  if (!parse_count_line(rs, 1, "NODES", nv)) return set_error(RBF_EPARSE, "NODES");
  if (!parse_count_line(rs, 2 + nv, "BOUNDARY", nb)) return set_error(RBF_EPARSE, "BOUNDARY");
  if (!parse_count_line(rs, 3 + nv + nb, "CELLS", ne)) return set_error(RBF_EPARSE, "CELLS");
  if (total != 4 + nv + nb + ne) return set_error(RBF_EPARSE, "line count");
  counts[0] = nv;
  counts[1] = nb;
  counts[2] = ne;
  return RBF_OK;
}

extern "C" int rbf_mdk1_parse(const char* text, size_t len, int64_t nv, int64_t nb, int64_t ne,
                              double* nodes, int64_t* boundary, int64_t* cells, int threads) {
  // nodes (nv,3); boundary (nb) in file order; cells (ne,5): arity then up to 4 indices
  if (!text || (nv && !nodes) || (nb && !boundary) || (ne && !cells)) return set_error(RBF_EARG, "null pointer");
  auto rs = split_ranges(text, len, clamp_threads(threads, len));
  count_content(rs);
  const int64_t b0 = 3 + nv, c0 = 4 + nv + nb;  // first boundary / cell content line
  std::atomic<bool> ok{true};
  parallel((int)rs.size(), [&](int i) {
    int64_t k = rs[i].first;
    Tok t[6];
    for_lines(rs[i].b, rs[i].e, [&](const char* b, const char* e) {
      if (!ok.load(std::memory_order_relaxed) || !has_content(b, e)) return;
      const int64_t line = k++;
      if (line >= 2 && line < 2 + nv) {
        double* out = nodes + 3 * (line - 2);
        if (tokenize(b, e, t, 3) != 3 || !parse_f64(t[0], out[0]) || !parse_f64(t[1], out[1]) ||
            !parse_f64(t[2], out[2]))
          ok = false;
      } else if (line >= b0 && line < b0 + nb) {
        int64_t v;
        if (tokenize(b, e, t, 1) != 1 || !parse_i64(t[0], v) || v < 0 || v >= nv) ok = false;
        else boundary[line - b0] = v;
      } else if (line >= c0 && line < c0 + ne) {
        int64_t* out = cells + 5 * (line - c0);
        const int nt = tokenize(b, e, t, 5);
        int64_t arity;
        if (nt < 1 || !parse_i64(t[0], arity) || (arity != 3 && arity != 4) || nt != arity + 1) {
          ok = false;
          return;
        }
        out[0] = arity;
        for (int q = 0; q < arity; ++q) {
          int64_t v;
          if (!parse_i64(t[1 + q], v) || v < 0 || v >= nv) {
            ok = false;
            return;
          }
          out[1 + q] = v;
        }
      }
    });
  });
  if (!ok) return set_error(RBF_EPARSE, "mesh body");
  // duplicate boundary indices (the reference rejects the second occurrence)
  std::vector<uint8_t> seen((size_t)nv, 0);
  for (int64_t i = 0; i < nb; ++i) {
    if (seen[(size_t)boundary[i]]) return set_error(RBF_EPARSE, "duplicate boundary index");
    seen[(size_t)boundary[i]] = 1;
  }
  return RBF_OK;
}

extern "C" int rbf_disp_parse(const char* text, size_t len, const int64_t* boundary, int64_t nb,
                              double* disp, int threads) {
  // MDK1-DISP: "idx dx dy dz" for every (sorted, unique) boundary index exactly once
  if (!text || (nb && (!boundary || !disp))) return set_error(RBF_EARG, "null pointer");
  auto rs = split_ranges(text, len, clamp_threads(threads, len));
  const int64_t total = count_content(rs);
  const char* le = nullptr;
  const char* b = seek_content(rs, 0, &le);
  Tok t[5];
  if (!b || tokenize(b, le, t, 1) != 1 || t[0].e - t[0].b != 9 || memcmp(t[0].b, "MDK1-DISP", 9) != 0)
    return set_error(RBF_EPARSE, "header");
  if (total - 1 != nb) return set_error(RBF_EPARSE, "line count");
  std::vector<int64_t> slot((size_t)nb, -1);  // position -> content line that filled it
  std::atomic<bool> ok{true};
  parallel((int)rs.size(), [&](int i) {
    int64_t k = rs[i].first;
    Tok tk[5];
    for_lines(rs[i].b, rs[i].e, [&](const char* lb, const char* lend) {
      if (!ok.load(std::memory_order_relaxed) || !has_content(lb, lend)) return;
      const int64_t line = k++;
      if (line == 0) return;
      int64_t idx;
      double v[3];
      if (tokenize(lb, lend, tk, 4) != 4 || !parse_i64(tk[0], idx) || !parse_f64(tk[1], v[0]) ||
          !parse_f64(tk[2], v[1]) || !parse_f64(tk[3], v[2])) {
        ok = false;
        return;
      }
      const int64_t* it = std::lower_bound(boundary, boundary + nb, idx);
      if (it == boundary + nb || *it != idx) {
        ok = false;
        return;
      }
      const int64_t pos = it - boundary;
      slot[(size_t)pos] = line;  // a duplicate leaves some slot unfilled (counts match)
      disp[3 * pos] = v[0];
      disp[3 * pos + 1] = v[1];
      disp[3 * pos + 2] = v[2];
    });
  });
  if (!ok) return set_error(RBF_EPARSE, "displacement body");
  for (int64_t p = 0; p < nb; ++p)
    if (slot[(size_t)p] < 0) return set_error(RBF_EPARSE, "missing or duplicate node");
  return RBF_OK;
}

// ------------------------------------------------------------------ writing
namespace {

inline char* put_g17(char* p, double x) {
  auto r = std::to_chars(p, p + 32, x, std::chars_format::general, 17);  // == printf("%.17g")
  return r.ptr;
}

inline char* put_i64(char* p, int64_t v) { return std::to_chars(p, p + 24, v).ptr; }

constexpr size_t kRowMax = 3 * 32 + 4;  // bytes of one formatted coordinate row, upper bound

// rows [0, n) formatted by fmt_row(i, p) -> end, chunked over threads into
// `out` (capacity cap); returns the bytes written
template <class F>
int64_t format_rows(int64_t n, char* out, int64_t cap, int threads, F&& fmt_row) {
  const int nt = std::max(1, std::min<int>(threads, (int)std::max<int64_t>(1, n / 65536)));
  std::vector<std::string> parts((size_t)nt);
  parallel(nt, [&](int t) {
    const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    std::string& s = parts[(size_t)t];
    s.resize((size_t)((hi - lo) * kRowMax));
    char* p = s.data();
    for (int64_t i = lo; i < hi; ++i) p = fmt_row(i, p);
    s.resize((size_t)(p - s.data()));
  });
  int64_t off = 0;
  for (auto& s : parts) {
    if (off + (int64_t)s.size() > cap) return -1;
    memcpy(out + off, s.data(), s.size());
    off += (int64_t)s.size();
  }
  return off;
}

}  // namespace

extern "C" int64_t rbf_mdk1_format_nodes(const double* xyz, int64_t n, char* out, int64_t cap, int threads) {
  // "x y z\n" per row, %.17g; returns bytes written or -1 (capacity: 100 bytes per row)
  if (n < 0 || (n && (!xyz || !out))) return -1;
  return format_rows(n, out, cap, clamp_threads(threads, (size_t)n * 64), [&](int64_t i, char* p) {
    p = put_g17(p, xyz[3 * i]);
    *p++ = ' ';
    p = put_g17(p, xyz[3 * i + 1]);
    *p++ = ' ';
    p = put_g17(p, xyz[3 * i + 2]);
    *p++ = '\n';
    return p;
  });
}

extern "C" int64_t rbf_disp_format(const int64_t* idx, const double* xyz, int64_t n, char* out, int64_t cap,
                                   int threads) {
  // "idx dx dy dz\n" per row; capacity: 124 bytes per row
  if (n < 0 || (n && (!idx || !xyz || !out))) return -1;
  return format_rows(n, out, cap, clamp_threads(threads, (size_t)n * 64), [&](int64_t i, char* p) {
    p = put_i64(p, idx[i]);
    *p++ = ' ';
    p = put_g17(p, xyz[3 * i]);
    *p++ = ' ';
    p = put_g17(p, xyz[3 * i + 1]);
    *p++ = ' ';
    p = put_g17(p, xyz[3 * i + 2]);
    *p++ = '\n';
    return p;
  });
}
