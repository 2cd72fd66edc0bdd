// Dataset ingest, host side (reference: histgnn/data.py:81-151
// and graphs.py:186-226): multi-threaded parsers for the reference's text
// formats, feeding the device CSR2 build and the feature placement
// (paper_2301_07482_b200/ingest.py). The file is mapped read-only, cut into
// per-thread byte ranges at line boundaries; pass 1 counts lines (so every
// chunk knows its first line number) and records, pass 2 parses into the
// caller's arrays at each chunk's offset. Errors are reported as the FIRST
// offending line of the file (kind, 1-based line number, value), the message
// itself is composed by the caller exactly as the reference words it.
//
//   hg_parse_int_lines   data.py:109-129 (_read_int_lines): one integer per
//                        line, blank lines skipped, no comments
//   hg_parse_edge_list   graphs.py:186-218 (read_edge_list): "src dst" per
//                        line, '#' starts a comment, blank lines skipped
//
// Integers follow Python's int(): optional sign, ASCII digits, single '_'
// between digits; surrounding whitespace ignored.
#include "hgb200.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <climits>
#include <string>
#include <thread>
#include <vector>

#include "hg_common.cuh"

namespace hg {
namespace {

enum ParseErr : int {
  kPeNone = 0,
  kPeNotInt = 1,      // int lines: not an integer / edges: non-integer id
  kPeNegative = 2,    // negative value / id
  kPeRange = 3,       // int lines: value >= upper
  kPeFields = 4,      // edges: not exactly two fields
};

struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p && n) munmap(const_cast<char*>(p), n);
    if (fd >= 0) close(fd);
  }
};

int map_file(const char* path, Mapped& m, const char* W) {
  m.fd = open(path, O_RDONLY);
  if (m.fd < 0) return fail(W, kBadArg, std::string("cannot open ") + path);
  struct stat st;
  if (fstat(m.fd, &st) != 0) return fail(W, kBadArg, std::string("cannot stat ") + path);
  m.n = (size_t)st.st_size;
  if (m.n == 0) return kOk;
  void* q = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
  if (q == MAP_FAILED) return fail(W, kBadArg, std::string("cannot map ") + path);
  madvise(q, m.n, MADV_SEQUENTIAL);
  m.p = static_cast<const char*>(q);
  return kOk;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// Python int() over [a, b) (already stripped): sign, digits, single '_' between digits
bool parse_int(const char* a, const char* b, long long& v) {
  if (a >= b) return false;
  bool neg = false;
  if (*a == '+' || *a == '-') {
    neg = *a == '-';
    ++a;
  }
  if (a >= b || !is_digit(*a)) return false;
  unsigned long long acc = 0;
  bool prev_us = false;
  for (; a < b; ++a) {
    if (*a == '_') {
      if (prev_us) return false;
      prev_us = true;
      continue;
    }
    if (!is_digit(*a)) return false;
    prev_us = false;
    acc = acc * 10 + (unsigned)(*a - '0');
    if (acc > (unsigned long long)LLONG_MAX) return false;
  }
  if (prev_us) return false;
  v = neg ? -(long long)acc : (long long)acc;
  return true;
}

struct Chunk {
  size_t a = 0, b = 0;        // byte range [a, b), starts at a line start
  long long lines = 0;        // newline-terminated (or final) lines in the chunk
  long long records = 0;      // non-blank records
  long long first_line = 1;   // 1-based number of the chunk's first line
  long long off = 0;          // output offset (records before the chunk)
  long long err_line = 0;     // first error in the chunk (0 = none)
  int err_kind = 0;
  long long err_val = 0;
  long long max_a = -1, max_b = -1;
};

std::vector<Chunk> cut(const Mapped& m, int nthreads) {
  const size_t min_chunk = 1 << 20;
  int T = std::max(1, std::min(nthreads, (int)std::max<size_t>(1, m.n / min_chunk)));
  std::vector<Chunk> cs;
  size_t a = 0;
  for (int t = 0; t < T && a < m.n; ++t) {
    size_t b = t == T - 1 ? m.n : std::max(a, m.n * (size_t)(t + 1) / (size_t)T);
    while (b < m.n && m.p[b - 1] != '\n') ++b;     // end after a newline
    if (b <= a) continue;
    Chunk c;
    c.a = a;
    c.b = b;
    cs.push_back(c);
    a = b;
  }
  return cs;
}

template <typename F>
void run_threads(std::vector<Chunk>& cs, F f) {
  std::vector<std::thread> th;
  for (size_t i = 0; i < cs.size(); ++i) th.emplace_back([&, i] { f(cs[i]); });
  for (auto& t : th) t.join();
}

// visit every line of a chunk: fn(line_begin, line_end, line_number)
template <typename Fn>
void each_line(const Mapped& m, Chunk& c, long long line0, Fn fn) {
  const char* p = m.p + c.a;
  const char* e = m.p + c.b;
  long long ln = line0;
  while (p < e) {
    const char* q = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* le = q ? q : e;
    if (!fn(p, le, ln)) return;
    ++ln;
    p = q ? q + 1 : e;
  }
}

inline void strip(const char*& a, const char*& b) {
  while (a < b && is_space(*a)) ++a;
  while (b > a && is_space(b[-1])) --b;
}

void finish_counts(std::vector<Chunk>& cs) {
  long long line = 1, off = 0;
  for (auto& c : cs) {
    c.first_line = line;
    c.off = off;
    line += c.lines;
    off += c.records;
  }
}

int first_error(const std::vector<Chunk>& cs, int* err, long long* err_line, long long* err_val) {
  for (const auto& c : cs)
    if (c.err_line) {
      if (err) *err = c.err_kind;
      if (err_line) *err_line = c.err_line;
      if (err_val) *err_val = c.err_val;
      return 1;
    }
  if (err) *err = 0;
  if (err_line) *err_line = 0;
  return 0;
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

int hg_parse_int_lines(const char* path, long long upper, int64_t* out, long long* count, int* err,
                       long long* err_line, long long* err_val, int nthreads) {
  const char* W = "hg_parse_int_lines";
  Mapped m;
  int s = map_file(path, m, W);
  if (s) return s;
  if (count) *count = 0;
  if (err) *err = 0;
  if (m.n == 0) return kOk;
  std::vector<Chunk> cs = cut(m, nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency());
  // pass 1: lines, records and the first error per chunk (local line numbers)
  run_threads(cs, [&](Chunk& c) {
    each_line(m, c, 1, [&](const char* a, const char* b, long long ln) {
      ++c.lines;
      strip(a, b);
      if (a == b) return true;
      long long v;
      int kind = kPeNone;
      if (!parse_int(a, b, v)) kind = kPeNotInt;
      else if (v < 0) kind = kPeNegative;
      else if (upper >= 0 && v >= upper) kind = kPeRange;
      if (kind && !c.err_line) {
        c.err_line = ln;
        c.err_kind = kind;
        c.err_val = kind == kPeNotInt ? 0 : v;
      }
      ++c.records;
      return true;
    });
  });
  finish_counts(cs);
  for (auto& c : cs)
    if (c.err_line) c.err_line += c.first_line - 1;
  long long total = 0;
  for (auto& c : cs) total += c.records;
  if (count) *count = total;
  if (first_error(cs, err, err_line, err_val) || !out) return kOk;
  // pass 2: values at each chunk's offset
  run_threads(cs, [&](Chunk& c) {
    long long k = c.off;
    each_line(m, c, c.first_line, [&](const char* a, const char* b, long long) {
      strip(a, b);
      if (a == b) return true;
      long long v = 0;
      parse_int(a, b, v);
      out[k++] = v;
      return true;
    });
  });
  return kOk;
}

int hg_parse_edge_list(const char* path, int32_t* src, int32_t* dst, long long* count, long long* max_src,
                       long long* max_dst, int* err, long long* err_line, int nthreads) {
  const char* W = "hg_parse_edge_list";
  Mapped m;
  int s = map_file(path, m, W);
  if (s) return s;
  if (count) *count = 0;
  if (max_src) *max_src = -1;
  if (max_dst) *max_dst = -1;
  if (err) *err = 0;
  if (m.n == 0) return kOk;
  std::vector<Chunk> cs = cut(m, nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency());
  auto fields = [](const char* a, const char* b, const char** f, int& nf) {
    const char* h = static_cast<const char*>(memchr(a, '#', (size_t)(b - a)));
    if (h) b = h;
    nf = 0;
    while (a < b) {
      while (a < b && (is_space(*a))) ++a;
      if (a >= b) break;
      const char* s0 = a;
      while (a < b && !is_space(*a)) ++a;
      if (nf < 3) {
        f[2 * nf] = s0;
        f[2 * nf + 1] = a;
      }
      ++nf;
    }
  };
  run_threads(cs, [&](Chunk& c) {
    each_line(m, c, 1, [&](const char* a, const char* b, long long ln) {
      ++c.lines;
      const char* f[6];
      int nf;
      fields(a, b, f, nf);
      if (nf == 0) return true;
      int kind = kPeNone;
      long long u = 0, v = 0;
      if (nf != 2) kind = kPeFields;
      else if (!parse_int(f[0], f[1], u) || !parse_int(f[2], f[3], v)) kind = kPeNotInt;
      else if (u < 0 || v < 0) kind = kPeNegative;
      else if (u > INT_MAX || v > INT_MAX) kind = kPeRange;
      if (kind && !c.err_line) {
        c.err_line = ln;
        c.err_kind = kind;
      }
      if (!kind) {
        c.max_a = std::max(c.max_a, u);
        c.max_b = std::max(c.max_b, v);
      }
      ++c.records;
      return true;
    });
  });
  finish_counts(cs);
  for (auto& c : cs)
    if (c.err_line) c.err_line += c.first_line - 1;
  long long total = 0, ms = -1, md = -1;
  for (auto& c : cs) {
    total += c.records;
    ms = std::max(ms, c.max_a);
    md = std::max(md, c.max_b);
  }
  if (count) *count = total;
  if (max_src) *max_src = ms;
  if (max_dst) *max_dst = md;
  if (first_error(cs, err, err_line, nullptr) || !src || !dst) return kOk;
  run_threads(cs, [&](Chunk& c) {
    long long k = c.off;
    each_line(m, c, c.first_line, [&](const char* a, const char* b, long long) {
      const char* f[6];
      int nf;
      fields(a, b, f, nf);
      if (nf == 0) return true;
      long long u = 0, v = 0;
      parse_int(f[0], f[1], u);
      parse_int(f[2], f[3], v);
      src[k] = (int32_t)u;
      dst[k] = (int32_t)v;
      ++k;
      return true;
    });
  });
  return kOk;
}

}  // extern "C"
