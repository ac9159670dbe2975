// sd_jsonl.cpp — native JSON-lines codec for the `solve` front end
// (reference cli.py:29-137).
//
// The reference parses every MatrixRecord with json.loads and writes every
// ResultRecord with its own 17-significant-digit dumps (cli.py:33-48), one
// matrix at a time in Python.  Here the host side is split in two batch
// calls around the GPU solve:
//   sd_jsonl_parse  : split a buffer into lines and parse, in parallel, the
//                     records it can parse *exactly* like json.loads +
//                     parse_record would; everything else (malformed JSON,
//                     non-finite or non-numeric values, escaped or non-ASCII
//                     ids, duplicate keys, ...) is left to the Python parser
//                     (kind 0) so error messages stay the reference's.
//   sd_jsonl_format : format ResultRecords with the reference's key order
//                     and `format(x, ".17g")` floats (std::to_chars general
//                     / precision 17 is the same correctly rounded
//                     conversion), in parallel.
// Numbers are converted with std::from_chars (correctly rounded, like
// CPython's float()).  No CUDA here; host threads only.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/symdiag_b200.h"

namespace {

inline bool json_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
// characters str.strip() removes that can appear in an ASCII line
inline bool strip_ws(char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= '\x1c' && c <= '\x1f');
}

// key ids: 0..5 = a11 a22 a33 a12 a13 a23 (cli.py:29-30 order), 6 = id
int key_id(const char* p, int len) {
  if (len == 2 && p[0] == 'i' && p[1] == 'd') return 6;
  if (len != 3 || p[0] != 'a') return -1;
  const int r = p[1] - '0', c = p[2] - '0';
  if (r == 1 && c == 1) return 0;
  if (r == 2 && c == 2) return 1;
  if (r == 3 && c == 3) return 2;
  if (r == 1 && c == 2) return 3;
  if (r == 1 && c == 3) return 4;
  if (r == 2 && c == 3) return 5;
  return -1;
}

// strict JSON number grammar: -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)?
const char* scan_number(const char* p, const char* e) {
  if (p < e && *p == '-') p++;
  if (p >= e) return nullptr;
  if (*p == '0') {
    p++;
  } else if (*p >= '1' && *p <= '9') {
    while (p < e && *p >= '0' && *p <= '9') p++;
  } else {
    return nullptr;
  }
  if (p < e && *p == '.') {
    p++;
    const char* d = p;
    while (p < e && *p >= '0' && *p <= '9') p++;
    if (p == d) return nullptr;
  }
  if (p < e && (*p == 'e' || *p == 'E')) {
    p++;
    if (p < e && (*p == '+' || *p == '-')) p++;
    const char* d = p;
    while (p < e && *p >= '0' && *p <= '9') p++;
    if (p == d) return nullptr;
  }
  return p;
}

// One stripped, non-empty line.  Returns 3 or 2 with the packed row, or 0
// when the Python parser must handle it.
int parse_line(const char* p, const char* e, double* row, int64_t* id_b, int64_t* id_e,
               const char* base) {
  double v[6];
  unsigned seen = 0;
  *id_b = *id_e = -1;
  while (p < e && json_ws(*p)) p++;
  if (p >= e || *p != '{') return 0;
  p++;
  while (p < e && json_ws(*p)) p++;
  if (p < e && *p == '}') return 0;  // {} -> wrong keys: Python's message
  for (;;) {
    if (p >= e || *p != '"') return 0;
    const char* k0 = ++p;
    while (p < e && *p != '"' && *p != '\\') p++;
    if (p >= e || *p != '"') return 0;
    const int key = key_id(k0, (int)(p - k0));
    p++;
    if (key < 0 || (seen >> key) & 1u) return 0;  // unexpected or duplicate key
    seen |= 1u << key;
    while (p < e && json_ws(*p)) p++;
    if (p >= e || *p != ':') return 0;
    p++;
    while (p < e && json_ws(*p)) p++;
    if (p >= e) return 0;
    if (key == 6) {
      if (*p == '"') {
        const char* s0 = p++;
        // printable ASCII without escapes: json.dumps(json.loads(t)) == t
        while (p < e && *p != '"' && *p != '\\' && (unsigned char)*p >= 0x20 &&
               (unsigned char)*p < 0x7f)
          p++;
        if (p >= e || *p != '"') return 0;
        p++;
        *id_b = s0 - base;
        *id_e = p - base;
      } else if (e - p >= 4 && std::memcmp(p, "null", 4) == 0) {
        p += 4;
      } else {
        return 0;
      }
    } else {
      const char* q = scan_number(p, e);
      if (!q) return 0;
      double x;
      // from_chars does not accept a leading '+' (JSON does not either)
      const auto r = std::from_chars(p, q, x);
      if (r.ec != std::errc() || r.ptr != q) return 0;  // out of range -> Python
      if (!(x - x == 0.0)) return 0;                     // non-finite -> ParseError there
      v[key] = x;
      p = q;
    }
    while (p < e && json_ws(*p)) p++;
    if (p >= e) return 0;
    if (*p == ',') {
      p++;
      while (p < e && json_ws(*p)) p++;
      continue;
    }
    if (*p != '}') return 0;
    p++;
    break;
  }
  while (p < e && json_ws(*p)) p++;
  if (p != e) return 0;
  const unsigned vals = seen & 0x3fu;
  if (vals == 0x3fu) {  // packed (a11, a12, a13, a22, a23, a33)
    row[0] = v[0];
    row[1] = v[3];
    row[2] = v[4];
    row[3] = v[1];
    row[4] = v[5];
    row[5] = v[2];
    return 3;
  }
  if (vals == 0x0bu) {  // a11, a22, a12 -> packed (a11, a12, a22)
    row[0] = v[0];
    row[1] = v[3];
    row[2] = v[1];
    return 2;
  }
  return 0;
}

template <typename F>
void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 1 || n < 4096) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  const int64_t step = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; t++) {
    const int64_t b = t * step, e = std::min(n, b + step);
    if (b >= e) break;
    ts.emplace_back([=] { f(b, e); });
  }
  for (auto& t : ts) t.join();
}

// Writers into a caller-sized buffer (the caller reserves kRecMax + id bytes
// per record).
constexpr int64_t kRecMax = 1024;  // > longest 3x3 record without its id (~800 B)

inline char* put_str(char* o, const char* t) {
  const size_t n = std::strlen(t);
  std::memcpy(o, t, n);
  return o + n;
}

inline char* put_double(char* o, double x) {
  return std::to_chars(o, o + 32, x, std::chars_format::general, 17).ptr;
}

char* put_list(char* o, const double* v, int n) {
  *o++ = '[';
  for (int i = 0; i < n; i++) {
    if (i) o = put_str(o, ", ");
    o = put_double(o, v[i]);
  }
  *o++ = ']';
  return o;
}

// dumps_result (paper_1306_6291_b200/cli.py) == dumps(result_record(...)),
// '\n'-terminated; returns the end of the record
char* format_record(char* o, int dim, const char* id, int64_t id_len, const double* lam,
                    const double* ang, const double* d, const double* res, uint8_t status) {
  static const char* kBranch[4] = {"\"Generic\"", "\"AlreadyDiagonal2D\"", "\"DoubleRoot\"",
                                   "\"TripleRoot\""};
  o = put_str(o, "{\"id\": ");
  if (id_len > 0) {
    std::memcpy(o, id, (size_t)id_len);
    o += id_len;
  } else {
    o = put_str(o, "null");
  }
  o = put_str(o, ", \"dim\": ");
  *o++ = (char)('0' + dim);
  o = put_str(o, ", \"eigenvalues\": ");
  o = put_list(o, lam, dim);
  double srt[3];
  std::copy(lam, lam + dim, srt);
  std::stable_sort(srt, srt + dim, [](double a, double b) { return a > b; });
  o = put_str(o, ", \"eigenvalues_sorted\": ");
  o = put_list(o, srt, dim);
  const int na = dim == 3 ? 3 : 1;
  o = put_str(o, ", \"angles\": ");
  o = put_list(o, ang, na);
  o = put_str(o, ", \"euler_angles\": ");
  o = put_list(o, ang, na);
  o = put_str(o, ", \"eigenvectors\": [");
  for (int c = 0; c < dim; c++) {
    if (c) o = put_str(o, ", ");
    double col[3];
    for (int r = 0; r < dim; r++) col[r] = d[r * dim + c];
    o = put_list(o, col, dim);
  }
  o = put_str(o, "], \"branch\": ");
  o = put_str(o, dim == 3 ? kBranch[status & 3] : "null");
  o = put_str(o, ", \"residuals\": {\"recon_rel\": ");
  o = put_double(o, res[0]);
  o = put_str(o, ", \"ortho\": ");
  o = put_double(o, res[1]);
  o = put_str(o, ", \"max_eigvec_res\": ");
  double mx = res[2];
  for (int k = 1; k < dim; k++)
    if (res[2 + k] > mx) mx = res[2 + k];  // Python max(): first of the maxima
  o = put_double(o, mx);
  return put_str(o, "}}\n");
}

}  // namespace

extern "C" {

int64_t sd_jsonl_parse(const char* buf, int64_t len, int64_t cap, int nthreads, int8_t* kind,
                       double* rows, int64_t* span, int64_t* consumed) {
  if (!buf || len < 0 || cap < 0 || !kind || !rows || !span || !consumed) return -1;
  // line boundaries (serial memchr scan), blank lines dropped like the
  // reference's `line.strip()` / `continue`
  std::vector<int64_t> lb, le;
  lb.reserve((size_t)std::min<int64_t>(cap, 1 << 20));
  int64_t pos = 0;
  while (pos < len && (int64_t)lb.size() < cap) {
    const char* nl = static_cast<const char*>(std::memchr(buf + pos, '\n', (size_t)(len - pos)));
    const int64_t end = nl ? nl - buf : len;
    int64_t b = pos, e = end;
    while (b < e && strip_ws(buf[b])) b++;
    while (e > b && strip_ws(buf[e - 1])) e--;
    if (e > b) {
      lb.push_back(b);
      le.push_back(e);
    }
    pos = nl ? end + 1 : len;
  }
  *consumed = pos;
  const int64_t n = (int64_t)lb.size();
  parallel_for(n, nthreads, [&](int64_t b, int64_t e) {
    for (int64_t k = b; k < e; k++) {
      span[4 * k] = lb[k];
      span[4 * k + 1] = le[k];
      kind[k] = (int8_t)parse_line(buf + lb[k], buf + le[k], rows + 6 * k, &span[4 * k + 2],
                                   &span[4 * k + 3], buf);
    }
  });
  return n;
}

int64_t sd_jsonl_format(int64_t n, const int8_t* dim, const char* idbuf, const int64_t* id_span,
                        const double* lam, const double* ang, const double* d, const double* res,
                        const uint8_t* status, int nthreads, char* out, int64_t out_cap,
                        int64_t* offsets) {
  if (n < 0 || !dim || !lam || !ang || !d || !res || !status || !offsets || (n > 0 && !out))
    return -1;
  auto id_len = [&](int64_t k) -> int64_t {
    if (!id_span || !idbuf || id_span[2 * k] < 0) return 0;
    return id_span[2 * k + 1] - id_span[2 * k];
  };
  // worst-case start of every record; threads write their range in place
  std::vector<int64_t> ub((size_t)n + 1);
  ub[0] = 0;
  for (int64_t k = 0; k < n; k++) ub[k + 1] = ub[k] + ((dim[k] == 2 || dim[k] == 3) ? kRecMax + id_len(k) : 0);
  if (ub[n] > out_cap) return -ub[n];
  const int nthr = std::max(1, nthreads);
  const int64_t step = (n + nthr - 1) / nthr;
  std::vector<int64_t> used((size_t)nthr, 0);
  parallel_for(n, nthr, [&](int64_t b, int64_t e) {
    char* const o0 = out + ub[b];
    char* o = o0;
    for (int64_t k = b; k < e; k++) {
      char* const r0 = o;
      const int dk = dim[k];
      if (dk == 2 || dk == 3) {
        const int64_t il = id_len(k);
        double dd[9];
        for (int r = 0; r < dk; r++)
          for (int c = 0; c < dk; c++) dd[r * dk + c] = d[9 * k + r * dk + c];
        o = format_record(o, dk, il ? idbuf + id_span[2 * k] : nullptr, il, lam + 3 * k,
                          ang + 3 * k, dd, res + 5 * k, status[k]);
      }
      offsets[k + 1] = o - r0;  // length for now
    }
    used[(size_t)(b / std::max<int64_t>(1, step))] = o - o0;
  });
  // close the gaps between the threads' ranges (left moves, in order)
  int64_t at = 0;
  for (int t = 0; t < nthr; t++) {
    const int64_t b = std::min(n, (int64_t)t * step);
    if (b >= n) break;
    if (out + at != out + ub[b]) std::memmove(out + at, out + ub[b], (size_t)used[(size_t)t]);
    at += used[(size_t)t];
  }
  int64_t total = 0;
  offsets[0] = 0;
  for (int64_t k = 0; k < n; k++) {
    total += offsets[k + 1];
    offsets[k + 1] = total;
  }
  return total;
}

}  // extern "C"
