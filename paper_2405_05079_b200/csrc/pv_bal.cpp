// Native BAL input path (include/povar_bal.h): a two-pass, multi-threaded
// tokenizer/parser with the grammar and error behaviour of the reference's
// parse_bal (pkg/src/stratba/bal_io.py:115-203), and the distinct-camera count
// of prune_underobserved (bal_io.py:244-278).
//
// Pass 1 (parallel): the text is cut into chunks at ASCII whitespace; each
// thread counts its tokens and line breaks.  A prefix sum gives every chunk the
// global index and line number of its first token, so pass 2 (parallel) knows
// which field each token fills: header (3), observations (4 each), cameras
// (9 each), points (3 each).  The first error in token order wins, which is the
// error the reference's sequential loop raises.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/povar_bal.h"

namespace {

// byte classes: 1 = ASCII whitespace, 2 = line break (\n, \r), 4 = lead byte of a possible
// UTF-8 whitespace character, 8 = plain number character [0-9.eE-]
struct ByteClass {
  unsigned char c[256];
  constexpr ByteClass() : c() {
    const char ws[] = {' ', '\t', '\n', '\r', '\v', '\f', 0x1c, 0x1d, 0x1e, 0x1f};
    for (char w : ws) c[(unsigned char)w] |= 1;
    c[(unsigned char)'\n'] |= 2;
    c[(unsigned char)'\r'] |= 2;
    c[0xC2] |= 4;
    c[0xE1] |= 4;
    c[0xE2] |= 4;
    c[0xE3] |= 4;
    for (int d = '0'; d <= '9'; ++d) c[d] |= 8;
    c[(unsigned char)'.'] |= 8;
    c[(unsigned char)'e'] |= 8;
    c[(unsigned char)'E'] |= 8;
    c[(unsigned char)'-'] |= 8;
  }
};
constexpr ByteClass kClass{};

inline bool ascii_ws(unsigned char c) { return kClass.c[c] & 1; }

// length of a UTF-8 encoded Unicode whitespace character at p (str.split() separators
// beyond ASCII: U+0085, U+00A0, U+1680, U+2000-200A, U+2028, U+2029, U+202F, U+205F,
// U+3000), else 0
inline int utf8_ws(const unsigned char* p, const unsigned char* end) {
  if (p[0] == 0xC2 && p + 1 < end && (p[1] == 0x85 || p[1] == 0xA0)) return 2;
  if (p + 2 >= end) return 0;
  if (p[0] == 0xE1 && p[1] == 0x9A && p[2] == 0x80) return 3;
  if (p[0] == 0xE2 && p[1] == 0x80 &&
      ((p[2] >= 0x80 && p[2] <= 0x8A) || p[2] == 0xA8 || p[2] == 0xA9 || p[2] == 0xAF))
    return 3;
  if (p[0] == 0xE2 && p[1] == 0x81 && p[2] == 0x9F) return 3;
  if (p[0] == 0xE3 && p[1] == 0x80 && p[2] == 0x80) return 3;
  return 0;
}

// Token scanner over [p, end) with universal-newline line counting (\n, \r, \r\n).
struct Scanner {
  const unsigned char* p;
  const unsigned char* end;
  int64_t line;  // current line (1-based)
  // next token -> [b, e); false at end
  bool next(const unsigned char*& b, const unsigned char*& e) {
    for (;;) {
      if (p >= end) return false;
      const unsigned char c = *p;
      const unsigned char k = kClass.c[c];
      if (k & 2) {
        ++line;
        ++p;
        if (c == '\r' && p < end && *p == '\n') ++p;
      } else if (k & 1) {
        ++p;
      } else if (k & 4) {
        const int w = utf8_ws(p, end);
        if (!w) break;
        p += w;
      } else {
        break;
      }
    }
    b = p;
    while (p < end) {
      const unsigned char k = kClass.c[*p];
      if (k & 1) break;
      if ((k & 4) && utf8_ws(p, end)) break;
      ++p;
    }
    e = p;
    return true;
  }
};

// Python repr() of a token (no whitespace inside)
std::string py_repr(const unsigned char* b, const unsigned char* e) {
  bool has_sq = false, has_dq = false;
  for (const unsigned char* q = b; q < e; ++q) {
    has_sq |= *q == '\'';
    has_dq |= *q == '"';
  }
  const char quote = (has_sq && !has_dq) ? '"' : '\'';
  std::string s(1, quote);
  for (const unsigned char* q = b; q < e; ++q) {
    const unsigned char c = *q;
    if (c == '\\') {
      s += "\\\\";
    } else if (c == (unsigned char)quote) {
      s += '\\';
      s += quote;
    } else if (c < 0x20 || c == 0x7f) {
      static const char hx[] = "0123456789abcdef";
      s += "\\x";
      s += hx[c >> 4];
      s += hx[c & 15];
    } else {
      s += (char)c;
    }
  }
  s += quote;
  return s;
}

// Python int() token syntax: [+-] digit (["_"] digit)*.  Returns false if invalid.
// *canon = canonical decimal (for messages), *v = value, *big = out of int64 range.
bool parse_int(const unsigned char* b, const unsigned char* e, int64_t* v, bool* big,
               std::string* canon) {
  if (e - b <= 18 && e > b) {  // fast path: plain decimal digits
    int64_t val = 0;
    const unsigned char* q = b;
    for (; q < e && *q >= '0' && *q <= '9'; ++q) val = val * 10 + (*q - '0');
    if (q == e) {
      *v = val;
      *big = false;
      if (canon) *canon = std::to_string(val);
      return true;
    }
  }
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b >= e || !(*b >= '0' && *b <= '9')) return false;
  std::string digits;
  bool prev_us = false;
  for (const unsigned char* q = b; q < e; ++q) {
    if (*q >= '0' && *q <= '9') {
      digits += (char)*q;
      prev_us = false;
    } else if (*q == '_' && !prev_us && q > b) {
      prev_us = true;
    } else {
      return false;
    }
  }
  if (prev_us) return false;
  size_t nz = digits.find_first_not_of('0');
  digits = nz == std::string::npos ? "0" : digits.substr(nz);
  *big = digits.size() > 18;
  int64_t val = 0;
  if (!*big)
    for (char d : digits) val = val * 10 + (d - '0');
  *v = *big ? (neg ? INT64_MIN : INT64_MAX) : (neg ? -val : val);
  if (canon) *canon = (neg && digits != "0" ? "-" : "") + digits;
  return true;
}

// Python float() token syntax -> value (correctly rounded via from_chars)
bool parse_float(const unsigned char* b, const unsigned char* e, double* out) {
  {  // fast path: tokens of [0-9.eE-] only, where from_chars and float() agree
    const unsigned char* q = b;
    while (q < e && (kClass.c[*q] & 8)) ++q;
    if (q == e && e > b) {
      const char* cb = reinterpret_cast<const char*>(b);
      const char* ce = reinterpret_cast<const char*>(e);
      double v = 0.0;
      const auto r = std::from_chars(cb, ce, v, std::chars_format::general);
      if (r.ec == std::errc() && r.ptr == ce) {
        *out = v;
        return true;
      }
      if (r.ec == std::errc::result_out_of_range && r.ptr == ce) {
        char buf[512];
        const size_t n = std::min<size_t>(ce - cb, sizeof(buf) - 1);
        std::memcpy(buf, cb, n);
        buf[n] = 0;
        *out = std::strtod(buf, nullptr);
        return true;
      }
      // anything else: the validating path below decides
    }
  }
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  const size_t n = e - b;
  if (n == 0) return false;
  auto ieq = [&](const char* w) {
    const size_t m = std::strlen(w);
    if (m != n) return false;
    for (size_t i = 0; i < m; ++i)
      if (std::tolower(b[i]) != w[i]) return false;
    return true;
  };
  if (ieq("inf") || ieq("infinity")) {
    *out = neg ? -__builtin_inf() : __builtin_inf();
    return true;
  }
  if (ieq("nan")) {
    *out = neg ? -__builtin_nan("") : __builtin_nan("");
    return true;
  }
  // validate: digitpart ["." [digitpart]] | "." digitpart, then [eE [+-] digitpart]
  char buf[512];
  size_t k = 0;
  const unsigned char* q = b;
  auto digitpart = [&]() -> bool {  // digit (["_"] digit)*
    if (q >= e || !(*q >= '0' && *q <= '9')) return false;
    while (q < e) {
      if (*q >= '0' && *q <= '9') {
        if (k < sizeof(buf) - 8) buf[k++] = (char)*q;
        else return false;
        ++q;
      } else if (*q == '_' && q + 1 < e && q[1] >= '0' && q[1] <= '9') {
        ++q;
      } else {
        break;
      }
    }
    return true;
  };
  bool have_int = false, have_frac = false;
  if (q < e && *q >= '0' && *q <= '9') have_int = digitpart();
  if (q < e && *q == '.') {
    buf[k++] = '.';
    ++q;
    if (q < e && *q >= '0' && *q <= '9') have_frac = digitpart();
  }
  if (!have_int && !have_frac) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    buf[k++] = 'e';
    ++q;
    if (q < e && (*q == '+' || *q == '-')) buf[k++] = (char)*q++;
    if (!digitpart()) return false;
  }
  if (q != e) return false;
  double v = 0.0;
  const auto r = std::from_chars(buf, buf + k, v, std::chars_format::general);
  if (r.ec == std::errc::result_out_of_range) {
    // overflow -> inf, underflow -> subnormal / 0 (Python float semantics; strtod rounds)
    buf[k] = 0;
    v = std::strtod(buf, nullptr);
  } else if (r.ec != std::errc() || r.ptr != buf + k) {
    return false;
  }
  *out = neg ? -v : v;
  return true;
}

struct Err {
  int64_t tok = INT64_MAX;  // global token index of the error
  int64_t line = 0;
  std::string msg;
};

struct Layout {
  int64_t n_cam, n_pt, n_obs;
  int64_t obs_end, cam_end, total;  // token index boundaries
};

std::string field_name(const Layout& L, int64_t t) {
  if (t == 0) return "camera count";
  if (t == 1) return "point count";
  if (t == 2) return "observation count";
  if (t < L.obs_end) {
    static const char* f[4] = {"camera index", "point index", "measurement x", "measurement y"};
    return f[(t - 3) % 4];
  }
  if (t < L.cam_end) {
    const int64_t u = t - L.obs_end;
    return "camera " + std::to_string(u / 9) + " parameter " + std::to_string(u % 9);
  }
  const int64_t u = t - L.cam_end;
  return "point " + std::to_string(u / 3) + " coordinate " + std::to_string(u % 3);
}

void set_err(char* err_msg, size_t cap, int64_t* err_line, const Err& e) {
  if (err_line) *err_line = e.line;
  if (err_msg && cap) {
    const size_t n = std::min(cap - 1, e.msg.size());
    std::memcpy(err_msg, e.msg.data(), n);
    err_msg[n] = 0;
  }
}

// reads the three header counts; returns the scanner positioned after them
bool read_header(const unsigned char* text, size_t len, Layout* L, Scanner* sc, Err* err) {
  *sc = Scanner{text, text + len, 1};
  int64_t vals[3];
  int64_t last_line = 0;
  for (int i = 0; i < 3; ++i) {
    const unsigned char *b, *e;
    Layout dummy{};
    if (!sc->next(b, e)) {
      err->tok = i;
      err->line = last_line;
      err->msg = "truncated file: expected " + field_name(dummy, i);
      return false;
    }
    last_line = sc->line;
    bool big = false;
    if (!parse_int(b, e, &vals[i], &big, nullptr)) {
      err->tok = i;
      err->line = sc->line;
      err->msg = "expected integer " + field_name(dummy, i) + ", got " + py_repr(b, e);
      return false;
    }
  }
  if (vals[0] < 0 || vals[1] < 0 || vals[2] < 0) {
    err->tok = 2;
    err->line = sc->line;
    err->msg = "malformed header: negative count";
    return false;
  }
  const int64_t lim = (int64_t)1 << 40;
  if (vals[0] > lim || vals[1] > lim || vals[2] > lim) {
    err->tok = 2;
    err->line = sc->line;
    err->msg = "malformed header: count too large";
    return false;
  }
  L->n_cam = vals[0];
  L->n_pt = vals[1];
  L->n_obs = vals[2];
  L->obs_end = 3 + 4 * L->n_obs;
  L->cam_end = L->obs_end + 9 * L->n_cam;
  L->total = L->cam_end + 3 * L->n_pt;
  return true;
}

}  // namespace

extern "C" {

int pv_bal_header(const char* text, size_t len, int64_t* n_cameras, int64_t* n_points,
                  int64_t* n_observations, int64_t* err_line, char* err_msg, size_t err_cap) {
  Layout L{};
  Scanner sc{};
  Err err;
  if (!read_header(reinterpret_cast<const unsigned char*>(text), len, &L, &sc, &err)) {
    set_err(err_msg, err_cap, err_line, err);
    return PV_BAL_EPARSE;
  }
  *n_cameras = L.n_cam;
  *n_points = L.n_pt;
  *n_observations = L.n_obs;
  return PV_BAL_OK;
}

int pv_bal_parse(const char* text_c, size_t len, int n_threads, int64_t* cam_idx, int64_t* pt_idx,
                 double* meas, double* cams, double* pts, int64_t* err_line, char* err_msg,
                 size_t err_cap) {
  const unsigned char* text = reinterpret_cast<const unsigned char*>(text_c);
  Layout L{};
  Scanner hs{};
  Err herr;
  if (!read_header(text, len, &L, &hs, &herr)) {
    set_err(err_msg, err_cap, err_line, herr);
    return PV_BAL_EPARSE;
  }
  const size_t body0 = hs.p - text;
  const int64_t line0 = hs.line;
  const size_t body_len = len - body0;
  // auto: all hardware threads, >= 1 MB of text each; explicit: as asked (>= 64 B each)
  int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  const size_t min_chunk = n_threads > 0 ? 64 : (1 << 20);
  T = (int)std::max<size_t>(1, std::min<size_t>((size_t)T, body_len / min_chunk + 1));
  // chunk boundaries at ASCII whitespace (never inside a token or a \r\n pair)
  std::vector<size_t> cut(T + 1);
  cut[0] = body0;
  cut[T] = len;
  for (int k = 1; k < T; ++k) {
    size_t b = std::max(cut[k - 1], body0 + body_len * k / T);
    while (b < len && !ascii_ws(text[b])) ++b;
    if (b < len && b > 0 && text[b] == '\n' && text[b - 1] == '\r') ++b;
    cut[k] = b;
  }
  // pass 1: tokens and line breaks per chunk
  std::vector<int64_t> ntok(T, 0), nline(T, 0);
  auto count = [&](int k) {
    Scanner sc{text + cut[k], text + cut[k + 1], 0};
    const unsigned char *b, *e;
    int64_t n = 0;
    while (sc.next(b, e)) ++n;
    ntok[k] = n;
    nline[k] = sc.line;
  };
  {
    std::vector<std::thread> th;
    for (int k = 1; k < T; ++k) th.emplace_back(count, k);
    count(0);
    for (auto& t : th) t.join();
  }
  std::vector<int64_t> tok0(T + 1), ln0(T + 1);
  tok0[0] = 3;
  ln0[0] = line0;
  for (int k = 0; k < T; ++k) {
    tok0[k + 1] = tok0[k] + ntok[k];
    ln0[k + 1] = ln0[k] + nline[k];
  }
  const int64_t n_tokens = tok0[T];
  // pass 2: fill
  std::vector<Err> errs(T);
  auto fill = [&](int k) {
    Scanner sc{text + cut[k], text + cut[k + 1], ln0[k]};
    const unsigned char *b, *e;
    int64_t t = tok0[k];
    Err& er = errs[k];
    auto fail = [&](int64_t line, std::string m) {
      er.tok = t;
      er.line = line;
      er.msg = std::move(m);
    };
    while (sc.next(b, e)) {
      if (t >= L.total) {
        fail(sc.line, "trailing data after point block");
        return;
      }
      if (t < L.obs_end) {
        const int64_t o = (t - 3) >> 2;
        const int f = (int)((t - 3) & 3);
        if (f < 2) {
          int64_t v;
          bool big;
          if (!parse_int(b, e, &v, &big, nullptr)) {
            fail(sc.line, "expected integer " + field_name(L, t) + ", got " + py_repr(b, e));
            return;
          }
          const int64_t n = f == 0 ? L.n_cam : L.n_pt;
          if (big || v < 0 || v >= n) {
            std::string canon;
            parse_int(b, e, &v, &big, &canon);
            fail(sc.line, std::string(f == 0 ? "camera" : "point") + " index " + canon +
                              " out of range [0, " + std::to_string(n) + ")");
            return;
          }
          (f == 0 ? cam_idx : pt_idx)[o] = v;
        } else {
          double v;
          if (!parse_float(b, e, &v)) {
            fail(sc.line, "non-numeric token for " + field_name(L, t) + ": " + py_repr(b, e));
            return;
          }
          meas[2 * o + (f - 2)] = v;
        }
      } else {
        double v;
        if (!parse_float(b, e, &v)) {
          fail(sc.line, "non-numeric token for " + field_name(L, t) + ": " + py_repr(b, e));
          return;
        }
        if (t < L.cam_end) cams[t - L.obs_end] = v;
        else pts[t - L.cam_end] = v;
      }
      ++t;
    }
  };
  {
    std::vector<std::thread> th;
    for (int k = 1; k < T; ++k) th.emplace_back(fill, k);
    fill(0);
    for (auto& t : th) t.join();
  }
  Err first;
  for (const Err& er : errs)
    if (er.tok < first.tok) first = er;
  if (first.tok == INT64_MAX && n_tokens < L.total) {
    // truncated: reported at the line of the last token read (0 if none)
    first.tok = n_tokens;
    int64_t last_line = hs.line;  // header's last token
    for (int k = T - 1; k >= 0; --k)
      if (ntok[k] > 0) {
        Scanner sc{text + cut[k], text + cut[k + 1], ln0[k]};
        const unsigned char *b, *e;
        int64_t ln = ln0[k];
        while (sc.next(b, e)) ln = sc.line;
        last_line = ln;
        break;
      }
    first.line = last_line;
    first.msg = "truncated file: expected " + field_name(L, n_tokens);
  }
  if (first.tok != INT64_MAX) {
    set_err(err_msg, err_cap, err_line, first);
    return PV_BAL_EPARSE;
  }
  return PV_BAL_OK;
}

int pv_bal_prune_masks(int64_t n_cam, int64_t n_pt, int64_t n_obs, const int64_t* cam_idx,
                       const int64_t* pt_idx, int64_t min_cameras, uint8_t* keep_lm,
                       uint8_t* cam_seen, int64_t* n_obs_kept) {
  if (n_cam < 0 || n_pt < 0 || n_obs < 0) return 1;
  // landmark-major counting sort of the camera indices, then distinct cameras per
  // landmark with a last-seen stamp (no sort, O(n_obs))
  std::vector<int64_t> off(n_pt + 1, 0);
  for (int64_t k = 0; k < n_obs; ++k) {
    if (pt_idx[k] < 0 || pt_idx[k] >= n_pt || cam_idx[k] < 0 || cam_idx[k] >= n_cam) return 1;
    ++off[pt_idx[k] + 1];
  }
  for (int64_t j = 0; j < n_pt; ++j) off[j + 1] += off[j];
  std::vector<int64_t> pos(off.begin(), off.end() - 1), cams(n_obs);
  for (int64_t k = 0; k < n_obs; ++k) cams[pos[pt_idx[k]]++] = cam_idx[k];
  std::vector<int64_t> stamp(n_cam, -1);
  for (int64_t j = 0; j < n_pt; ++j) {
    int64_t distinct = 0;
    for (int64_t q = off[j]; q < off[j + 1]; ++q)
      if (stamp[cams[q]] != j) {
        stamp[cams[q]] = j;
        ++distinct;
      }
    keep_lm[j] = distinct >= min_cameras ? 1 : 0;
  }
  std::memset(cam_seen, 0, (size_t)n_cam);
  int64_t kept = 0;
  for (int64_t k = 0; k < n_obs; ++k)
    if (keep_lm[pt_idx[k]]) {
      cam_seen[cam_idx[k]] = 1;
      ++kept;
    }
  *n_obs_kept = kept;
  return 0;
}

}  // extern "C"
