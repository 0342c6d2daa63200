// evr_events.cpp -- host-side text event parser.
//
// The reference reads events through a per-line Python generator
// (events.py:65-130, ~3.3 us/event, 0.3 Mev/s per core -- the bottleneck
// feeding a 1 Mev/s sensor from files).  This is the same grammar and the
// same validation, straight into the packed evr_event layout the device
// ingest consumes:
//
//   line  := blank | '#' comment | t x y p      (whitespace separated)
//   ints  := Python int() of base-10 text: optional sign, digits with
//            single '_' separators
//   t >= 0, x >= 0, y >= 0, p in {0, -1 (-> -1), 1}, (x, y) inside the
//   sensor, t >= running_max - slack (running_max = max timestamp so far)
//
// On the first invalid line the parser stops and reports the kind and the
// byte offset of that line; the Python wrapper re-raises it through the
// reference-compatible Python parser so the exception type and message are
// exactly the reference's.
#include <cstdint>
#include <cstring>

#include "../../include/evr.h"

namespace {

inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f' || c == '\n';
}

// Python int() for ASCII base-10 tokens; false on any other token or overflow
bool parse_int(const char* s, const char* e, int64_t* out) {
  bool neg = false;
  if (s < e && (*s == '+' || *s == '-')) {
    neg = *s == '-';
    ++s;
  }
  if (s == e) return false;
  unsigned long long v = 0;
  bool last_digit = false;
  for (; s < e; ++s) {
    const char c = *s;
    if (c >= '0' && c <= '9') {
      if (v > (unsigned long long)INT64_MAX / 10) return false;
      v = v * 10 + (unsigned long long)(c - '0');
      if (v > (unsigned long long)INT64_MAX) return false;
      last_digit = true;
    } else if (c == '_' && last_digit && s + 1 < e && s[1] >= '0' && s[1] <= '9') {
      last_digit = false;
    } else {
      return false;
    }
  }
  *out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

}  // namespace

extern "C" int evr_parse_events(const char* text, int64_t len, int width, int height,
                                int64_t slack, evr_parse_state* st, evr_event* out, int64_t cap,
                                int64_t* n_out, int64_t* consumed, int64_t* err_offset,
                                int32_t* err_kind) {
  if (!text || !st || !out || !n_out || !consumed || !err_offset || !err_kind || len < 0)
    return EVR_ERR_INVALID;
  int64_t n = 0;
  int64_t pos = 0;
  *err_kind = EVR_PARSE_OK;
  *err_offset = -1;
  while (pos < len && n < cap) {
    const char* line = text + pos;
    const char* nl = static_cast<const char*>(memchr(line, '\n', (size_t)(len - pos)));
    const char* end = nl ? nl : text + len;
    const int64_t next = nl ? (nl - text) + 1 : len;
    st->line_no += 1;
    const char* s = line;
    const char* e = end;
    while (s < e && is_space(*s)) ++s;
    while (e > s && is_space(e[-1])) --e;
    if (s == e || *s == '#') {
      pos = next;
      continue;
    }
    // split into exactly four tokens
    const char* tb[5];
    const char* te[5];
    int nt = 0;
    const char* c = s;
    while (c < e && nt < 5) {
      while (c < e && is_space(*c)) ++c;
      if (c >= e) break;
      tb[nt] = c;
      while (c < e && !is_space(*c)) ++c;
      te[nt] = c;
      ++nt;
    }
    int64_t v[4];
    bool ok = nt == 4;
    for (int k = 0; ok && k < 4; ++k) ok = parse_int(tb[k], te[k], &v[k]);
    const int64_t t = ok ? v[0] : 0, x = ok ? v[1] : 0, y = ok ? v[2] : 0, p = ok ? v[3] : 0;
    ok = ok && t >= 0 && x >= 0 && y >= 0 && (p == 0 || p == 1 || p == -1);
    ok = ok && x < width && y < height;
    if (!ok) {
      *err_kind = EVR_PARSE_BAD_LINE;
      *err_offset = pos;
      st->line_no -= 1;  // the wrapper re-reads this line
      break;
    }
    if (st->have_max && t < st->running_max - slack) {
      *err_kind = EVR_PARSE_ORDER;
      *err_offset = pos;
      st->line_no -= 1;
      break;
    }
    if (!st->have_max || t > st->running_max) {
      st->running_max = t;
      st->have_max = 1;
    }
    out[n].t = t;
    out[n].x = (int32_t)x;
    out[n].y = (int16_t)y;
    out[n].polarity = (int16_t)(p == 1 ? 1 : -1);
    ++n;
    st->index += 1;
    pos = next;
  }
  *n_out = n;
  *consumed = pos;
  return *err_kind == EVR_PARSE_OK ? EVR_OK : EVR_ERR_INVALID;
}
