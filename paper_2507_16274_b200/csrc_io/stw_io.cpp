// libstw_io -- trace and plan files natively (include/stw_io.h).
//
// Reading: one pass over the file, a small JSON decoder per line (trace
// files) or per document (plan files) into a node tape, the reference's
// record semantics (traceio.py:48-215, 357-391) and Trace.validate
// (model.py:219-251) straight into structure-of-arrays columns.
// Writing: the reference's canonical JSON (sorted keys; compact lines for
// traces, indent=2 for plans; ASCII-only escapes) byte for byte
// (traceio.py:222-291, 334-354).
//
// Conversions follow Python's int() / str() / bool() on the JSON value types
// that occur in these files (integers, floats, booleans, decimal strings,
// null). Anything that fails -- or a value shape this reader does not model --
// is reported as STW_IOE_RECORD / _HEADER / _PLANDOC with its line, and the
// caller re-derives the exact exception text from that one record.
#include "../../include/stw_io.h"

#include <errno.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// JSON decoding into a tape of nodes (children linked through `next`)

enum JT : uint8_t { J_NULL, J_FALSE, J_TRUE, J_INT, J_FLT, J_STR, J_ARR, J_OBJ, J_BIG, J_ODD };

struct JNode {
  JT t;
  int64_t i;  // J_INT value; J_ARR/J_OBJ child count
  double f;
  uint32_t s, sl;  // string value (offset, length) in Doc::buf
  uint32_t k, kl;  // member key (objects)
  int32_t first, next;
};

struct Doc {
  std::vector<JNode> n;
  std::string buf;
  const char *p, *e;
  bool bad = false;
  void clear() {
    n.clear();
    buf.clear();
    bad = false;
  }
  std::string str(int x) const { return buf.substr(n[x].s, n[x].sl); }
  bool is_str(int x, const char *lit) const {
    return n[x].t == J_STR && n[x].sl == strlen(lit) && memcmp(buf.data() + n[x].s, lit, n[x].sl) == 0;
  }
  // object member lookup; duplicate keys: the last one wins (json.loads)
  int get(int obj, const char *key) const {
    const size_t kl = strlen(key);
    int hit = -1;
    for (int c = n[obj].first; c >= 0; c = n[c].next)
      if (n[c].kl == kl && memcmp(buf.data() + n[c].k, key, kl) == 0) hit = c;
    return hit;
  }

  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) p++;
  }
  static void put_utf8(std::string &o, uint32_t cp) {
    if (cp < 0x80) {
      o += (char)cp;
    } else if (cp < 0x800) {
      o += (char)(0xC0 | (cp >> 6));
      o += (char)(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      o += (char)(0xE0 | (cp >> 12));
      o += (char)(0x80 | ((cp >> 6) & 0x3F));
      o += (char)(0x80 | (cp & 0x3F));
    } else {
      o += (char)(0xF0 | (cp >> 18));
      o += (char)(0x80 | ((cp >> 12) & 0x3F));
      o += (char)(0x80 | ((cp >> 6) & 0x3F));
      o += (char)(0x80 | (cp & 0x3F));
    }
  }
  bool hex4(uint32_t *v) {
    if (e - p < 4) return false;
    uint32_t x = 0;
    for (int k = 0; k < 4; k++) {
      const char c = p[k];
      x <<= 4;
      if (c >= '0' && c <= '9') x |= c - '0';
      else if (c >= 'a' && c <= 'f') x |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') x |= c - 'A' + 10;
      else return false;
    }
    p += 4;
    *v = x;
    return true;
  }
  // decodes a string starting after the opening quote into buf
  bool string(uint32_t *off, uint32_t *len) {
    *off = (uint32_t)buf.size();
    while (true) {
      if (p >= e) return false;
      const unsigned char c = (unsigned char)*p++;
      if (c == '"') break;
      if (c < 0x20) return false;  // strict: no raw control characters
      if (c != '\\') {
        buf += (char)c;
        continue;
      }
      if (p >= e) return false;
      const char x = *p++;
      switch (x) {
        case '"': buf += '"'; break;
        case '\\': buf += '\\'; break;
        case '/': buf += '/'; break;
        case 'b': buf += '\b'; break;
        case 'f': buf += '\f'; break;
        case 'n': buf += '\n'; break;
        case 'r': buf += '\r'; break;
        case 't': buf += '\t'; break;
        case 'u': {
          uint32_t cp;
          if (!hex4(&cp)) return false;
          if (cp >= 0xD800 && cp < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            const char *save = p;
            p += 2;
            uint32_t lo;
            if (hex4(&lo) && lo >= 0xDC00 && lo < 0xE000) {
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else {
              p = save;
            }
          }
          if (cp >= 0xD800 && cp < 0xE000) bad = true;  // lone surrogate: valid JSON, not modelled here
          put_utf8(buf, cp);
          break;
        }
        default: return false;
      }
    }
    *len = (uint32_t)buf.size() - *off;
    return true;
  }
  int node(JT t) {
    JNode x{};
    x.t = t;
    x.first = x.next = -1;
    n.push_back(x);
    return (int)n.size() - 1;
  }
  bool lit(const char *w) {
    const size_t l = strlen(w);
    if ((size_t)(e - p) < l || memcmp(p, w, l) != 0) return false;
    p += l;
    return true;
  }
  int flt(double v) {
    const int x = node(J_FLT);
    n[x].f = v;
    return x;
  }
  int number() {
    const char *s = p;
    if (p < e && *p == '-') p++;
    if (p >= e) return -1;
    if (*p == '0') {
      p++;
    } else if (*p >= '1' && *p <= '9') {
      while (p < e && *p >= '0' && *p <= '9') p++;
    } else {
      return -1;
    }
    bool flt = false;
    if (p < e && *p == '.' && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      flt = true;
      p++;
      while (p < e && *p >= '0' && *p <= '9') p++;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      const char *q = p + 1;
      if (q < e && (*q == '+' || *q == '-')) q++;
      if (q < e && *q >= '0' && *q <= '9') {
        flt = true;
        p = q;
        while (p < e && *p >= '0' && *p <= '9') p++;
      }
    }
    std::string lit(s, p - s);
    if (flt) {
      const int x = node(J_FLT);
      n[x].f = strtod(lit.c_str(), nullptr);
      return x;
    }
    errno = 0;
    const long long v = strtoll(lit.c_str(), nullptr, 10);
    const int x = node(errno == ERANGE ? J_BIG : J_INT);
    n[x].i = v;
    n[x].s = (uint32_t)buf.size();  // the literal, for str() of integers beyond int64
    n[x].sl = (uint32_t)lit.size();
    buf += lit;
    return x;
  }
  int value(int depth) {
    ws();
    if (p >= e || depth > 64) return -1;
    const char c = *p;
    if (c == '{') {
      p++;
      const int x = node(J_OBJ);
      int last = -1;
      ws();
      if (p < e && *p == '}') {
        p++;
        return x;
      }
      while (true) {
        ws();
        if (p >= e || *p != '"') return -1;
        p++;
        uint32_t ko, kl;
        if (!string(&ko, &kl)) return -1;
        ws();
        if (p >= e || *p != ':') return -1;
        p++;
        const int v = value(depth + 1);
        if (v < 0) return -1;
        n[v].k = ko;
        n[v].kl = kl;
        if (last < 0) n[x].first = v;
        else n[last].next = v;
        last = v;
        n[x].i++;
        ws();
        if (p < e && *p == ',') {
          p++;
          continue;
        }
        if (p < e && *p == '}') {
          p++;
          return x;
        }
        return -1;
      }
    }
    if (c == '[') {
      p++;
      const int x = node(J_ARR);
      int last = -1;
      ws();
      if (p < e && *p == ']') {
        p++;
        return x;
      }
      while (true) {
        const int v = value(depth + 1);
        if (v < 0) return -1;
        if (last < 0) n[x].first = v;
        else n[last].next = v;
        last = v;
        n[x].i++;
        ws();
        if (p < e && *p == ',') {
          p++;
          continue;
        }
        if (p < e && *p == ']') {
          p++;
          return x;
        }
        return -1;
      }
    }
    if (c == '"') {
      p++;
      const int x = node(J_STR);
      uint32_t o, l;
      if (!string(&o, &l)) return -1;
      n[x].s = o;
      n[x].sl = l;
      return x;
    }
    if (lit("true")) return node(J_TRUE);
    if (lit("false")) return node(J_FALSE);
    if (lit("null")) return node(J_NULL);
    // accepted by json.loads
    if (lit("NaN")) return flt(NAN);
    if (lit("Infinity")) return flt(INFINITY);
    if (lit("-Infinity")) return flt(-INFINITY);
    return number();
  }
  // whole input must be one value (json.loads: "Extra data" otherwise)
  int parse(const char *b, const char *end) {
    clear();
    p = b;
    e = end;
    const int r = value(0);
    if (r < 0) return -1;
    ws();
    return p == e ? r : -1;
  }
};

// Python int(v) for the value shapes these files hold; false = conversion
// error or shape not modelled
bool py_int(const Doc &d, int x, int64_t *out) {
  const JNode &v = d.n[x];
  switch (v.t) {
    case J_INT: *out = v.i; return true;
    case J_TRUE: *out = 1; return true;
    case J_FALSE: *out = 0; return true;
    case J_FLT:
      if (!isfinite(v.f) || fabs(v.f) >= 9.2e18) return false;
      *out = (int64_t)trunc(v.f);
      return true;
    case J_STR: {  // [ws][+-]digits with single underscores between digits[ws], ASCII only
      const std::string s = d.str(x);
      size_t a = 0, b = s.size();
      auto sp = [](char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; };
      while (a < b && sp(s[a])) a++;
      while (b > a && sp(s[b - 1])) b--;
      bool neg = false;
      if (a < b && (s[a] == '+' || s[a] == '-')) neg = s[a++] == '-';
      if (a >= b) return false;
      __int128 acc = 0;
      bool prev_digit = false;
      for (size_t k = a; k < b; k++) {
        const char c = s[k];
        if (c >= '0' && c <= '9') {
          acc = acc * 10 + (c - '0');
          if (acc > ((__int128)1 << 63)) return false;
          prev_digit = true;
        } else if (c == '_' && prev_digit && k + 1 < b && s[k + 1] >= '0' && s[k + 1] <= '9') {
          prev_digit = false;
        } else {
          return false;
        }
      }
      if (neg) acc = -acc;
      if (acc > INT64_MAX || acc < INT64_MIN) return false;
      *out = (int64_t)acc;
      return true;
    }
    default: return false;
  }
}

bool py_truth(const Doc &d, int x) {
  const JNode &v = d.n[x];
  switch (v.t) {
    case J_NULL: case J_FALSE: return false;
    case J_INT: return v.i != 0;
    case J_FLT: return v.f != 0.0;
    case J_STR: return v.sl > 0;
    case J_ARR: case J_OBJ: return v.i > 0;
    default: return true;
  }
}

// Python repr(float): the shortest digits that round-trip, fixed notation for
// decimal exponents in [-4, 16), else d.ddde+XX
std::string py_float(double f) {
  if (isnan(f)) return "nan";
  if (isinf(f)) return f > 0 ? "inf" : "-inf";
  char b[40];
  int prec = 0;
  for (; prec < 17; prec++) {
    snprintf(b, sizeof b, "%.*e", prec, f);
    if (strtod(b, nullptr) == f) break;
  }
  snprintf(b, sizeof b, "%.*e", prec, f);
  std::string s(b);
  const bool neg = s[0] == '-';
  if (neg) s = s.substr(1);
  const size_t epos = s.find('e');
  const int ex = atoi(s.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; i++)
    if (s[i] != '.') digits += s[i];
  std::string o;
  if (ex >= -4 && ex < 16) {
    if (ex < 0) {
      o = "0." + std::string(-ex - 1, '0') + digits;
    } else if ((int)digits.size() <= ex + 1) {
      o = digits + std::string(ex + 1 - digits.size(), '0') + ".0";
    } else {
      o = digits.substr(0, ex + 1) + "." + digits.substr(ex + 1);
    }
  } else {
    o = digits.substr(0, 1);
    if (digits.size() > 1) o += "." + digits.substr(1);
    char eb[8];
    snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    o += eb;
  }
  return neg ? "-" + o : o;
}

std::string py_repr(const std::string &s);

// Python repr() of a decoded JSON value (str() of a container uses it)
std::string py_repr_value(const Doc &d, int x) {
  const JNode &v = d.n[x];
  switch (v.t) {
    case J_NULL: return "None";
    case J_FALSE: return "False";
    case J_TRUE: return "True";
    case J_INT: return std::to_string(v.i);
    case J_BIG: return d.str(x);
    case J_FLT: return py_float(v.f);
    case J_STR: return py_repr(d.str(x));
    case J_ARR: {
      std::string o = "[";
      for (int c = v.first; c >= 0; c = d.n[c].next) o += (c == v.first ? "" : ", ") + py_repr_value(d, c);
      return o + "]";
    }
    case J_OBJ: {  // duplicate keys collapse to the last value, at the first key's position
      std::vector<int> keep;
      for (int c = v.first; c >= 0; c = d.n[c].next) {
        bool dup = false;
        for (int &k : keep)
          if (d.n[k].kl == d.n[c].kl && memcmp(d.buf.data() + d.n[k].k, d.buf.data() + d.n[c].k, d.n[c].kl) == 0)
            k = c, dup = true;
        if (!dup) keep.push_back(c);
      }
      std::string o = "{";
      for (size_t j = 0; j < keep.size(); j++) {
        const int c = keep[j];
        o += (j ? ", " : "") + py_repr(d.buf.substr(d.n[c].k, d.n[c].kl)) + ": " + py_repr_value(d, c);
      }
      return o + "}";
    }
    default: return "?";
  }
}

// Python str(v) for module names; false = shape not modelled
bool py_str(const Doc &d, int x, std::string *out) {
  const JNode &v = d.n[x];
  switch (v.t) {
    case J_ARR: case J_OBJ: *out = py_repr_value(d, x); return !d.bad;
    case J_STR: *out = d.str(x); return true;
    case J_BIG: *out = d.str(x); return true;
    case J_FLT: *out = py_float(v.f); return true;
    case J_INT: *out = std::to_string(v.i); return true;
    case J_TRUE: *out = "True"; return true;
    case J_FALSE: *out = "False"; return true;
    case J_NULL: *out = "None"; return true;
    default: return false;
  }
}

// ---------------------------------------------------------------------------
// phases: (kind, microbatch, chunk) packed like PhaseId's ordering

typedef int64_t PKey;

bool parse_phase(const std::string &tag, PKey *k) {  // PhaseId.parse (model.py:78-88)
  if (tag == "init") return *k = 0, true;
  if (tag == "opt") return *k = (int64_t)3 << 60, true;
  if (tag.size() < 3 || (tag[0] != 'F' && tag[0] != 'B') || tag[1] != ':') return false;
  size_t i = 2;
  auto digits = [&](int64_t *v) {
    const size_t s = i;
    int64_t acc = 0;
    while (i < tag.size() && tag[i] >= '0' && tag[i] <= '9') {
      acc = acc * 10 + (tag[i] - '0');
      if (acc >= ((int64_t)1 << 30)) return false;
      i++;
    }
    *v = acc;
    return i > s;
  };
  int64_t mb = 0, ch = 0;
  if (!digits(&mb)) return false;
  if (i < tag.size()) {
    if (tag[i] != '.') return false;
    i++;
    if (!digits(&ch)) return false;
  }
  if (i != tag.size()) return false;
  *k = ((int64_t)(tag[0] == 'F' ? 1 : 2) << 60) | (mb << 30) | ch;
  return true;
}

std::string phase_tag(PKey k) {  // PhaseId.tag (model.py:66-75)
  const int kind = (int)(k >> 60);
  if (kind == 0) return "init";
  if (kind == 3) return "opt";
  const int64_t mb = (k >> 30) & ((1 << 30) - 1), ch = k & ((1 << 30) - 1);
  std::string s = (kind == 1 ? "F:" : "B:") + std::to_string(mb);
  if (ch) s += "." + std::to_string(ch);
  return s;
}

// Python repr() of a str (the message of unknown-layer errors)
std::string py_repr(const std::string &s) {
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string o(1, q);
  for (size_t i = 0; i < s.size(); i++) {
    const unsigned char c = (unsigned char)s[i];
    if (c == '\\') o += "\\\\";
    else if (c == (unsigned char)q) o += '\\', o += (char)c;
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c == '\t') o += "\\t";
    else if (c < 0x20 || c == 0x7F) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      o += b;
    } else o += (char)c;
  }
  return o + q;
}

}  // namespace

// ---------------------------------------------------------------------------
// parsed trace

struct stw_trace_file {
  std::vector<int64_t> id, size, t_s, t_e;
  std::vector<int32_t> ps, pe, ls, le;
  std::vector<uint8_t> dyn;
  std::vector<std::string> tags, names;
  std::vector<int64_t> ph_start, ph_end, ly_start, ly_end;
  int64_t n_sched = 0, n_known = 0;
};

namespace {

void set_err(stw_io_error *e, int kind, int64_t line, const char *fmt, ...) {
  if (!e) return;
  e->kind = kind;
  e->line = line;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(e->text, sizeof e->text, fmt, ap);
  va_end(ap);
}

bool read_file(const char *path, std::string *out, stw_io_error *e) {
  FILE *f = fopen(path, "rb");
  if (!f) {
    set_err(e, STW_IOE_OS, errno, "%s", strerror(errno));
    return false;
  }
  char chunk[1 << 16];
  size_t k;
  while ((k = fread(chunk, 1, sizeof chunk, f)) > 0) out->append(chunk, k);
  const bool ok = !ferror(f);
  fclose(f);
  if (!ok) set_err(e, STW_IOE_OS, EIO, "read error");
  return ok;
}

// str.splitlines() boundaries (incl. \v \f \x1c-\x1e, U+0085, U+2028/9)
void split_lines(const std::string &s, std::vector<std::pair<size_t, size_t>> *lines) {
  size_t a = 0, i = 0;
  const size_t n = s.size();
  while (i < n) {
    const unsigned char c = (unsigned char)s[i];
    size_t adv = 0;
    if (c == '\n' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e) adv = 1;
    else if (c == '\r') adv = (i + 1 < n && s[i + 1] == '\n') ? 2 : 1;
    else if (c == 0xC2 && i + 1 < n && (unsigned char)s[i + 1] == 0x85) adv = 2;
    else if (c == 0xE2 && i + 2 < n && (unsigned char)s[i + 1] == 0x80 &&
             ((unsigned char)s[i + 2] == 0xA8 || (unsigned char)s[i + 2] == 0xA9)) adv = 3;
    if (adv) {
      lines->push_back({a, i});
      i += adv;
      a = i;
    } else {
      i++;
    }
  }
  if (a < n) lines->push_back({a, n});
}

struct Ev {
  int64_t id, size, t_s, t_e;
  PKey ps, pe;
  bool dyn;
  std::string ls, le;
};

// Trace.validate (model.py:219-251) over the columns
bool validate(stw_trace_file &T, const std::vector<PKey> &sched_keys, const std::vector<PKey> &tag_keys,
              stw_io_error *e) {
  const int64_t horizon = T.n_sched ? T.ph_end[T.n_sched - 1] : 0;
  int64_t prev = 0;
  for (int64_t s = 0; s < T.n_sched; s++) {
    if (T.ph_start[s] < prev || T.ph_end[s] <= T.ph_start[s]) {
      set_err(e, STW_IOE_MSG, 0, "phase schedule not ordered/disjoint at %s", T.tags[s].c_str());
      return false;
    }
    prev = T.ph_end[s];
  }
  std::unordered_map<PKey, int64_t> index;  // last occurrence wins (dict comprehension)
  for (int64_t s = 0; s < T.n_sched; s++) index[sched_keys[s]] = s;
  if ((int64_t)index.size() != T.n_sched) {
    set_err(e, STW_IOE_MSG, 0, "duplicate phase in schedule");
    return false;
  }
  std::unordered_set<std::string> known;
  for (int64_t k = 0; k < T.n_known; k++) known.insert(T.names[k]);
  if ((int64_t)known.size() != T.n_known) {
    set_err(e, STW_IOE_MSG, 0, "duplicate layer instance in schedule");
    return false;
  }
  std::unordered_set<int64_t> seen;
  seen.reserve(T.id.size() * 2);
  auto pidx = [&](int32_t tag) -> int64_t {
    auto it = index.find(tag_keys[tag]);
    return it == index.end() ? -1 : it->second;
  };
  auto inside = [&](int32_t tag, int64_t t) {
    const int64_t s = pidx(tag);
    return s >= 0 && T.ph_start[s] <= t && t < T.ph_end[s];
  };
  for (size_t i = 0; i < T.id.size(); i++) {
    const long long id = (long long)T.id[i];
    if (!seen.insert(T.id[i]).second) {
      set_err(e, STW_IOE_MSG, 0, "duplicate event id %lld", id);
      return false;
    }
    if (!(0 <= T.t_s[i] && T.t_s[i] < horizon) || T.t_e[i] > horizon) {
      set_err(e, STW_IOE_MSG, 0, "event %lld: timestamps outside [0, horizon]", id);
      return false;
    }
    if (!inside(T.ps[i], T.t_s[i])) {
      set_err(e, STW_IOE_MSG, 0, "event %lld: t_s not inside phase %s", id, T.tags[T.ps[i]].c_str());
      return false;
    }
    if (T.t_e[i] < horizon && !inside(T.pe[i], T.t_e[i])) {
      set_err(e, STW_IOE_MSG, 0, "event %lld: t_e not inside phase %s", id, T.tags[T.pe[i]].c_str());
      return false;
    }
    const int64_t a = pidx(T.ps[i]), b = pidx(T.pe[i]);
    if (b < 0) {
      set_err(e, STW_IOE_MSG, 0, "phase %s not in schedule", T.tags[T.pe[i]].c_str());
      return false;
    }
    if (a > b) {
      set_err(e, STW_IOE_MSG, 0, "event %lld: p_s after p_e in phase order", id);
      return false;
    }
    if (T.dyn[i])
      for (int32_t l : {T.ls[i], T.le[i]}) {
        if (T.names[l][0] == '\x02') {  // `name in dict` on a list / dict value
          set_err(e, STW_IOE_TYPE, 0, "unhashable type: '%s'", T.names[l].c_str() + 1);
          return false;
        }
        if (!known.count(T.names[l]) || T.names[l][0] == '\x01') {
          const std::string &nm = T.names[l];
          set_err(e, STW_IOE_MSG, 0, "event %lld: unknown layer %s", id,
                  nm[0] == '\x01' ? nm.c_str() + 1 : py_repr(nm).c_str());
          return false;
        }
      }
  }
  return true;
}

// ---- raw layout (traceio.py:90-182) --------------------------------------

bool parse_raw(const char *path, const std::string &s, const std::vector<std::pair<size_t, size_t>> &lines,
               stw_trace_file &T, std::vector<PKey> &sched, stw_io_error *e) {
  struct Open {
    int64_t t_s, size;
    PKey phase;
    std::string module;
    bool dyn, open;
  };
  std::unordered_map<int64_t, size_t> open_at;  // rid -> index into opens (alloc order)
  std::vector<std::pair<int64_t, Open>> opens;
  std::unordered_set<int64_t> alloc_ids;
  std::unordered_set<PKey> seen_phase;
  std::map<std::string, std::pair<int64_t, int64_t>> layer;  // name -> (lo, hi), sorted by name
  std::vector<Ev> closed;
  std::vector<int64_t> sp_start, sp_end;
  Doc d;
  const int64_t nrec = (int64_t)lines.size() - 1;
  closed.reserve(nrec / 2 + 1);
  for (int64_t t = 0; t < nrec; t++) {
    const int64_t lineno = t + 2;
    const auto &L = lines[t + 1];
    const int r = d.parse(s.data() + L.first, s.data() + L.second);
    if (r < 0) return set_err(e, STW_IOE_JSON, lineno, "json"), false;
    if (d.n[r].t != J_OBJ) return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: expected a JSON object", path, (long long)lineno), false;
    const int op = d.get(r, "op"), idn = d.get(r, "id"), phn = d.get(r, "phase");
    int64_t rid;
    PKey phase;
    if (d.bad || op < 0 || idn < 0 || phn < 0 || !py_int(d, idn, &rid) || d.n[phn].t != J_STR ||
        !parse_phase(d.str(phn), &phase))
      return set_err(e, STW_IOE_RECORD, lineno, "record"), false;
    std::string module;
    const int mn = d.get(r, "module");
    if (mn >= 0 && !py_str(d, mn, &module)) return set_err(e, STW_IOE_RECORD, lineno, "module"), false;
    if (sched.empty() || sched.back() != phase) {
      if (seen_phase.count(phase))
        return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: phase %s re-opened", path, (long long)lineno,
                       phase_tag(phase).c_str()), false;
      seen_phase.insert(phase);
      sched.push_back(phase);
      sp_start.push_back(t);
      sp_end.push_back(t + 1);
    } else {
      sp_end.back() = t + 1;
    }
    if (d.is_str(op, "alloc")) {
      if (!alloc_ids.insert(rid).second)
        return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: duplicate alloc id %lld", path, (long long)lineno,
                       (long long)rid), false;
      const int dn = d.get(r, "dynamic");
      const bool dyn = dn >= 0 && py_truth(d, dn);
      if (dyn && module.empty())
        return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: dynamic event missing layer", path, (long long)lineno),
               false;
      const int sn = d.get(r, "size");
      int64_t size;
      if (sn < 0 || !py_int(d, sn, &size) || size <= 0 || size > INT64_MAX - 511)
        return set_err(e, STW_IOE_RECORD, lineno, "size"), false;
      size = (size + 511) / 512 * 512;  // align_up (model.py:34-37)
      open_at[rid] = opens.size();
      opens.push_back({rid, Open{t, size, phase, module, dyn, true}});
      if (dyn) {
        layer.emplace(module, std::make_pair(t, t + 1)).first->second.second = t + 1;
      }
    } else if (d.is_str(op, "free")) {
      auto it = open_at.find(rid);
      if (it == open_at.end())
        return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: free without matching alloc (id %lld)", path,
                       (long long)lineno, (long long)rid), false;
      Open &st = opens[it->second].second;
      open_at.erase(it);
      st.open = false;
      Ev ev{rid, st.size, st.t_s, t, st.phase, phase, st.dyn, "", ""};
      if (st.dyn) {
        if (module.empty())
          return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: dynamic event missing layer", path, (long long)lineno),
                 false;
        ev.ls = st.module;
        ev.le = module;
        layer.emplace(module, std::make_pair(t, t + 1)).first->second.second = t + 1;
      }
      closed.push_back(std::move(ev));
    } else {
      return set_err(e, STW_IOE_RECORD, lineno, "op"), false;  // unknown op {op!r}: repr by the caller
    }
  }
  const int64_t horizon = nrec;
  if (sched.empty()) return set_err(e, STW_IOE_MSG, 0, "%s: trace has no records", path), false;
  const PKey last = sched.back();
  for (auto &kv : opens) {
    if (!kv.second.open) continue;
    if (kv.second.dyn)
      return set_err(e, STW_IOE_MSG, 0, "%s: dynamic event %lld never freed", path, (long long)kv.first), false;
    closed.push_back(Ev{kv.first, kv.second.size, kv.second.t_s, horizon, kv.second.phase, last, false, "", ""});
  }
  std::sort(closed.begin(), closed.end(),
            [](const Ev &a, const Ev &b) { return a.t_s != b.t_s ? a.t_s < b.t_s : a.id < b.id; });
  // columns: the schedule is every phase (unique here); layers sorted by name
  std::unordered_map<PKey, int32_t> pix;
  for (size_t k = 0; k < sched.size(); k++) {
    pix[sched[k]] = (int32_t)k;
    T.tags.push_back(phase_tag(sched[k]));
  }
  T.n_sched = (int64_t)sched.size();
  T.ph_start = sp_start;
  T.ph_end = sp_end;
  std::unordered_map<std::string, int32_t> lix;
  for (auto &kv : layer) {
    lix[kv.first] = (int32_t)T.names.size();
    T.names.push_back(kv.first);
    T.ly_start.push_back(kv.second.first);
    T.ly_end.push_back(kv.second.second);
  }
  T.n_known = (int64_t)T.names.size();
  const size_t n = closed.size();
  T.id.resize(n), T.size.resize(n), T.t_s.resize(n), T.t_e.resize(n);
  T.ps.resize(n), T.pe.resize(n), T.ls.resize(n), T.le.resize(n), T.dyn.resize(n);
  for (size_t i = 0; i < n; i++) {
    const Ev &v = closed[i];
    T.id[i] = v.id, T.size[i] = v.size, T.t_s[i] = v.t_s, T.t_e[i] = v.t_e;
    T.ps[i] = pix[v.ps], T.pe[i] = pix[v.pe], T.dyn[i] = v.dyn;
    T.ls[i] = v.dyn ? lix[v.ls] : -1;
    T.le[i] = v.dyn ? lix[v.le] : -1;
  }
  return true;
}

// ---- paired layout (traceio.py:185-215) ----------------------------------

bool parse_paired(const char *path, const std::string &s, const std::vector<std::pair<size_t, size_t>> &lines,
                  Doc &hd, int hr, stw_trace_file &T, std::vector<PKey> &sched, std::vector<PKey> &tag_keys,
                  stw_io_error *e) {
  // header schedules: [tag, start, end] triples
  // an empty str / dict iterates like an empty list
  auto empty_iter = [&](int x) {
    return (hd.n[x].t == J_OBJ && hd.n[x].i == 0) || (hd.n[x].t == J_STR && hd.n[x].sl == 0);
  };
  const int phs = hd.get(hr, "phases");
  if (phs < 0 || (hd.n[phs].t != J_ARR && !empty_iter(phs))) return set_err(e, STW_IOE_HEADER, 1, "phases"), false;
  std::unordered_map<PKey, int32_t> tix;  // tag key -> index into T.tags (last schedule slot wins)
  for (int c = hd.n[phs].first; c >= 0; c = hd.n[c].next) {
    int64_t st, en;
    PKey k;
    const int a = hd.n[c].first;
    if (hd.n[c].t != J_ARR || hd.n[c].i != 3 || hd.n[a].t != J_STR || !parse_phase(hd.str(a), &k) ||
        !py_int(hd, hd.n[a].next, &st) || !py_int(hd, hd.n[hd.n[a].next].next, &en))
      return set_err(e, STW_IOE_HEADER, 1, "phases"), false;
    tix[k] = (int32_t)T.tags.size();
    sched.push_back(k);
    tag_keys.push_back(k);
    T.tags.push_back(phase_tag(k));
    T.ph_start.push_back(st);
    T.ph_end.push_back(en);
  }
  T.n_sched = (int64_t)sched.size();
  std::unordered_map<std::string, int32_t> lix;  // name -> first schedule slot
  const int lys = hd.get(hr, "layers");
  if (lys >= 0) {
    if (hd.n[lys].t != J_ARR && !empty_iter(lys)) return set_err(e, STW_IOE_HEADER, 1, "layers"), false;
    for (int c = hd.n[lys].first; c >= 0; c = hd.n[c].next) {
      int64_t st, en;
      std::string name;
      const int a = hd.n[c].first;
      if (hd.n[c].t != J_ARR || hd.n[c].i != 3 || !py_str(hd, a, &name) || !py_int(hd, hd.n[a].next, &st) ||
          !py_int(hd, hd.n[hd.n[a].next].next, &en))
        return set_err(e, STW_IOE_HEADER, 1, "layers"), false;
      lix.emplace(name, (int32_t)T.names.size());
      T.names.push_back(name);
      T.ly_start.push_back(st);
      T.ly_end.push_back(en);
    }
  }
  if (hd.bad) return set_err(e, STW_IOE_HEADER, 1, "header"), false;
  T.n_known = (int64_t)T.names.size();
  auto tag_index = [&](PKey k) {
    auto it = tix.find(k);
    if (it != tix.end()) return it->second;
    const int32_t x = (int32_t)T.tags.size();
    tix[k] = x;
    tag_keys.push_back(k);
    T.tags.push_back(phase_tag(k));
    return x;
  };
  auto name_index = [&](const std::string &nm) {
    auto it = lix.find(nm);
    if (it != lix.end()) return it->second;
    const int32_t x = (int32_t)T.names.size();
    lix[nm] = x;
    T.names.push_back(nm);
    return x;
  };
  Doc d;
  const size_t n = lines.size() - 1;
  T.id.reserve(n), T.size.reserve(n), T.t_s.reserve(n), T.t_e.reserve(n);
  for (size_t i = 1; i < lines.size(); i++) {
    const int64_t lineno = (int64_t)i + 1;
    const int r = d.parse(s.data() + lines[i].first, s.data() + lines[i].second);
    if (r < 0) return set_err(e, STW_IOE_JSON, lineno, "json"), false;
    if (d.n[r].t != J_OBJ) return set_err(e, STW_IOE_MSG, lineno, "%s:%lld: expected a JSON object", path, (long long)lineno), false;
    const int in = d.get(r, "id"), sn = d.get(r, "size"), an = d.get(r, "t_s"), bn = d.get(r, "t_e");
    const int pn = d.get(r, "p_s"), qn = d.get(r, "p_e"), dn = d.get(r, "dynamic");
    const int l1 = d.get(r, "l_s"), l2 = d.get(r, "l_e");
    int64_t id, size, ts, te;
    PKey ps, pe;
    if (d.bad || in < 0 || sn < 0 || an < 0 || bn < 0 || pn < 0 || qn < 0 || dn < 0 || !py_int(d, in, &id) ||
        !py_int(d, sn, &size) || size <= 0 || size > INT64_MAX - 511 || !py_int(d, an, &ts) || !py_int(d, bn, &te) ||
        d.n[pn].t != J_STR || !parse_phase(d.str(pn), &ps) || d.n[qn].t != J_STR || !parse_phase(d.str(qn), &pe))
      return set_err(e, STW_IOE_RECORD, lineno, "record"), false;
    size = (size + 511) / 512 * 512;
    const bool dyn = py_truth(d, dn);
    const bool has1 = l1 >= 0 && d.n[l1].t != J_NULL, has2 = l2 >= 0 && d.n[l2].t != J_NULL;
    // a layer name that is not a string never matches the (str) layer schedule:
    // kept as "\x01" + its repr for validate's unknown-layer message
    auto lname = [&](int x) -> std::string {
      if (d.n[x].t == J_STR) return d.str(x);
      if (d.n[x].t == J_ARR) return "\x02" "list";
      if (d.n[x].t == J_OBJ) return "\x02" "dict";
      return "\x01" + py_repr_value(d, x);
    };
    // MemoryRequestEvent.__post_init__ (model.py:112-120)
    if (te <= ts) return set_err(e, STW_IOE_MSG, 0, "event %lld: t_e must exceed t_s", (long long)id), false;
    if (dyn && !(has1 && has2))
      return set_err(e, STW_IOE_MSG, 0, "event %lld: dynamic event missing layer", (long long)id), false;
    if (!dyn && (has1 || has2))
      return set_err(e, STW_IOE_MSG, 0, "event %lld: static event carries layer names", (long long)id), false;
    T.id.push_back(id), T.size.push_back(size), T.t_s.push_back(ts), T.t_e.push_back(te);
    T.ps.push_back(tag_index(ps)), T.pe.push_back(tag_index(pe)), T.dyn.push_back(dyn);
    T.ls.push_back(dyn ? name_index(lname(l1)) : -1);
    T.le.push_back(dyn ? name_index(lname(l2)) : -1);
  }
  return true;
}

// ---- writing ---------------------------------------------------------------

// json.dumps string (ensure_ascii): escapes, \uXXXX for non-ASCII (surrogate pairs above the BMP)
void jstr(std::string &o, const char *s) {
  o += '"';
  const unsigned char *p = (const unsigned char *)s;
  while (*p) {
    const unsigned char c = *p;
    if (c < 0x80) {
      switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        default:
          if (c < 0x20) {
            char b[8];
            snprintf(b, sizeof b, "\\u%04x", c);
            o += b;
          } else {
            o += (char)c;
          }
      }
      p++;
      continue;
    }
    uint32_t cp;
    int len;
    if ((c & 0xE0) == 0xC0) cp = c & 0x1F, len = 2;
    else if ((c & 0xF0) == 0xE0) cp = c & 0x0F, len = 3;
    else cp = c & 0x07, len = 4;
    for (int k = 1; k < len && p[k]; k++) cp = (cp << 6) | (p[k] & 0x3F);
    p += len;
    char b[16];
    if (cp >= 0x10000) {
      cp -= 0x10000;
      snprintf(b, sizeof b, "\\u%04x\\u%04x", 0xD800 + (cp >> 10), 0xDC00 + (cp & 0x3FF));
    } else {
      snprintf(b, sizeof b, "\\u%04x", cp);
    }
    o += b;
  }
  o += '"';
}

void jint(std::string &o, int64_t v) {
  char b[24];
  snprintf(b, sizeof b, "%lld", (long long)v);
  o += b;
}

bool write_file(const char *path, const std::string &data, stw_io_error *e) {
  FILE *f = fopen(path, "wb");
  if (!f) {
    set_err(e, STW_IOE_OS, errno, "%s", strerror(errno));
    return false;
  }
  const bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
  if (fclose(f) != 0 || !ok) {
    set_err(e, STW_IOE_OS, EIO, "write error");
    return false;
  }
  return true;
}

}  // namespace

// ---------------------------------------------------------------------------
// plan file

struct stw_plan_file {
  int64_t pool_size = 0, alignment = 512;
  std::vector<int64_t> id, addr, size, t_s, t_e;
  std::vector<std::string> ls, le;
  std::vector<int64_t> iv_off{0}, iv_lo, iv_hi;
};

extern "C" {

int stw_trace_read(const char *path, stw_trace_file **out, stw_io_error *e) {
  *out = nullptr;
  if (e) e->kind = 0, e->line = 0, e->text[0] = 0;
  std::string s;
  if (!read_file(path, &s, e)) return STW_ETRACE;
  std::vector<std::pair<size_t, size_t>> lines;
  split_lines(s, &lines);
  if (lines.empty()) return set_err(e, STW_IOE_MSG, 0, "%s: empty trace file", path), STW_ETRACE;
  Doc hd;
  const int hr = hd.parse(s.data() + lines[0].first, s.data() + lines[0].second);
  if (hr < 0) return set_err(e, STW_IOE_JSON, 1, "json"), STW_ETRACE;
  if (hd.n[hr].t != J_OBJ) return set_err(e, STW_IOE_MSG, 1, "%s:1: expected a JSON object", path), STW_ETRACE;
  const int kn = hd.get(hr, "kind");
  if (kn < 0 || !hd.is_str(kn, "trace")) return set_err(e, STW_IOE_MSG, 0, "%s: not a trace file", path), STW_ETRACE;
  const int vn = hd.get(hr, "version");
  const bool v1 = vn >= 0 && ((hd.n[vn].t == J_INT && hd.n[vn].i == 1) || hd.n[vn].t == J_TRUE ||
                              (hd.n[vn].t == J_FLT && hd.n[vn].f == 1.0));
  if (!v1) return set_err(e, STW_IOE_HEADER, 1, "version"), STW_ETRACE;  // message formatted by the caller
  const int fn = hd.get(hr, "format");
  const bool raw = fn < 0 || hd.is_str(fn, "raw"), paired = fn >= 0 && hd.is_str(fn, "paired");
  if (!raw && !paired) return set_err(e, STW_IOE_HEADER, 1, "format"), STW_ETRACE;
  stw_trace_file *T = new stw_trace_file();
  std::vector<PKey> sched, tag_keys;
  bool ok = raw ? parse_raw(path, s, lines, *T, sched, e) : parse_paired(path, s, lines, hd, hr, *T, sched, tag_keys, e);
  if (ok && raw) tag_keys = sched;
  if (ok) ok = validate(*T, sched, tag_keys, e);
  if (!ok) {
    delete T;
    return STW_ETRACE;
  }
  *out = T;
  return STW_OK;
}

void stw_trace_free(stw_trace_file *t) { delete t; }

void stw_trace_sizes(const stw_trace_file *t, int64_t *z) {
  z[0] = (int64_t)t->id.size();
  z[1] = (int64_t)t->tags.size();
  z[2] = t->n_sched;
  z[3] = (int64_t)t->names.size();
  z[4] = t->n_known;
}

void stw_trace_events(const stw_trace_file *t, int64_t *id, int64_t *size, int64_t *t_s, int64_t *t_e, int32_t *ps,
                      int32_t *pe, uint8_t *dyn, int32_t *ls, int32_t *le) {
  const size_t n = t->id.size();
  if (!n) return;
  memcpy(id, t->id.data(), n * 8), memcpy(size, t->size.data(), n * 8);
  memcpy(t_s, t->t_s.data(), n * 8), memcpy(t_e, t->t_e.data(), n * 8);
  memcpy(ps, t->ps.data(), n * 4), memcpy(pe, t->pe.data(), n * 4);
  memcpy(dyn, t->dyn.data(), n), memcpy(ls, t->ls.data(), n * 4), memcpy(le, t->le.data(), n * 4);
}

void stw_trace_schedules(const stw_trace_file *t, int64_t *ph_start, int64_t *ph_end, int64_t *ly_start,
                         int64_t *ly_end) {
  for (int64_t k = 0; k < t->n_sched; k++) ph_start[k] = t->ph_start[k], ph_end[k] = t->ph_end[k];
  for (int64_t k = 0; k < t->n_known; k++) ly_start[k] = t->ly_start[k], ly_end[k] = t->ly_end[k];
}

const char *stw_trace_phase_tag(const stw_trace_file *t, int64_t k) { return t->tags[k].c_str(); }
const char *stw_trace_layer_name(const stw_trace_file *t, int64_t k) { return t->names[k].c_str(); }

int stw_trace_write(const stw_trace_cols *c, int32_t form, const char *path, stw_io_error *e) {
  if (e) e->kind = 0, e->line = 0, e->text[0] = 0;
  const int64_t horizon = c->n_sched ? c->ph_end[c->n_sched - 1] : 0;
  std::string o;
  if (form == 0) {  // raw: one op per timestamp slot (traceio.py:235-270)
    std::vector<std::pair<int64_t, int8_t>> slot(horizon, {-1, 0});  // (event, 0 alloc / 1 free)
    auto claim = [&](int64_t t, int64_t i, int8_t k) {
      if (t < 0) t += horizon;  // Python negative list index
      if (t < 0 || t >= horizon) return set_err(e, STW_IOE_INDEX, 0, "list index out of range"), false;
      if (slot[t].first >= 0)
        return set_err(e, STW_IOE_MSG, 0, "two ops share timestamp %lld; raw layout impossible", (long long)t), false;
      slot[t] = {i, k};
      return true;
    };
    for (int64_t i = 0; i < c->n; i++) {
      if (!claim(c->t_s[i], i, 0)) return STW_ETRACE;
      if (c->t_e[i] < horizon && !claim(c->t_e[i], i, 1)) return STW_ETRACE;
    }
    for (auto &x : slot)
      if (x.first < 0) return set_err(e, STW_IOE_MSG, 0, "trace is not record-dense; use the paired layout"), STW_ETRACE;
    o.reserve((size_t)horizon * 96 + 64);
    o += "{\"format\":\"raw\",\"kind\":\"trace\",\"version\":1}\n";
    for (auto &x : slot) {
      const int64_t i = x.first;
      const bool d = c->dyn[i];
      if (x.second == 0) {
        o += "{\"dynamic\":";
        o += d ? "true" : "false";
        o += ",\"id\":";
        jint(o, c->id[i]);
        o += ",\"module\":";
        jstr(o, d ? c->names[c->ls[i]] : "");
        o += ",\"op\":\"alloc\",\"phase\":";
        jstr(o, c->tags[c->ps[i]]);
        o += ",\"size\":";
        jint(o, c->size[i]);
        o += "}\n";
      } else {
        o += "{\"id\":";
        jint(o, c->id[i]);
        o += ",\"module\":";
        jstr(o, d ? c->names[c->le[i]] : "");
        o += ",\"op\":\"free\",\"phase\":";
        jstr(o, c->tags[c->pe[i]]);
        o += "}\n";
      }
    }
  } else {  // paired (traceio.py:272-291)
    o.reserve((size_t)c->n * 160 + 256);
    o += "{\"format\":\"paired\",\"kind\":\"trace\",\"layers\":[";
    for (int64_t k = 0; k < c->n_layers; k++) {
      if (k) o += ',';
      o += '[';
      jstr(o, c->names[k]);
      o += ',';
      jint(o, c->ly_start[k]);
      o += ',';
      jint(o, c->ly_end[k]);
      o += ']';
    }
    o += "],\"phases\":[";
    for (int64_t k = 0; k < c->n_sched; k++) {
      if (k) o += ',';
      o += '[';
      jstr(o, c->tags[k]);
      o += ',';
      jint(o, c->ph_start[k]);
      o += ',';
      jint(o, c->ph_end[k]);
      o += ']';
    }
    o += "],\"version\":1}\n";
    for (int64_t i = 0; i < c->n; i++) {
      const bool d = c->dyn[i];
      o += "{\"dynamic\":";
      o += d ? "true" : "false";
      o += ",\"id\":";
      jint(o, c->id[i]);
      o += ",\"l_e\":";
      if (d) jstr(o, c->names[c->le[i]]);
      else o += "null";
      o += ",\"l_s\":";
      if (d) jstr(o, c->names[c->ls[i]]);
      else o += "null";
      o += ",\"p_e\":";
      jstr(o, c->tags[c->pe[i]]);
      o += ",\"p_s\":";
      jstr(o, c->tags[c->ps[i]]);
      o += ",\"size\":";
      jint(o, c->size[i]);
      o += ",\"t_e\":";
      jint(o, c->t_e[i]);
      o += ",\"t_s\":";
      jint(o, c->t_s[i]);
      o += "}\n";
    }
  }
  return write_file(path, o, e) ? STW_OK : STW_ETRACE;
}

int stw_plan_write(const stw_plan_cols *p, const char *path, stw_io_error *e) {
  if (e) e->kind = 0, e->line = 0, e->text[0] = 0;
  std::string o;
  o.reserve((size_t)p->n_dec * 120 + 256);
  o += "{\n  \"alignment\": ";
  jint(o, p->alignment);
  o += ",\n  \"decisions\": [";
  for (int64_t i = 0; i < p->n_dec; i++) {
    o += i ? ",\n    {\n      \"addr\": " : "\n    {\n      \"addr\": ";
    jint(o, p->addr[i]);
    o += ",\n      \"id\": ";
    jint(o, p->id[i]);
    o += ",\n      \"size\": ";
    jint(o, p->size[i]);
    o += ",\n      \"t_e\": ";
    jint(o, p->t_e[i]);
    o += ",\n      \"t_s\": ";
    jint(o, p->t_s[i]);
    o += "\n    }";
  }
  o += p->n_dec ? "\n  ],\n  \"pool_size\": " : "],\n  \"pool_size\": ";
  jint(o, p->pool_size);
  o += ",\n  \"reuse_map\": [";
  std::vector<int64_t> keys(p->n_keys);
  for (int64_t k = 0; k < p->n_keys; k++) keys[k] = k;
  std::stable_sort(keys.begin(), keys.end(), [&](int64_t a, int64_t b) {
    const int c = strcmp(p->l_s[a], p->l_s[b]);
    return c != 0 ? c < 0 : strcmp(p->l_e[a], p->l_e[b]) < 0;
  });
  for (size_t j = 0; j < keys.size(); j++) {
    const int64_t k = keys[j];
    o += j ? ",\n    {\n      \"intervals\": [" : "\n    {\n      \"intervals\": [";
    const int64_t a = p->iv_off[k], b = p->iv_off[k + 1];
    for (int64_t x = a; x < b; x++) {
      o += x > a ? ",\n        [\n          " : "\n        [\n          ";
      jint(o, p->iv_lo[x]);
      o += ",\n          ";
      jint(o, p->iv_hi[x]);
      o += "\n        ]";
    }
    o += b > a ? "\n      ],\n      \"l_e\": " : "],\n      \"l_e\": ";
    jstr(o, p->l_e[k]);
    o += ",\n      \"l_s\": ";
    jstr(o, p->l_s[k]);
    o += "\n    }";
  }
  o += p->n_keys ? "\n  ],\n  \"version\": 1\n}\n" : "],\n  \"version\": 1\n}\n";
  return write_file(path, o, e) ? STW_OK : STW_EPLAN;
}

int stw_plan_read(const char *path, stw_plan_file **out, stw_io_error *e) {
  *out = nullptr;
  if (e) e->kind = 0, e->line = 0, e->text[0] = 0;
  std::string s;
  if (!read_file(path, &s, e)) return STW_EPLAN;
  Doc d;
  const int r = d.parse(s.data(), s.data() + s.size());
  if (r < 0) return set_err(e, STW_IOE_JSON, 0, "json"), STW_EPLAN;
  if (d.n[r].t != J_OBJ) return set_err(e, STW_IOE_PLANDOC, 0, "doc"), STW_EPLAN;
  const int vn = d.get(r, "version");
  const bool v1 = vn >= 0 && ((d.n[vn].t == J_INT && d.n[vn].i == 1) || d.n[vn].t == J_TRUE ||
                              (d.n[vn].t == J_FLT && d.n[vn].f == 1.0));
  if (!v1) return set_err(e, STW_IOE_HEADER, 0, "version"), STW_EPLAN;
  stw_plan_file *P = new stw_plan_file();
  auto fail = [&]() {
    delete P;
    set_err(e, STW_IOE_PLANDOC, 0, "doc");
    return STW_EPLAN;
  };
  if (d.bad) return fail();
  const int dn = d.get(r, "decisions");
  if (dn < 0 || d.n[dn].t != J_ARR) return fail();
  const size_t nd = (size_t)d.n[dn].i;
  P->id.reserve(nd), P->addr.reserve(nd), P->size.reserve(nd), P->t_s.reserve(nd), P->t_e.reserve(nd);
  for (int c = d.n[dn].first; c >= 0; c = d.n[c].next) {
    if (d.n[c].t != J_OBJ) return fail();
    int64_t v[5];
    const char *keys[5] = {"id", "addr", "size", "t_s", "t_e"};
    for (int k = 0; k < 5; k++) {
      const int x = d.get(c, keys[k]);
      if (x < 0 || !py_int(d, x, &v[k])) return fail();
    }
    P->id.push_back(v[0]), P->addr.push_back(v[1]), P->size.push_back(v[2]), P->t_s.push_back(v[3]),
        P->t_e.push_back(v[4]);
  }
  const int rn = d.get(r, "reuse_map");
  std::map<std::pair<std::string, std::string>, size_t> seen;  // duplicate keys: the last entry wins
  std::vector<std::vector<std::pair<int64_t, int64_t>>> ivs;
  if (rn >= 0) {
    if (d.n[rn].t != J_ARR) return fail();
    for (int c = d.n[rn].first; c >= 0; c = d.n[c].next) {
      if (d.n[c].t != J_OBJ) return fail();
      const int a = d.get(c, "l_s"), b = d.get(c, "l_e"), in = d.get(c, "intervals");
      std::string ls, le;
      if (a < 0 || b < 0 || in < 0 || !py_str(d, a, &ls) || !py_str(d, b, &le) || d.n[in].t != J_ARR) return fail();
      std::vector<std::pair<int64_t, int64_t>> list;
      for (int x = d.n[in].first; x >= 0; x = d.n[x].next) {
        int64_t lo, hi;
        const int y = d.n[x].first;
        if (d.n[x].t != J_ARR || d.n[x].i != 2 || !py_int(d, y, &lo) || !py_int(d, d.n[y].next, &hi) || hi <= lo)
          return fail();
        list.push_back({lo, hi});
      }
      auto key = std::make_pair(ls, le);
      auto it = seen.find(key);
      if (it != seen.end()) {
        ivs[it->second] = std::move(list);
      } else {
        seen[key] = ivs.size();
        P->ls.push_back(ls);
        P->le.push_back(le);
        ivs.push_back(std::move(list));
      }
    }
  }
  const int pn = d.get(r, "pool_size"), an = d.get(r, "alignment");
  if (pn < 0 || !py_int(d, pn, &P->pool_size)) return fail();
  if (an >= 0 && !py_int(d, an, &P->alignment)) return fail();
  for (auto &l : ivs) {
    for (auto &iv : l) P->iv_lo.push_back(iv.first), P->iv_hi.push_back(iv.second);
    P->iv_off.push_back((int64_t)P->iv_lo.size());
  }
  // PlanBundle.validate (traceio.py:322-331); interval sets are normalised by
  // the caller, so the reuse bounds are checked there
  for (size_t i = 0; i < P->id.size(); i++) {
    if (P->addr[i] < 0 || P->addr[i] + P->size[i] > P->pool_size) {
      set_err(e, STW_IOE_MSG, 0, "decision %lld out of pool", (long long)P->id[i]);
      delete P;
      return STW_EPLAN;
    }
    if (P->alignment == 0 || P->addr[i] % P->alignment) {
      set_err(e, P->alignment == 0 ? STW_IOE_PLANDOC : STW_IOE_MSG, 0, "decision %lld misaligned address %lld",
              (long long)P->id[i], (long long)P->addr[i]);
      delete P;
      return STW_EPLAN;
    }
  }
  *out = P;
  return STW_OK;
}

void stw_plan_free(stw_plan_file *p) { delete p; }

void stw_plan_sizes(const stw_plan_file *p, int64_t *z) {
  z[0] = p->pool_size;
  z[1] = p->alignment;
  z[2] = (int64_t)p->id.size();
  z[3] = (int64_t)p->ls.size();
  z[4] = (int64_t)p->iv_lo.size();
}

void stw_plan_decisions(const stw_plan_file *p, int64_t *id, int64_t *addr, int64_t *size, int64_t *t_s,
                        int64_t *t_e) {
  const size_t n = p->id.size();
  if (!n) return;
  memcpy(id, p->id.data(), n * 8), memcpy(addr, p->addr.data(), n * 8), memcpy(size, p->size.data(), n * 8);
  memcpy(t_s, p->t_s.data(), n * 8), memcpy(t_e, p->t_e.data(), n * 8);
}

void stw_plan_reuse(const stw_plan_file *p, int64_t *iv_off, int64_t *iv_lo, int64_t *iv_hi) {
  for (size_t k = 0; k < p->iv_off.size(); k++) iv_off[k] = p->iv_off[k];
  for (size_t k = 0; k < p->iv_lo.size(); k++) iv_lo[k] = p->iv_lo[k], iv_hi[k] = p->iv_hi[k];
}

const char *stw_plan_key(const stw_plan_file *p, int64_t k, int32_t which) {
  return which ? p->le[k].c_str() : p->ls[k].c_str();
}

}  // extern "C"
