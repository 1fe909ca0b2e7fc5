// reader.cpp — native JSONL / CSV trace reader (host, C++17, threads).
//
// Replaces the per-line Python decoding of trace.py:87-151 (_parse_jsonl,
// _parse_csv, _event_from_fields) for the records that matter at scale:
// the canonical forms serialize_trace writes.  A line is decoded natively
// when it is a plain record (JSON object with exactly the five keys, integer
// literals, unescaped strings; CSV rows of five unquoted fields with decimal
// integers).  Anything else is not guessed at: its line number is handed back
// and the caller decodes exactly those lines with the reference semantics
// (json.loads / csv + _event_from_fields), so MalformedRecord line numbers
// and reasons stay identical.  Files whose line structure Python would see
// differently (str.splitlines separators other than \n / \r\n, CSV quoting)
// are refused whole (MP_E_UNSUPPORTED) and parsed by the Python path.
//
// Variable names are interned to dense ids in lexicographic (UTF-8 byte =
// code point) order, the id convention of the device library.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/memplan_b200.h"

namespace {

struct Rec {
  int64_t index, t_us, size;
  uint8_t kind;
  std::string_view var;
};

struct Chunk {
  std::vector<Rec> recs;
  std::vector<int64_t> rec_line;   // 1-based line of each record
  std::vector<int64_t> slow_lines; // lines for the reference decoder
  std::vector<int32_t> local;      // record -> chunk-local name id
  std::vector<std::string_view> uniq;  // chunk-local names, sorted after interning
  std::vector<int32_t> remap;      // chunk-local id -> global id
};

// chunk-local interning: names in first-seen order, then sorted, with the
// records' ids rewritten to sorted order
void intern_local(Chunk &C) {
  std::unordered_map<std::string_view, int32_t> m;
  m.reserve(C.recs.size() / 2 + 16);
  C.local.resize(C.recs.size());
  for (size_t i = 0; i < C.recs.size(); i++) {
    auto it = m.emplace(C.recs[i].var, (int32_t)C.uniq.size());
    if (it.second) C.uniq.push_back(C.recs[i].var);
    C.local[i] = it.first->second;
  }
  std::vector<int32_t> ord(C.uniq.size());
  for (size_t i = 0; i < ord.size(); i++) ord[i] = (int32_t)i;
  std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return C.uniq[(size_t)a] < C.uniq[(size_t)b]; });
  std::vector<int32_t> pos(ord.size());
  std::vector<std::string_view> su(ord.size());
  for (size_t r = 0; r < ord.size(); r++) { pos[(size_t)ord[r]] = (int32_t)r; su[r] = C.uniq[(size_t)ord[r]]; }
  C.uniq.swap(su);
  for (auto &x : C.local) x = pos[(size_t)x];
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; }

// -?(0|[1-9][0-9]*) exactly, no overflow; JSON integer literal
bool parse_json_int(const char *&p, const char *e, int64_t &out) {
  bool neg = false;
  if (p < e && *p == '-') { neg = true; p++; }
  if (p >= e || *p < '0' || *p > '9') return false;
  if (*p == '0' && p + 1 < e && p[1] >= '0' && p[1] <= '9') return false;
  unsigned long long v = 0;
  int nd = 0;
  while (p < e && *p >= '0' && *p <= '9') {
    if (++nd > 18) return false;  // leave big numbers to Python
    v = v * 10 + (unsigned)(*p - '0');
    p++;
  }
  if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) return false;  // a float: int() truncation
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

// a JSON string without escapes or control characters
bool parse_json_str(const char *&p, const char *e, std::string_view &out) {
  if (p >= e || *p != '"') return false;
  const char *s = ++p;
  while (p < e && *p != '"') {
    unsigned char c = (unsigned char)*p;
    if (c == '\\' || c < 0x20) return false;
    p++;
  }
  if (p >= e) return false;
  out = std::string_view(s, (size_t)(p - s));
  p++;
  return true;
}

int kind_code(std::string_view k) {
  if (k == "malloc") return MP_MALLOC;
  if (k == "free") return MP_FREE;
  if (k == "read") return MP_READ;
  if (k == "write") return MP_WRITE;
  return -1;
}

// {"index":..,"t_us":..,"kind":"..","var":"..","size":..} in any key order
bool fast_jsonl(const char *p, const char *e, Rec &r) {
  while (p < e && is_ws(*p)) p++;
  if (p >= e || *p != '{') return false;
  p++;
  int seen = 0;
  for (int f = 0; f < 5; f++) {
    while (p < e && is_ws(*p)) p++;
    std::string_view key;
    if (!parse_json_str(p, e, key)) return false;
    while (p < e && is_ws(*p)) p++;
    if (p >= e || *p != ':') return false;
    p++;
    while (p < e && is_ws(*p)) p++;
    int bit;
    if (key == "index") { bit = 1; if (!parse_json_int(p, e, r.index)) return false; }
    else if (key == "t_us") { bit = 2; if (!parse_json_int(p, e, r.t_us)) return false; }
    else if (key == "size") { bit = 4; if (!parse_json_int(p, e, r.size)) return false; }
    else if (key == "kind") {
      bit = 8;
      std::string_view k;
      if (!parse_json_str(p, e, k)) return false;
      int c = kind_code(k);
      if (c < 0) return false;
      r.kind = (uint8_t)c;
    } else if (key == "var") {
      bit = 16;
      if (!parse_json_str(p, e, r.var) || r.var.empty()) return false;
    } else {
      return false;
    }
    if (seen & bit) return false;  // duplicate key: json.loads keeps the last
    seen |= bit;
    while (p < e && is_ws(*p)) p++;
    if (f < 4) {
      if (p >= e || *p != ',') return false;
      p++;
    }
  }
  if (p >= e || *p != '}') return false;
  p++;
  while (p < e && is_ws(*p)) p++;
  return p == e && seen == 31;
}

// [0-9]+ with an optional leading '-', as int() of a CSV field reads it
bool parse_csv_int(std::string_view f, int64_t &out) {
  size_t i = 0;
  bool neg = false;
  if (i < f.size() && f[i] == '-') { neg = true; i++; }
  if (i >= f.size() || f.size() - i > 18) return false;
  unsigned long long v = 0;
  for (; i < f.size(); i++) {
    if (f[i] < '0' || f[i] > '9') return false;
    v = v * 10 + (unsigned)(f[i] - '0');
  }
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

bool fast_csv(const char *p, const char *e, Rec &r) {
  std::string_view f[5];
  int nf = 0;
  const char *s = p;
  for (const char *q = p;; q++) {
    if (q == e || *q == ',') {
      if (nf == 5) return false;
      f[nf++] = std::string_view(s, (size_t)(q - s));
      if (q == e) break;
      s = q + 1;
    }
  }
  if (nf != 5) return false;
  if (!parse_csv_int(f[0], r.index) || !parse_csv_int(f[1], r.t_us) || !parse_csv_int(f[4], r.size)) return false;
  int c = kind_code(f[2]);
  if (c < 0 || f[3].empty()) return false;
  r.kind = (uint8_t)c;
  r.var = f[3];
  return true;
}

// line-structure bytes Python's str.splitlines treats as separators, other
// than \n and \r\n: \v \f \x1c \x1d \x1e, a lone \r, U+0085, U+2028/2029
bool has_foreign_breaks(const char *d, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    unsigned char c = (unsigned char)d[i];
    if (c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) return true;
    if (c == '\r' && (i + 1 >= n || d[i + 1] != '\n')) return true;
    if (c == 0xc2 && i + 1 < n && (unsigned char)d[i + 1] == 0x85) return true;
    if (c == 0xe2 && i + 2 < n && (unsigned char)d[i + 1] == 0x80 &&
        ((unsigned char)d[i + 2] == 0xa8 || (unsigned char)d[i + 2] == 0xa9))
      return true;
  }
  return false;
}

bool blank(const char *p, const char *e) {
  // str.strip() whitespace subset that can occur here
  for (; p < e; p++)
    if (!(*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) return false;
  return true;
}

}  // namespace

struct mp_reader {
  int64_t n = 0;
  std::vector<uint8_t> kind;
  std::vector<int32_t> var;
  std::vector<int64_t> size, t_us, index, line;
  std::vector<std::string> names;
  std::vector<int64_t> slow_lines;
  std::string data;  // owned copy: records point into it
};

extern "C" int mp_read_trace(const char *data, int64_t nbytes, int32_t format, int32_t threads, mp_reader **out,
                             mp_err *err) {
  if (format != 0 && format != 1) {
    if (err) { memset(err, 0, sizeof *err); err->code = MP_E_VALUE; }
    return MP_E_VALUE;
  }
  if (has_foreign_breaks(data, nbytes) || (format == 1 && memchr(data, '"', (size_t)nbytes))) {
    if (err) { memset(err, 0, sizeof *err); err->code = MP_E_UNSUPPORTED; }
    return MP_E_UNSUPPORTED;
  }
  const bool timing = getenv("MP_READER_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t_start = now();
  auto lap = [&](const char *what) {
    if (timing) fprintf(stderr, "reader %-10s %8.3f s\n", what, std::chrono::duration<double>(now() - t_start).count());
  };
  mp_reader *R = new mp_reader();
  R->data.assign(data, (size_t)nbytes);
  lap("copy");
  const char *d = R->data.data();
  // line starts (\n-terminated; a final line without \n counts)
  std::vector<int64_t> starts;
  starts.reserve((size_t)(nbytes / 64 + 2));
  starts.push_back(0);
  for (int64_t i = 0; i < nbytes; i++)
    if (d[i] == '\n' && i + 1 < nbytes) starts.push_back(i + 1);
  int64_t nlines = nbytes ? (int64_t)starts.size() : 0;
  lap("lines");
  auto line_end = [&](int64_t l) -> int64_t {  // exclusive, without the \r\n / \n
    int64_t e = l + 1 < nlines ? starts[(size_t)l + 1] - 1 : nbytes;
    if (e > starts[(size_t)l] && d[e - 1] == '\n') e--;
    if (e > starts[(size_t)l] && d[e - 1] == '\r') e--;
    return e;
  };
  int64_t first = 0;
  if (format == 1) {
    // header: the caller re-checks it with the reference code when this fails
    if (nlines == 0) { delete R; if (err) { memset(err, 0, sizeof *err); err->code = MP_E_UNSUPPORTED; } return MP_E_UNSUPPORTED; }
    std::string_view h(d, (size_t)line_end(0));
    if (h != "index,t_us,kind,var,size") { delete R; if (err) { memset(err, 0, sizeof *err); err->code = MP_E_UNSUPPORTED; } return MP_E_UNSUPPORTED; }
    first = 1;
  }
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  if (nlines - first < 65536) T = 1;
  std::vector<Chunk> ch((size_t)T);
  auto work = [&](int c) {
    int64_t lo = first + (nlines - first) * c / T, hi = first + (nlines - first) * (c + 1) / T;
    Chunk &C = ch[(size_t)c];
    C.recs.reserve((size_t)(hi - lo));
    for (int64_t l = lo; l < hi; l++) {
      const char *p = d + starts[(size_t)l], *e = d + line_end(l);
      // skipped lines: JSONL `not line.strip()`, CSV empty rows
      if (format == 0 ? blank(p, e) : p == e) continue;
      Rec r;
      bool ok = format == 0 ? fast_jsonl(p, e, r) : fast_csv(p, e, r);
      if (ok) {
        C.recs.push_back(r);
        C.rec_line.push_back(l + 1);
      } else {
        C.slow_lines.push_back(l + 1);
      }
    }
  };
  auto run = [&](auto fn) {
    if (T == 1) { fn(0); return; }
    std::vector<std::thread> th;
    for (int c = 0; c < T; c++) th.emplace_back(fn, c);
    for (auto &x : th) x.join();
  };
  run([&](int c) { work(c); intern_local(ch[(size_t)c]); });
  lap("parse");
  // global names: k-way merge of the sorted chunk-local lists, deduplicated
  std::vector<std::string_view> uniq;
  {
    size_t tot = 0;
    for (auto &C : ch) tot += C.uniq.size();
    uniq.reserve(tot);
    std::vector<size_t> at((size_t)T, 0);
    for (;;) {
      int best = -1;
      for (int c = 0; c < T; c++)
        if (at[(size_t)c] < ch[(size_t)c].uniq.size() &&
            (best < 0 || ch[(size_t)c].uniq[at[(size_t)c]] < ch[(size_t)best].uniq[at[(size_t)best]]))
          best = c;
      if (best < 0) break;
      std::string_view v = ch[(size_t)best].uniq[at[(size_t)best]];
      if (uniq.empty() || uniq.back() != v) uniq.push_back(v);
      for (int c = 0; c < T; c++)
        if (at[(size_t)c] < ch[(size_t)c].uniq.size() && ch[(size_t)c].uniq[at[(size_t)c]] == v) at[(size_t)c]++;
    }
  }
  lap("merge");
  int64_t n = 0;
  std::vector<int64_t> base((size_t)T + 1, 0);
  for (int c = 0; c < T; c++) base[(size_t)c + 1] = base[(size_t)c] + (int64_t)ch[(size_t)c].recs.size();
  n = base[(size_t)T];
  R->n = n;
  R->kind.resize((size_t)n); R->var.resize((size_t)n); R->size.resize((size_t)n);
  R->t_us.resize((size_t)n); R->index.resize((size_t)n); R->line.resize((size_t)n);
  run([&](int c) {
    Chunk &C = ch[(size_t)c];
    // both lists sorted: one forward walk maps local ids to global ones
    C.remap.resize(C.uniq.size());
    size_t g = (size_t)(std::lower_bound(uniq.begin(), uniq.end(), C.uniq.empty() ? std::string_view() : C.uniq[0]) - uniq.begin());
    for (size_t i = 0; i < C.uniq.size(); i++) {
      while (uniq[g] != C.uniq[i]) g++;
      C.remap[i] = (int32_t)g;
    }
    int64_t o = base[(size_t)c];
    for (size_t i = 0; i < C.recs.size(); i++, o++) {
      const Rec &r = C.recs[i];
      R->kind[(size_t)o] = r.kind;
      R->var[(size_t)o] = C.remap[(size_t)C.local[i]];
      R->size[(size_t)o] = r.size;
      R->t_us[(size_t)o] = r.t_us;
      R->index[(size_t)o] = r.index;
      R->line[(size_t)o] = C.rec_line[i];
    }
  });
  for (auto &C : ch) R->slow_lines.insert(R->slow_lines.end(), C.slow_lines.begin(), C.slow_lines.end());
  lap("ids");
  R->names.reserve(uniq.size());
  for (auto &u : uniq) R->names.emplace_back(u);
  lap("names");
  *out = R;
  return MP_OK;
}

extern "C" int mp_reader_dims(mp_reader *R, int64_t *n, int64_t *nvars, int64_t *name_bytes, int64_t *nslow) {
  *n = R->n;
  *nvars = (int64_t)R->names.size();
  int64_t b = 0;
  for (auto &s : R->names) b += (int64_t)s.size();
  *name_bytes = b;
  *nslow = (int64_t)R->slow_lines.size();
  return MP_OK;
}

extern "C" int mp_reader_copy(mp_reader *R, uint8_t *kind, int32_t *var, int64_t *size, int64_t *t_us,
                              int64_t *index, int64_t *line, uint8_t *name_blob, int64_t *name_off,
                              int64_t *slow_lines) {
  size_t n = (size_t)R->n;
  if (n) {
    memcpy(kind, R->kind.data(), n);
    memcpy(var, R->var.data(), n * 4);
    memcpy(size, R->size.data(), n * 8);
    memcpy(t_us, R->t_us.data(), n * 8);
    memcpy(index, R->index.data(), n * 8);
    memcpy(line, R->line.data(), n * 8);
  }
  int64_t o = 0;
  name_off[0] = 0;
  for (size_t i = 0; i < R->names.size(); i++) {
    memcpy(name_blob + o, R->names[i].data(), R->names[i].size());
    o += (int64_t)R->names[i].size();
    name_off[i + 1] = o;
  }
  if (!R->slow_lines.empty()) memcpy(slow_lines, R->slow_lines.data(), R->slow_lines.size() * 8);
  return MP_OK;
}

extern "C" int mp_reader_free(mp_reader *R) {
  delete R;
  return MP_OK;
}
