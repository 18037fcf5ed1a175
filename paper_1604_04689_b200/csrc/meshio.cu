// meshio.cu — native OFF / OBJ ingestion into the polygon (CSR) connectivity form (host code;
// SURVEY.md §8(f) row 3 "OFF/OBJ ingestion"; SPEC.md mesh-io load_off / load_obj).
//
// The parsers read the whole file image from memory in one forward pass (no per-line allocation),
// keep the vertex coordinates out (topology only, "stored opaquely"), and produce
//   off[M+1] int64, idx[off[M]] int32 (0-based), num_nodes = vertex count,
// the input of mn_find_poly_neighbors (or, when every face has 3 / 4 nodes, a TRI3 / QUAD4 conn).
// Rules (R19):
//   * "#" starts a comment line; blank lines are skipped; tokens are separated by runs of spaces /
//     tabs; "\r\n" line ends are accepted.
//   * OFF: optional "OFF" line (counts may follow on it), counts "V F [E]" (E read and ignored), V
//     vertex lines (>= 3 numeric tokens), F face lines "k i0 .. i(k-1)" (extra tokens, e.g. colours,
//     ignored).  Missing lines -> MN_ERR_COUNT_MISMATCH; non-comment content after the faces ->
//     MN_ERR_COUNT_MISMATCH.
//   * OBJ: "v" (>= 3 numeric tokens) and "f" records, other records ignored; face tokens
//     "i", "i/t", "i//n", "i/t/n" keep i; i > 0 is 1-based, i < 0 is relative to the vertex count
//     at that line (-1 = last vertex), i == 0 -> MN_ERR_ZERO_INDEX.
//   * Malformed tokens -> MN_ERR_SYNTAX.  Error detail: elem = 1-based line number, pos = token
//     position in the line (0-based; -1 when not token-specific).
//   * The result is validated like every input of the library (R18 order: arity >= 3, index range,
//     repeated node), detail = (face index, position).
#include <algorithm>
#include <cerrno>
#include <new>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "meshnbr.h"

namespace {

struct Cursor {
  const char* p;
  const char* end;
  int64_t line = 0;   // 1-based number of the line last returned
};

// Next line that is not blank and not a comment; [b, e) excludes the line end.  false at EOF.
bool next_line(Cursor& c, const char*& b, const char*& e) {
  while (c.p < c.end) {
    const char* s = c.p;
    const char* nl = static_cast<const char*>(std::memchr(s, '\n', (size_t)(c.end - s)));
    const char* le = nl ? nl : c.end;
    c.p = nl ? nl + 1 : c.end;
    ++c.line;
    const char* t = le;
    if (t > s && t[-1] == '\r') --t;
    while (s < t && (*s == ' ' || *s == '\t')) ++s;
    if (s == t || *s == '#') continue;
    b = s;
    e = t;
    return true;
  }
  return false;
}

// Tokeniser over one line.
struct Tokens {
  const char* p;
  const char* e;
  bool next(const char*& tb, const char*& te) {
    while (p < e && (*p == ' ' || *p == '\t')) ++p;
    if (p >= e) return false;
    tb = p;
    while (p < e && *p != ' ' && *p != '\t') ++p;
    te = p;
    return true;
  }
};

bool parse_i64(const char* b, const char* e, int64_t& v) {
  if (b >= e) return false;
  bool neg = false;
  const char* p = b;
  if (*p == '+' || *p == '-') { neg = *p == '-'; ++p; }
  if (p >= e) return false;
  int64_t x = 0;
  for (; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    if (x > (INT64_MAX - 9) / 10) return false;
    x = x * 10 + (*p - '0');
  }
  v = neg ? -x : x;
  return true;
}

bool is_number(const char* b, const char* e) {
  if (b >= e || e - b > 63) return false;
  char buf[64];
  std::memcpy(buf, b, (size_t)(e - b));
  buf[e - b] = 0;
  char* q = nullptr;
  errno = 0;
  std::strtod(buf, &q);
  return q == buf + (e - b);
}

mn_status fail(mn_error_detail* err, mn_status st, int64_t elem, int32_t pos) {
  if (err) { err->elem = elem; err->pos = pos; }
  return st;
}

// R18 validation of the parsed faces.
mn_status validate(const std::vector<int64_t>& off, const std::vector<int32_t>& idx, int64_t N,
                   mn_error_detail* err) {
  const int64_t M = (int64_t)off.size() - 1;
  for (int64_t f = 0; f < M; ++f) {
    const int64_t b = off[f], k = off[f + 1] - b;
    if (k < 3) return fail(err, MN_ERR_ARITY, f, -1);
    for (int64_t p = 0; p < k; ++p)
      if (idx[b + p] < 0 || idx[b + p] >= N) return fail(err, MN_ERR_INDEX_OUT_OF_RANGE, f, (int32_t)p);
    for (int64_t p = 1; p < k; ++p)
      for (int64_t q = 0; q < p; ++q)
        if (idx[b + q] == idx[b + p]) return fail(err, MN_ERR_DEGENERATE, f, (int32_t)p);
  }
  return MN_OK;
}

mn_status finish(std::vector<int64_t>& off, std::vector<int32_t>& idx, int64_t N, mn_host_mesh* out,
                 mn_error_detail* err) {
  mn_status st = validate(off, idx, N, err);
  if (st != MN_OK) return st;
  const int64_t M = (int64_t)off.size() - 1;
  int32_t uni = 0;
  for (int64_t f = 0; f < M; ++f) {
    const int32_t k = (int32_t)(off[f + 1] - off[f]);
    if (f == 0) uni = k;
    else if (k != uni) { uni = 0; break; }
  }
  out->off = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * off.size()));
  out->idx = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (idx.empty() ? 1 : idx.size())));
  if (!out->off || !out->idx) {
    std::free(out->off);
    std::free(out->idx);
    out->off = nullptr;
    out->idx = nullptr;
    return MN_ERR_OOM;
  }
  std::memcpy(out->off, off.data(), sizeof(int64_t) * off.size());
  if (!idx.empty()) std::memcpy(out->idx, idx.data(), sizeof(int32_t) * idx.size());
  out->num_nodes = N;
  out->num_elems = M;
  out->conn_len = (int64_t)idx.size();
  out->uniform_arity = uni;
  return MN_OK;
}

mn_status parse_off(const char* bytes, size_t len, mn_host_mesh* out, mn_error_detail* err) {
  if (err) { err->elem = -1; err->pos = -1; }
  if (!out || (len && !bytes)) return MN_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof(*out));
  Cursor c{bytes, bytes + len};
  const char *b, *e, *tb, *te;
  if (!next_line(c, b, e)) return fail(err, MN_ERR_COUNT_MISMATCH, c.line, -1);
  Tokens tk{b, e};
  tk.next(tb, te);
  int64_t cnt[3] = {0, 0, 0};
  int nc = 0, pos = 0;
  if (te - tb == 3 && std::memcmp(tb, "OFF", 3) == 0) {   // header; counts may follow on the same line
    ++pos;
    if (!tk.next(tb, te)) {
      if (!next_line(c, b, e)) return fail(err, MN_ERR_COUNT_MISMATCH, c.line, -1);
      tk = Tokens{b, e};
      pos = 0;
      tk.next(tb, te);
    }
  }
  for (;;) {   // counts "V F [E]"
    if (nc == 3) break;
    if (!parse_i64(tb, te, cnt[nc]) || cnt[nc] < 0) return fail(err, MN_ERR_SYNTAX, c.line, pos);
    ++nc;
    ++pos;
    if (!tk.next(tb, te)) break;
  }
  if (nc < 2) return fail(err, MN_ERR_SYNTAX, c.line, -1);
  const int64_t V = cnt[0], F = cnt[1];
  if (V > INT32_MAX || F > INT32_MAX) return fail(err, MN_ERR_CAPACITY, c.line, -1);
  for (int64_t v = 0; v < V; ++v) {
    if (!next_line(c, b, e)) return fail(err, MN_ERR_COUNT_MISMATCH, c.line, -1);
    Tokens t{b, e};
    for (int q = 0; q < 3; ++q)
      if (!t.next(tb, te) || !is_number(tb, te)) return fail(err, MN_ERR_SYNTAX, c.line, q);
  }
  std::vector<int64_t> off;
  std::vector<int32_t> idx;
  // the face count is untrusted: every face line takes at least 2 bytes, so never reserve more
  off.reserve((size_t)std::min<int64_t>(F, (int64_t)(c.end - c.p) / 2) + 1);
  off.push_back(0);
  for (int64_t f = 0; f < F; ++f) {
    if (!next_line(c, b, e)) return fail(err, MN_ERR_COUNT_MISMATCH, c.line, -1);
    Tokens t{b, e};
    int64_t k = 0;
    if (!t.next(tb, te) || !parse_i64(tb, te, k) || k < 0) return fail(err, MN_ERR_SYNTAX, c.line, 0);
    for (int64_t q = 0; q < k; ++q) {
      int64_t x = 0;
      if (!t.next(tb, te) || !parse_i64(tb, te, x)) return fail(err, MN_ERR_SYNTAX, c.line, (int32_t)(q + 1));
      if (x < INT32_MIN || x > INT32_MAX) x = -1;   // out of range either way
      idx.push_back((int32_t)x);
    }
    off.push_back((int64_t)idx.size());
  }
  if (next_line(c, b, e)) return fail(err, MN_ERR_COUNT_MISMATCH, c.line, -1);
  return finish(off, idx, V, out, err);
}

mn_status parse_obj(const char* bytes, size_t len, mn_host_mesh* out, mn_error_detail* err) {
  if (err) { err->elem = -1; err->pos = -1; }
  if (!out || (len && !bytes)) return MN_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof(*out));
  Cursor c{bytes, bytes + len};
  const char *b, *e, *tb, *te;
  int64_t nv = 0;
  std::vector<int64_t> off;
  std::vector<int32_t> idx;
  off.push_back(0);
  while (next_line(c, b, e)) {
    Tokens t{b, e};
    t.next(tb, te);
    const size_t n = (size_t)(te - tb);
    if (n == 1 && *tb == 'v') {
      for (int q = 1; q <= 3; ++q)
        if (!t.next(tb, te) || !is_number(tb, te)) return fail(err, MN_ERR_SYNTAX, c.line, q);
      if (++nv > INT32_MAX) return fail(err, MN_ERR_CAPACITY, c.line, -1);
    } else if (n == 1 && *tb == 'f') {
      int q = 1;
      while (t.next(tb, te)) {
        const char* slash = static_cast<const char*>(std::memchr(tb, '/', (size_t)(te - tb)));
        int64_t x = 0;
        if (!parse_i64(tb, slash ? slash : te, x)) return fail(err, MN_ERR_SYNTAX, c.line, q);
        if (x == 0) return fail(err, MN_ERR_ZERO_INDEX, c.line, q);
        const int64_t v = x > 0 ? x - 1 : nv + x;
        idx.push_back(v < INT32_MIN || v > INT32_MAX ? -1 : (int32_t)v);
        ++q;
      }
      off.push_back((int64_t)idx.size());
    }
    // every other record type (vt, vn, vp, o, g, s, usemtl, mtllib, l, p, ...) is ignored
  }
  return finish(off, idx, nv, out, err);
}

}  // namespace

extern "C" {

// No C++ exception crosses the C ABI: an allocation failure while parsing is MN_ERR_OOM.
mn_status mn_parse_off(const char* bytes, size_t len, mn_host_mesh* out, mn_error_detail* err) {
  try {
    return parse_off(bytes, len, out, err);
  } catch (const std::bad_alloc&) {
    if (out) mn_host_mesh_free(out);
    return MN_ERR_OOM;
  } catch (...) {
    if (out) mn_host_mesh_free(out);
    return MN_ERR_INVALID_ARG;
  }
}

mn_status mn_parse_obj(const char* bytes, size_t len, mn_host_mesh* out, mn_error_detail* err) {
  try {
    return parse_obj(bytes, len, out, err);
  } catch (const std::bad_alloc&) {
    if (out) mn_host_mesh_free(out);
    return MN_ERR_OOM;
  } catch (...) {
    if (out) mn_host_mesh_free(out);
    return MN_ERR_INVALID_ARG;
  }
}

void mn_host_mesh_free(mn_host_mesh* m) {
  if (!m) return;
  std::free(m->off);
  std::free(m->idx);
  std::memset(m, 0, sizeof(*m));
}

}  // extern "C"
