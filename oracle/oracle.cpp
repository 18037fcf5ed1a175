// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously correct CPU implementation of what the CUDA path computes: the
// paper's serial baseline (§1 "loop over all elements in a mesh to identify
// (1) which pair of nodes is connected by an edge and (2) which nodes are contained in an
// element"; §3.2.2 "a STL container ... to dynamically store the indices of
// neighboring nodes for each vertex"), with a std::set per node as north_star asks, flattened
// to CSR.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
// load this library.  It shares no code, header, table or helper with paper_1604_04689_b200/:
// the edge tables below are written out here independently from the paper's definitions.
//
// Readings of the paper (DESIGN.md §"Readings"): duplicate pairs are collapsed (a one-ring is a
// set), lists are ascending, invalid input is rejected reporting the lowest element id, then
// the lowest position, range errors before repeated-node errors within an element.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <set>
#include <thread>
#include <vector>

namespace {

// Element edge tables (§2.1.1: "any pair of neighboring nodes is connected
// using an edge"; the paper spells out triangles only, §2.2; the other element types
// follow DESIGN.md reading R4: quad ring, all 6 tet edges, VTK hexahedron's 12 edges).
struct EdgeTable { int arity; int nedges; int a[12]; int b[12]; };

const EdgeTable kTables[4] = {
    // TRI3: three edges of the triangle (§2.2.1)
    {3, 3, {0, 1, 2}, {1, 2, 0}},
    // QUAD4: the 4 ring edges, no diagonals
    {4, 4, {0, 1, 2, 3}, {1, 2, 3, 0}},
    // TET4: every pair of the 4 nodes
    {4, 6, {0, 0, 0, 1, 1, 2}, {1, 2, 3, 2, 3, 3}},
    // HEX8 (VTK order: 0-3 bottom ring, 4-7 top ring, node 4 above node 0)
    {8, 12, {0, 1, 2, 3, 4, 5, 6, 7, 0, 1, 2, 3}, {1, 2, 3, 0, 5, 6, 7, 4, 4, 5, 6, 7}},
};

enum { OK = 0, ERR_ARG = 1, ERR_RANGE = 2, ERR_DEGENERATE = 3 };

// Validation in ascending element order; the first offending element decides.
int validate(int etype, const int32_t* conn, int64_t M, int64_t N, int64_t* eelem, int32_t* epos) {
  const int k = kTables[etype].arity;
  for (int64_t e = 0; e < M; ++e) {
    const int32_t* row = conn + e * k;
    for (int p = 0; p < k; ++p) {
      if (row[p] < 0 || (int64_t)row[p] >= N) { *eelem = e; *epos = p; return ERR_RANGE; }
    }
    for (int p = 1; p < k; ++p) {
      for (int q = 0; q < p; ++q) {
        if (row[q] == row[p]) { *eelem = e; *epos = p; return ERR_DEGENERATE; }
      }
    }
  }
  return OK;
}

template <class Container>
void flatten(const std::vector<Container>& lists, int64_t N, int64_t** offsets, int32_t** indices,
             int64_t* nnz) {
  int64_t* off = (int64_t*)std::malloc(sizeof(int64_t) * (size_t)(N + 1));
  off[0] = 0;
  for (int64_t v = 0; v < N; ++v) off[v + 1] = off[v] + (int64_t)lists[v].size();
  int32_t* idx = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)(off[N] > 0 ? off[N] : 1));
  int64_t pos = 0;
  for (int64_t v = 0; v < N; ++v)
    for (int32_t x : lists[v]) idx[pos++] = x;
  *offsets = off;
  *indices = idx;
  *nnz = off[N];
}

}  // namespace

extern "C" {

int oracle_validate(int etype, const int32_t* conn, int64_t M, int64_t N, int64_t* err_elem,
                    int32_t* err_pos) {
  if (etype < 0 || etype > 3 || M < 0 || N < 0) return ERR_ARG;
  *err_elem = -1;
  *err_pos = -1;
  return validate(etype, conn, M, N, err_elem, err_pos);
}

// Node mode: adj(v) = { u != v : some element has an edge {u, v} }, ascending.
int oracle_node_csr(int etype, const int32_t* conn, int64_t M, int64_t N, int64_t** offsets,
                    int32_t** indices, int64_t* nnz, int64_t* err_elem, int32_t* err_pos) {
  int rc = oracle_validate(etype, conn, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  const EdgeTable& t = kTables[etype];
  std::vector<std::set<int32_t>> S((size_t)N);
  for (int64_t e = 0; e < M; ++e) {
    const int32_t* row = conn + e * t.arity;
    for (int j = 0; j < t.nedges; ++j) {
      int32_t a = row[t.a[j]], b = row[t.b[j]];
      S[(size_t)a].insert(b);
      S[(size_t)b].insert(a);
    }
  }
  flatten(S, N, offsets, indices, nnz);
  return OK;
}

// Element-sharing ("FEM sparsity") node mode: adj(v) = { u != v : some element
// contains both u and v }.  Equals the edge adjacency for simplices; adds the diagonals of quads
// and hexes.
int oracle_node_shared_csr(int etype, const int32_t* conn, int64_t M, int64_t N, int64_t** offsets,
                           int32_t** indices, int64_t* nnz, int64_t* err_elem, int32_t* err_pos) {
  int rc = oracle_validate(etype, conn, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  const int k = kTables[etype].arity;
  std::vector<std::set<int32_t>> S((size_t)N);
  for (int64_t e = 0; e < M; ++e) {
    const int32_t* row = conn + e * k;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        if (i != j) S[(size_t)row[i]].insert(row[j]);
  }
  flatten(S, N, offsets, indices, nnz);
  return OK;
}

// Element mode: inc(v) = { e : v in conn[e] }, ascending (elements are visited in order).
int oracle_elem_csr(int etype, const int32_t* conn, int64_t M, int64_t N, int64_t** offsets,
                    int32_t** indices, int64_t* nnz, int64_t* err_elem, int32_t* err_pos) {
  int rc = oracle_validate(etype, conn, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  const int k = kTables[etype].arity;
  std::vector<std::vector<int32_t>> L((size_t)N);
  for (int64_t e = 0; e < M; ++e)
    for (int p = 0; p < k; ++p) L[(size_t)conn[e * k + p]].push_back((int32_t)e);
  flatten(L, N, offsets, indices, nnz);
  return OK;
}

// ---- polygon / mixed-arity surface meshes (SPEC Mesh.element_kind Polygon) ----
// Element e is the ring idx[off[e]], ..., idx[off[e+1]-1]; its edges are consecutive ring entries
// plus the closing edge (SPEC Element: "order defines the edge ring for surface elements").
// Validation per element, ascending (reading R18): arity >= 3 first (ERR_ARITY, pos -1), then the
// range check over the ring, then the repeated-node check, as for the fixed types.
enum { ERR_ARITY = 4 };

int oracle_poly_validate(const int64_t* off, const int32_t* idx, int64_t M, int64_t N, int64_t* eelem,
                         int32_t* epos) {
  if (M < 0 || N < 0 || (M > 0 && off[0] != 0)) return ERR_ARG;
  for (int64_t e = 0; e < M; ++e)
    if (off[e + 1] < off[e]) return ERR_ARG;
  *eelem = -1;
  *epos = -1;
  for (int64_t e = 0; e < M; ++e) {
    const int64_t k = off[e + 1] - off[e];
    const int32_t* row = idx + off[e];
    if (k < 3) { *eelem = e; *epos = -1; return ERR_ARITY; }
    for (int64_t p = 0; p < k; ++p)
      if (row[p] < 0 || (int64_t)row[p] >= N) { *eelem = e; *epos = (int32_t)p; return ERR_RANGE; }
    for (int64_t p = 1; p < k; ++p)
      for (int64_t q = 0; q < p; ++q)
        if (row[q] == row[p]) { *eelem = e; *epos = (int32_t)p; return ERR_DEGENERATE; }
  }
  return OK;
}

// mode 0: ring-edge node adjacency; 1: element incidence; 2: element-sharing node adjacency
int oracle_poly_csr(int mode, const int64_t* off, const int32_t* idx, int64_t M, int64_t N, int64_t** offsets,
                    int32_t** indices, int64_t* nnz, int64_t* err_elem, int32_t* err_pos) {
  int rc = oracle_poly_validate(off, idx, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  if (mode == 1) {
    std::vector<std::vector<int32_t>> L((size_t)N);
    for (int64_t e = 0; e < M; ++e)
      for (int64_t p = off[e]; p < off[e + 1]; ++p) L[(size_t)idx[p]].push_back((int32_t)e);
    flatten(L, N, offsets, indices, nnz);
    return OK;
  }
  std::vector<std::set<int32_t>> S((size_t)N);
  for (int64_t e = 0; e < M; ++e) {
    const int64_t k = off[e + 1] - off[e];
    const int32_t* row = idx + off[e];
    for (int64_t i = 0; i < k; ++i) {
      if (mode == 0) {
        const int32_t a = row[i], b = row[(i + 1) % k];
        S[(size_t)a].insert(b);
        S[(size_t)b].insert(a);
      } else {
        for (int64_t j = 0; j < k; ++j)
          if (i != j) S[(size_t)row[i]].insert(row[j]);
      }
    }
  }
  flatten(S, N, offsets, indices, nnz);
  return OK;
}

// ---- node-range mode ("an optional T-thread mode where thread t owns node range t
// and scans all elements; the output is identical") ----
// The same two loops as oracle_node_csr / oracle_elem_csr, restricted to the vertices v with
// lo <= v < hi: every element is still visited in ascending order, and a pair / incidence is kept
// only when its first node lies in the range.  The slice's offsets are relative to its first
// entry (offsets[0] = 0, hi - lo + 1 entries).  Validation is the caller's (it is global).
namespace {

struct Slice {
  int64_t* off = nullptr;
  int32_t* idx = nullptr;
  int64_t nnz = 0;
};

// mode 0: edge node adjacency; 1: element incidence; 2: element-sharing node adjacency
void range_csr(int mode, int etype, const int32_t* conn, int64_t M, int64_t lo, int64_t hi, Slice* out) {
  const EdgeTable& t = kTables[etype];
  const int k = t.arity;
  const int64_t R = hi - lo;
  if (mode == 1) {
    std::vector<std::vector<int32_t>> L((size_t)R);
    for (int64_t e = 0; e < M; ++e)
      for (int p = 0; p < k; ++p) {
        const int64_t n = conn[e * k + p];
        if (n >= lo && n < hi) L[(size_t)(n - lo)].push_back((int32_t)e);
      }
    flatten(L, R, &out->off, &out->idx, &out->nnz);
    return;
  }
  std::vector<std::set<int32_t>> S((size_t)R);
  for (int64_t e = 0; e < M; ++e) {
    const int32_t* row = conn + e * k;
    if (mode == 0) {
      for (int j = 0; j < t.nedges; ++j) {
        const int32_t a = row[t.a[j]], b = row[t.b[j]];
        if (a >= lo && a < hi) S[(size_t)(a - lo)].insert(b);
        if (b >= lo && b < hi) S[(size_t)(b - lo)].insert(a);
      }
    } else {
      for (int i = 0; i < k; ++i)
        if (row[i] >= lo && row[i] < hi)
          for (int j = 0; j < k; ++j)
            if (i != j) S[(size_t)(row[i] - lo)].insert(row[j]);
    }
  }
  flatten(S, R, &out->off, &out->idx, &out->nnz);
}

}  // namespace

// The CSR slice of vertices [lo, hi) (0 <= lo <= hi <= N), after validating the whole mesh.
int oracle_csr_range(int mode, int etype, const int32_t* conn, int64_t M, int64_t N, int64_t lo, int64_t hi,
                     int64_t** offsets, int32_t** indices, int64_t* nnz, int64_t* err_elem, int32_t* err_pos) {
  if (mode < 0 || mode > 2 || lo < 0 || hi < lo || hi > N) return ERR_ARG;
  int rc = oracle_validate(etype, conn, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  Slice s;
  range_csr(mode, etype, conn, M, lo, hi, &s);
  *offsets = s.off;
  *indices = s.idx;
  *nnz = s.nnz;
  return OK;
}

// T threads: thread t owns vertices [t*N/T, (t+1)*N/T) and scans all elements; the slices are
// concatenated in t order, shifting each slice's offsets by the nnz before it.  Identical to the
// one-thread oracle by construction (each vertex's list is built by exactly one thread from the
// same ascending element scan).  *threads_used reports T after clamping to [1, max(N, 1)].
int oracle_csr_mt(int mode, int etype, const int32_t* conn, int64_t M, int64_t N, int T, int64_t** offsets,
                  int32_t** indices, int64_t* nnz, int64_t* err_elem, int32_t* err_pos, int* threads_used) {
  if (mode < 0 || mode > 2) return ERR_ARG;
  int rc = oracle_validate(etype, conn, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  if (T < 1) T = 1;
  if ((int64_t)T > N && N > 0) T = (int)N;
  if (threads_used) *threads_used = T;
  std::vector<Slice> slices((size_t)T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) {
    const int64_t lo = N * t / T, hi = N * (t + 1) / T;
    pool.emplace_back(range_csr, mode, etype, conn, M, lo, hi, &slices[(size_t)t]);
  }
  for (auto& th : pool) th.join();
  int64_t total = 0;
  for (const Slice& s : slices) total += s.nnz;
  int64_t* off = (int64_t*)std::malloc(sizeof(int64_t) * (size_t)(N + 1));
  int32_t* idx = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)(total > 0 ? total : 1));
  off[0] = 0;
  int64_t v = 0, base = 0;
  for (int t = 0; t < T; ++t) {
    const Slice& s = slices[(size_t)t];
    const int64_t R = N * (t + 1) / T - N * t / T;
    for (int64_t i = 0; i < R; ++i) off[v + i + 1] = base + s.off[i + 1];
    if (s.nnz) std::memcpy(idx + base, s.idx, sizeof(int32_t) * (size_t)s.nnz);
    v += R;
    base += s.nnz;
    std::free(s.off);
    std::free(s.idx);
  }
  *offsets = off;
  *indices = idx;
  *nnz = total;
  return OK;
}

// Polygon meshes, node-range mode: oracle_poly_csr's loops restricted to vertices [lo, hi).
int oracle_poly_csr_range(int mode, const int64_t* off, const int32_t* idx, int64_t M, int64_t N, int64_t lo,
                          int64_t hi, int64_t** offsets, int32_t** indices, int64_t* nnz, int64_t* err_elem,
                          int32_t* err_pos) {
  if (mode < 0 || mode > 2 || lo < 0 || hi < lo || hi > N) return ERR_ARG;
  int rc = oracle_poly_validate(off, idx, M, N, err_elem, err_pos);
  if (rc != OK) return rc;
  const int64_t R = hi - lo;
  if (mode == 1) {
    std::vector<std::vector<int32_t>> L((size_t)R);
    for (int64_t e = 0; e < M; ++e)
      for (int64_t p = off[e]; p < off[e + 1]; ++p)
        if (idx[p] >= lo && idx[p] < hi) L[(size_t)(idx[p] - lo)].push_back((int32_t)e);
    flatten(L, R, offsets, indices, nnz);
    return OK;
  }
  std::vector<std::set<int32_t>> S((size_t)R);
  for (int64_t e = 0; e < M; ++e) {
    const int64_t k = off[e + 1] - off[e];
    const int32_t* row = idx + off[e];
    for (int64_t i = 0; i < k; ++i) {
      if (mode == 0) {
        const int32_t a = row[i], b = row[(i + 1) % k];
        if (a >= lo && a < hi) S[(size_t)(a - lo)].insert(b);
        if (b >= lo && b < hi) S[(size_t)(b - lo)].insert(a);
      } else if (row[i] >= lo && row[i] < hi) {
        for (int64_t j = 0; j < k; ++j)
          if (i != j) S[(size_t)(row[i] - lo)].insert(row[j]);
      }
    }
  }
  flatten(S, R, offsets, indices, nnz);
  return OK;
}

void oracle_free(void* p) { std::free(p); }

}  // extern "C"
