/* meshnbr.h — C ABI of libmeshnbr.so: one-ring nodal neighbours of generic meshes on B200.
 *
 * Method: Mei, Xu, Tian, Li, "A Parallel Solution to Finding Nodal Neighbors in Generic Meshes"
 * (arXiv 1604.04689; /root/reference/PAPER.md).  Every vertex gets
 *   - its one-ring neighbouring NODES: "any pair of nodes connected by an edge is the one-ring
 *     neighboring node for each other" (§1, §2.1.1), and
 *   - its one-ring neighbouring ELEMENTS: "any element is directly the one-ring neighboring
 *     element for those nodes it contains" (§1, §2.1.2),
 * returned as CSR: int64 offsets[N+1] + int32 indices[nnz], every slice strictly ascending
 * (the paper's "number" and "first indices" of each vertex's neighbours, L234-237, L487-489;
 * readings R1-R3, R7, R12, R13 of DESIGN.md).
 *
 * Conventions for every entry point below
 *   - Pointers named d_* are CUDA device pointers, h_* host pointers.  Connectivity is
 *     int32 conn[num_elems][arity] row-major, 0-based, owned by the caller, read-only here.
 *   - All work is stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream) on the calling thread's current device, and the mn_find_* calls return
 *     with the outputs complete on `stream`.  They block the calling thread to read device
 *     words whose values size the outputs or choose the algorithm:
 *       - mn_find_{node,elem}_neighbors, _both, _shared: once (validation word + nnz), plus once
 *         before it on meshes of >= 2^20 elements with the automatic element path (the locality
 *         sample that picks the element-CSR algorithm);
 *       - mn_find_poly_neighbors: three times (offset bounds; validation + element offsets; node nnz);
 *       - mn_find_neighbors_both_chunked: once per node range, plus once;
 *       - mn_find_neighbors_both_host: as _both, plus the final D2H;
 *       - mn_host_pipeline_submit: as _both (its uploads and downloads do not block);
 *         mn_host_pipeline_wait: until that ticket's downloads are complete;
 *       - mn_find_neighbors_dist: as _both, plus the exchange's count step (see there).
 *     Stage primitives (mn_emit_*, mn_radix_sort_*, ...) do not block unless stated.
 *   - Memory: outputs and workspace come from the caller's mn_allocator (NULL = the library's
 *     cudaMallocAsync on `stream`); the library allocates and releases on `stream` only.  Outputs
 *     are owned by the caller; release them with mn_csr_release.  Workspace is released before
 *     return (stream-ordered: an allocator must not hand a released block to another stream
 *     before `stream` has passed the release point).
 *   - Global state: (1) the optional profiler (mn_profile_*; not thread-safe; bench only);
 *     (2) two process-wide test knobs, mn_set_elem_path and mn_set_chunk_cap (defaults: auto,
 *     0), which change the algorithm but never the result; (3) per-device one-time setup
 *     (kernel shared-memory attributes, an occupancy-derived grid size), guarded per device, so
 *     one process may drive several GPUs and several threads may call concurrently; (4) per
 *     thread and device: a pinned staging word pair and the host path's side stream + event.
 *   - Errors: invalid input is reported as the LOWEST offending element id, then the lowest
 *     position in it; an index outside [0, N) is reported before a repeated node of the same
 *     element (reading R8).  On any error no output is returned (out->offsets == NULL).
 *   - Deterministic: identical inputs give bit-identical outputs.
 *   - Limits: 0 <= num_nodes <= INT32_MAX, 0 <= num_elems, num_elems*arity*... pairs < 2^53.
 */
#ifndef MESHNBR_H_
#define MESHNBR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MN_ABI_VERSION 1

/* Element types (arity): edge sets per DESIGN.md reading R4 — TRI3 3 edges,
 * QUAD4 4 ring edges, TET4 all 6 node pairs, HEX8 the 12 edges of a VTK_HEXAHEDRON (nodes 0-3
 * bottom ring, 4-7 top ring, 4 above 0). */
typedef enum { MN_TRI3 = 0, MN_QUAD4 = 1, MN_TET4 = 2, MN_HEX8 = 3 } mn_elem_type;

typedef enum {
  MN_OK = 0,
  MN_ERR_INVALID_ARG = 1,        /* null pointer, negative size, N > INT32_MAX, unknown type   */
  MN_ERR_INDEX_OUT_OF_RANGE = 2, /* conn[e][p] < 0 or >= N; detail = (e, p)                     */
  MN_ERR_DEGENERATE = 3,         /* conn[e][p] == conn[e][q] for some q < p; detail = (e, p)    */
  MN_ERR_CAPACITY = 4,           /* too many pairs for the 54-bit counters, or caller capacity */
  MN_ERR_OOM = 5,                /* the allocator returned NULL                                  */
  MN_ERR_CUDA = 6,               /* a CUDA runtime error (launch, copy, sync)                    */
  MN_ERR_ARITY = 7,              /* polygon meshes: an element with fewer than 3 nodes;
                                    detail = (e, -1) (SPEC ArityMismatch, R18)         */
  MN_ERR_SYNTAX = 8,             /* OFF/OBJ: malformed line; detail = (line, token position)    */
  MN_ERR_COUNT_MISMATCH = 9,     /* OFF: fewer / more vertex or face lines than the counts line  */
  MN_ERR_ZERO_INDEX = 10,        /* OBJ: face index 0; detail = (line, token position)           */
  MN_ERR_COMM = 11               /* multi-GPU: an exchange operation (NCCL or the caller's mn_comm)
                                    failed, or NCCL could not be loaded                          */
} mn_status;

typedef void* mn_stream; /* cudaStream_t */

/* Stream-ordered allocator.  alloc returns NULL on failure; release may be called with NULL. */
typedef struct mn_allocator {
  void* (*alloc)(void* ctx, size_t bytes, mn_stream stream);
  void (*release)(void* ctx, void* ptr, mn_stream stream);
  void* ctx;
} mn_allocator;

/* CSR result.  offsets: num_nodes+1 entries, offsets[0] = 0, offsets[num_nodes] = nnz.
 * indices: nnz entries (NULL when nnz == 0); the slice of vertex v, indices[offsets[v] ..
 * offsets[v+1]), is strictly ascending.  Both arrays were obtained from `owner`. */
typedef struct mn_csr {
  int64_t num_nodes;
  int64_t nnz;
  int64_t* offsets;
  int32_t* indices;
  mn_allocator owner;
} mn_csr;

typedef struct mn_error_detail {
  int64_t elem; /* offending element id, -1 if none */
  int32_t pos;  /* offending local position, -1 if none */
} mn_error_detail;

/* ---------------------------------------------------------------------------------------------
 * Whole path
 * ------------------------------------------------------------------------------------------- */

/* One-ring neighbouring NODES of every vertex (§2.2.1: create the pairs of
 * every edge in both directions, sort them by the first integer, segmented reduction and scan).
 * d_conn: device int32[num_elems * arity].  out: device CSR (allocator `alloc`).  err: nullable. */
mn_status mn_find_node_neighbors(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                                 int64_t num_nodes, const mn_allocator* alloc, mn_stream stream,
                                 mn_csr* out, mn_error_detail* err);

/* Same result as mn_find_node_neighbors, computed by the paper's node pipeline verbatim: every
 * node pair (a, v) of every element edge is created (§2.2.1), the packed keys
 * (a << b | v) are LSD-radix-sorted over all 2b bits (L228-232), adjacent duplicates dropped and
 * run lengths scanned into offsets (L234-245).  mn_find_node_neighbors reaches the identical CSR
 * from the element-pair sort instead (DESIGN.md §"Node path"); this entry is kept for parity and
 * measurement. */
mn_status mn_find_node_neighbors_sortpairs(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                                           int64_t num_nodes, const mn_allocator* alloc, mn_stream stream,
                                           mn_csr* out, mn_error_detail* err);

/* Element-sharing ("FEM sparsity") node adjacency (the title's "generic
 * meshes"): u and v are neighbours iff some element contains both, i.e. the pattern of B^T B minus
 * the diagonal.  Identical to mn_find_node_neighbors for TRI3/TET4; adds the face and body
 * diagonals of QUAD4/HEX8.  Same conventions and outputs as mn_find_node_neighbors. */
mn_status mn_find_node_neighbors_shared(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                                        int64_t num_nodes, const mn_allocator* alloc, mn_stream stream,
                                        mn_csr* out, mn_error_detail* err);

/* Polygon / mixed-arity surface meshes (PAPER.md title "generic meshes",
 * §2.2; SPEC.md Mesh element_kind Polygon S:L32-36).  Connectivity in CSR form, device
 * memory: element e is the ring d_idx[d_off[e]], ..., d_idx[d_off[e+1]-1] (arity >= 3), its edges
 * are consecutive ring entries plus the closing edge.  d_off: num_elems + 1 int64 with d_off[0] = 0
 * and d_off[num_elems] = conn_len (else MN_ERR_INVALID_ARG); d_idx: conn_len int32.
 * Outputs (each nullable, at least one non-null), same conventions as mn_find_node_neighbors:
 *   node_out   ring-edge node adjacency (one-ring neighbouring nodes)
 *   elem_out   one-ring neighbouring elements (ascending)
 *   shared_out element-sharing node adjacency (pattern of B^T B minus the diagonal)
 * Validation per element in ascending order (R18): arity >= 3 (MN_ERR_ARITY, pos -1), then the
 * range check, then the repeated-node check; the lowest offending element is reported.
 * Blocks three times (offset bounds, validation + sizes, the node nnz values). */
mn_status mn_find_poly_neighbors(const int64_t* d_off, const int32_t* d_idx, int64_t num_elems,
                                 int64_t conn_len, int64_t num_nodes, const mn_allocator* alloc,
                                 mn_stream stream, mn_csr* node_out, mn_csr* elem_out, mn_csr* shared_out,
                                 mn_error_detail* err);

/* One-ring neighbouring ELEMENTS of every vertex (§2.2.2: pairs (node, element
 * itself), sorted by node, segmented reduction and scan).  Slices list element ids ascending. */
mn_status mn_find_elem_neighbors(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                                 int64_t num_nodes, const mn_allocator* alloc, mn_stream stream,
                                 mn_csr* out, mn_error_detail* err);

/* Both outputs from one validation/histogram read of the connectivity (the bench's "step"). */
mn_status mn_find_neighbors_both(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                                 int64_t num_nodes, const mn_allocator* alloc, mn_stream stream,
                                 mn_csr* node_out, mn_csr* elem_out, mn_error_detail* err);

/* Memory-bounded form of mn_find_neighbors_both (the device-memory cost the
 * paper names as its shortcoming, §3.2.2): the nodes are processed in contiguous
 * ranges, first K of them (K the smallest power of two whose per-range estimate,
 * mn_chunk_workspace_bytes, fits), each by the counting-sort transpose + per-node expansion
 * restricted to its nodes.  A range whose actual workspace (known after its count pass) exceeds
 * max_workspace_bytes is halved until it fits, so the workspace never exceeds the budget except
 * for a single node whose own incidences do (processed alone).  Not counted in the budget: the
 * outputs, and the node-index slices of the finished ranges (node nnz in total), which are
 * concatenated into the output at the end (2 x node nnz at that moment).  Same outputs as
 * mn_find_neighbors_both; blocks twice per range.  *chunks_used (nullable) receives the number of
 * ranges processed. */
mn_status mn_find_neighbors_both_chunked(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                                         int64_t num_nodes, size_t max_workspace_bytes,
                                         const mn_allocator* alloc, mn_stream stream, mn_csr* node_out,
                                         mn_csr* elem_out, int64_t* chunks_used, mn_error_detail* err);

/* Same as mn_find_neighbors_both with HOST buffers: h_conn is host memory (pinned for full PCIe
 * speed); the connectivity is copied to the device, both CSRs are computed and copied back into
 * host memory obtained from `host_alloc` (its alloc receives the byte count; stream unused).
 * Device workspace comes from `dev_alloc`.  The outputs' `owner` is host_alloc. */
mn_status mn_find_neighbors_both_host(mn_elem_type type, const int32_t* h_conn, int64_t num_elems,
                                      int64_t num_nodes, const mn_allocator* dev_alloc,
                                      const mn_allocator* host_alloc, mn_stream stream,
                                      mn_csr* node_out, mn_csr* elem_out, mn_error_detail* err);

/* Pipelined host-buffer form (a stream of meshes, e.g. many time steps or many parts): the same
 * outputs as mn_find_neighbors_both_host, but the PCIe transfers of consecutive meshes overlap.
 * The pipeline owns three streams on the current device: upload (H2D of the connectivity), compute
 * (mn_find_neighbors_both) and download (D2H of both CSRs; the element CSR starts during the node
 * pass).  PCIe is full duplex, so the upload of mesh i + 1 runs while the download of mesh i is
 * still in flight (B200 box, measured: 55 GB/s one way, 92 GB/s both ways at once).
 *   create:  dev_alloc / host_alloc as for mn_find_neighbors_both_host (NULL dev_alloc =
 *            cudaMallocAsync on the stream given to alloc); device = the current device.
 *   submit:  validates and copies h_conn (host memory, pinned for full speed; it must stay
 *            unchanged until mn_host_pipeline_wait(ticket) returns), computes both CSRs (blocks
 *            like mn_find_neighbors_both: one read of the validation word and nnz), enqueues the
 *            downloads and returns.  node_out / elem_out receive host CSRs (owner = host_alloc)
 *            whose CONTENTS are valid only after mn_host_pipeline_wait(*ticket).  On an error
 *            (invalid mesh: lowest element, then position, reading R8) nothing is returned and no
 *            ticket is issued; earlier tickets are unaffected.
 *   wait:    blocks until the downloads of `ticket` are complete, then releases its device
 *            buffers.  Tickets may be waited in any order; each exactly once.
 *   destroy: waits for every outstanding ticket and releases the streams.
 * Device memory: the workspace of one call plus, per outstanding ticket, its connectivity and
 * device CSRs.  Not thread-safe per pipeline. */
typedef struct mn_host_pipeline mn_host_pipeline;
mn_status mn_host_pipeline_create(const mn_allocator* dev_alloc, const mn_allocator* host_alloc,
                                  mn_host_pipeline** out);
mn_status mn_host_pipeline_submit(mn_host_pipeline* p, mn_elem_type type, const int32_t* h_conn, int64_t num_elems,
                                  int64_t num_nodes, mn_csr* node_out, mn_csr* elem_out, int64_t* ticket,
                                  mn_error_detail* err);
mn_status mn_host_pipeline_wait(mn_host_pipeline* p, int64_t ticket);
void mn_host_pipeline_destroy(mn_host_pipeline* p);

/* Releases offsets/indices through csr->owner on `stream` and zeroes the struct. */
void mn_csr_release(mn_csr* csr, mn_stream stream);

const char* mn_status_string(mn_status status);
int mn_abi_version(void);

/* Peak device workspace (bytes, excluding the returned outputs) of the call above for this mesh
 * (the memory cost the paper names as its shortcoming, §3.2.2).
 * modes: 1 = nodes, 2 = elements, 3 = both. */
mn_status mn_workspace_bytes(mn_elem_type type, int64_t num_elems, int64_t num_nodes, int modes,
                             size_t* bytes);

/* Estimated per-range workspace of mn_find_neighbors_both_chunked with `chunks` node ranges. */
size_t mn_chunk_workspace_bytes(mn_elem_type type, int64_t num_elems, int64_t num_nodes, int64_t chunks);

/* ---------------------------------------------------------------------------------------------
 * Stage primitives (one per §8(a) row; the tests check each against oracle/stages.py)
 * ------------------------------------------------------------------------------------------- */

/* Node-key width in bytes for a mesh of num_nodes nodes: 4 when 2*b <= 32, else 8, where
 * b = max(1, bit_length(num_nodes - 1)).  Key of pair (a, v) = (a << b) | v. */
int mn_node_key_bits(int64_t num_nodes);   /* returns b */
int mn_node_key_bytes(int64_t num_nodes);

/* Row a1 — validate + create the node pairs of PAPER.md §2.2.1 L220-226 ("a triangle can produce
 * six pairs"): for element e and edge j=(i0,i1) of the type's edge table, slot e*2E + 2j holds the
 * packed key (conn[e][i0], conn[e][i1]) and slot e*2E + 2j + 1 the reverse.  d_keys: device,
 * 2*E*num_elems keys of mn_node_key_bytes(num_nodes) bytes.  Blocks once (validation result). */
mn_status mn_emit_node_pairs(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                             int64_t num_nodes, void* d_keys, mn_stream stream,
                             mn_error_detail* err);

/* Row a2 — validate + create the element pairs of PAPER.md §2.2.2: slot e*arity + p
 * holds key conn[e][p] and value e.  d_keys, d_vals: device uint32[arity*num_elems]. */
mn_status mn_emit_elem_pairs(mn_elem_type type, const int32_t* d_conn, int64_t num_elems,
                             int64_t num_nodes, uint32_t* d_keys, uint32_t* d_vals,
                             mn_stream stream, mn_error_detail* err);

/* Row a3 — LSD radix sort (onesweep: decoupled look-back digit scans) of n unsigned keys of
 * key_bytes (4 or 8) bytes, ascending on their low key_bits bits (bits above must be 0).
 * In place on d_keys (workspace from alloc).  Stream-ordered, no blocking. */
mn_status mn_radix_sort_keys(void* d_keys, int key_bytes, int64_t n, int key_bits,
                             const mn_allocator* alloc, mn_stream stream);

/* Row a3e — STABLE LSD radix sort of uint32 (key, value) pairs on the low key_bits key bits. */
mn_status mn_radix_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_vals, int64_t n, int key_bits,
                                  const mn_allocator* alloc, mn_stream stream);

/* Rows a4+a5 (node mode) — from n ascending packed node keys (key_bytes 4/8, node bits b =
 * mn_node_key_bits(num_nodes)): drop keys equal to their predecessor (reading R1), write the
 * neighbour part (key & (2^b - 1)) of each survivor to d_indices (capacity n) and the CSR
 * offsets of every node to d_offsets[num_nodes+1] (run lengths of the node part, exclusive scan;
 * PAPER.md L234-245).  *h_nnz receives the survivor count (blocks once). */
mn_status mn_unique_node_csr(const void* d_sorted_keys, int key_bytes, int64_t n,
                             int64_t num_nodes, int64_t* d_offsets, int32_t* d_indices,
                             int64_t* h_nnz, const mn_allocator* alloc, mn_stream stream);

/* Rows a4+a5 (element mode) — CSR offsets d_offsets[num_nodes+1] from n ascending uint32 node
 * keys (run lengths per node, exclusive scan; no dedupe: element pairs are unique).  No blocking. */
mn_status mn_elem_offsets(const uint32_t* d_sorted_keys, int64_t n, int64_t num_nodes,
                          int64_t* d_offsets, mn_stream stream);

/* Row a5 — exclusive scan (single pass, decoupled look-back): d_out[0] = 0,
 * d_out[i+1] = d_out[i] + d_counts[i], for n int32 counts -> n+1 int64.  No blocking. */
mn_status mn_exclusive_scan_i32(const int32_t* d_counts, int64_t n, int64_t* d_out,
                                const mn_allocator* alloc, mn_stream stream);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU building blocks: nodes are owned in contiguous ranges
 * [r*ceil(N/G), (r+1)*ceil(N/G)); each rank holds an element shard with a global element base.
 * Only incidences travel: the owner of node a receives every (a, e) pair together with e's row,
 * which is all it needs for both CSR slices (the node pairs of a are the expansion of a's element
 * list).  mn_find_neighbors_dist (below) runs both with the exchange in between;
 * these stage entry points serve tests that emulate several ranks on one device.
 * ------------------------------------------------------------------------------------------- */

/* Validate the shard (error element ids are global) and bucket its incidences by owner rank,
 * stably, so each bucket stays element-major:
 *   d_pairs[i]        uint64 (node << 32 | global element id), arity*shard_elems entries (caller);
 *   h_counts[g]       incidences destined to rank g (host, world entries);
 *   *d_row_elems, *d_rows  (allocated here from `alloc`, released by the caller): one row per
 *                     distinct (destination g != self_rank, element) pair, grouped by destination,
 *                     element ids ascending within a group — the remote rows the owners need;
 *   h_row_counts[g]   rows destined to rank g (0 for self_rank).  Blocks once. */
mn_status mn_dist_bucket(mn_elem_type type, const int32_t* d_conn_shard, int64_t shard_elems,
                         int64_t global_elem_base, int64_t num_nodes, int world, int self_rank,
                         uint64_t* d_pairs, int64_t* h_counts, int32_t** d_row_elems, int32_t** d_rows,
                         int64_t* h_row_counts, const mn_allocator* alloc, mn_stream stream,
                         mn_error_detail* err);

/* Owner side: from the n received incidences (concatenated in source-rank order, so element ids
 * ascend per node) and the n_rows received remote rows (element ids ascending), build the CSR
 * slices of nodes [lo, hi): local offsets (slice offsets[0] = 0), global node / element ids as
 * indices.  Rows of local elements are read from the own shard (d_conn_shard, shard_elems,
 * global_elem_base).  Blocks once (node nnz). */
mn_status mn_dist_finish(mn_elem_type type, const uint64_t* d_pairs, int64_t n, const int32_t* d_row_elems,
                         const int32_t* d_rows, int64_t n_rows, const int32_t* d_conn_shard,
                         int64_t shard_elems, int64_t global_elem_base, int64_t num_nodes, int64_t lo,
                         int64_t hi, const mn_allocator* alloc, mn_stream stream, mn_csr* node_slice,
                         mn_csr* elem_slice);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU whole path (the paper's stated limit is one device's memory,
 * PAPER.md §3.2.2).  One process (or thread) per GPU; rank r holds the element shard
 * [global_elem_base, global_elem_base + shard_elems) of a mesh of num_nodes nodes (shards
 * contiguous, ascending with the rank) and receives the CSR slices of the nodes it owns,
 * [lo, hi) = [r * ceil(N/G), (r+1) * ceil(N/G)) clipped to N.  Inside one call, on `stream`:
 *   1. validate the shard, count its incidences per owner and (when the shard is coherent: the
 *      locality sample of the 1-GPU path) collect its REMOTE incidences (owner != r);
 *   2. count exchange: one all-gather of every rank's [error word, status, counts per owner,
 *      locality]; the lowest error over all ranks is returned by EVERY rank (so no rank is left
 *      waiting in a collective), before any payload moves;
 *   3. bucket-and-send: one owner-digit onesweep pass stores each remote incidence and its element
 *      row at its place in the owner's receive layout (source-rank order, element-major) — in a
 *      local send buffer followed by ONE grouped all-to-all(v) (mn_find_neighbors_dist), or directly
 *      in the owner's symmetric heap over peer memory followed by an all-gather as a barrier
 *      (mn_find_neighbors_dist_p2p);
 *   4. local finish: if every shard is coherent, an owner's own incidences are never materialised —
 *      its element CSR slice is the chunk transpose of (own shard filtered to [lo, hi)) + (received
 *      incidences), its node slice the per-node expansion + dedupe with rows from the own shard or
 *      the received rows; otherwise the own bucket is kept in place between the received ones and
 *      the slice is built from all of them (stable LSD on the local node id);
 *   5. one all-gather of the slice nnz values: the global offset bases of the slices.
 * Concatenating the slices of all ranks in rank order (offsets shifted by the bases) is
 * bit-identical to the single-GPU CSRs.  Blocks the calling thread a few times (the locality
 * sample, steps 1, 2, 4, 5).  All collectives are called in the same order on every rank.
 * ------------------------------------------------------------------------------------------- */

/* One all-to-all(v) exchange of a group: rank r sends send_counts[g] elements of elem_bytes bytes,
 * starting at element send_displs[g] of `send`, to rank g, and receives recv_counts[g] elements
 * from rank g at element recv_displs[g] of `recv`.  Device buffers; host count/displacement
 * arrays of `world` entries.  A zero count means no message. */
typedef struct {
  const void* send;
  const int64_t* send_counts;
  const int64_t* send_displs;
  void* recv;
  const int64_t* recv_counts;
  const int64_t* recv_displs;
  size_t elem_bytes;
} mn_a2a_op;

/* The exchange operations the multi-GPU path needs.  mn_comm_from_nccl fills one over NCCL
 * (NVLink / NVSwitch); a caller may supply its own (tests drive the path over gloo with host
 * staging this way).  Both callbacks return 0 on success, and must be stream-ordered on `stream`
 * or complete before returning. */
typedef struct {
  int rank;
  int world;
  void* ctx;
  /* every rank contributes `bytes` bytes at d_send; d_recv gets world * bytes in rank order */
  int (*allgather)(void* ctx, const void* d_send, void* d_recv, size_t bytes, mn_stream stream);
  /* the n_ops exchanges as one group (NCCL: one ncclGroupStart / ncclGroupEnd) */
  int (*alltoallv)(void* ctx, const mn_a2a_op* ops, int n_ops, mn_stream stream);
} mn_comm;

typedef struct {
  int64_t lo, hi;              /* owned node range                                          */
  int64_t node_base, elem_base;/* global offsets of this rank's slices in the 1-GPU CSRs       */
  int64_t node_nnz_total;      /* node CSR nnz over all ranks                                 */
  int64_t elem_nnz_total;      /* element CSR nnz over all ranks (= arity * total elements)  */
  int64_t sent_bytes;          /* payload bytes this rank sent to other ranks (step 3)        */
  int64_t recv_bytes;          /* payload bytes it received                                   */
  int64_t own_incidences;      /* incidences it kept (read in place, not exchanged)           */
} mn_dist_info;

/* Both CSR slices (node_slice, elem_slice: local offsets, slice offsets[0] = 0, hi - lo + 1
 * entries; global node / element ids as indices).  Validation errors are global: every rank
 * returns the lowest offending (global element id, position) of all shards.  A comm failure gives
 * MN_ERR_COMM; a local failure (OOM, CUDA) on any rank gives that status on every rank if it
 * happens before step 2, else on that rank only.  info may be NULL. */
mn_status mn_find_neighbors_dist(mn_elem_type type, const int32_t* d_conn_shard, int64_t shard_elems,
                                 int64_t global_elem_base, int64_t num_nodes, const mn_comm* comm,
                                 const mn_allocator* alloc, mn_stream stream, mn_csr* node_slice,
                                 mn_csr* elem_slice, mn_dist_info* info, mn_error_detail* err);

/* SURVEY.md §8(b)'s single-output forms over an NCCL communicator (an ncclComm_t passed as void*,
 * e.g. from mn_nccl_comm_init): the node (elem) slice of nodes [*lo, *hi) and its global offset
 * *global_nnz_base. */
mn_status mn_find_node_neighbors_dist(mn_elem_type type, const int32_t* d_conn_shard, int64_t shard_elems,
                                      int64_t global_elem_base, int64_t num_nodes, void* nccl_comm,
                                      const mn_allocator* alloc, mn_stream stream, mn_csr* slice, int64_t* lo,
                                      int64_t* hi, int64_t* global_nnz_base, mn_error_detail* err);
mn_status mn_find_elem_neighbors_dist(mn_elem_type type, const int32_t* d_conn_shard, int64_t shard_elems,
                                      int64_t global_elem_base, int64_t num_nodes, void* nccl_comm,
                                      const mn_allocator* alloc, mn_stream stream, mn_csr* slice, int64_t* lo,
                                      int64_t* hi, int64_t* global_nnz_base, mn_error_detail* err);

/* Fused bucket-and-send over peer memory (the dispatch all-to-all done inside the bucketing kernel):
 * the same result as mn_find_neighbors_dist, but step 3's all-to-all disappears — after the count
 * exchange, the owner-digit onesweep pass stores each incidence (and, for remote owners, the element
 * row) directly into its owner's receive region of a symmetric heap that every rank maps from every
 * other rank with CUDA IPC (NVLink / NVSwitch peer memory on one node; processes sharing a device in
 * tests).  Then one all-gather as a barrier, the local finish reading the heap in place, and the nnz
 * all-gather.  The heap grows collectively when a call needs more (all ranks decide the same size
 * from the all-gathered counts).  Single node only (CUDA IPC). */
typedef struct mn_symm mn_symm;
/* Collective over comm (only its allgather is used): every rank allocates `initial_bytes` (0 =
 * on first use) with cudaMalloc and maps the others'.  comm is copied (its ctx must stay valid). */
mn_status mn_symm_create(const mn_comm* comm, size_t initial_bytes, mn_symm** out);
/* Teardown: mn_symm_unmap on every rank (closes the mappings of the other ranks' heaps), then a
 * barrier of the caller's, then mn_symm_destroy (frees the own heap; unmaps first if needed). */
mn_status mn_symm_unmap(mn_symm* symm);
mn_status mn_symm_destroy(mn_symm* symm);
size_t mn_symm_capacity(const mn_symm* symm);
mn_status mn_find_neighbors_dist_p2p(mn_elem_type type, const int32_t* d_conn_shard, int64_t shard_elems,
                                     int64_t global_elem_base, int64_t num_nodes, mn_symm* symm,
                                     const mn_allocator* alloc, mn_stream stream, mn_csr* node_slice,
                                     mn_csr* elem_slice, mn_dist_info* info, mn_error_detail* err);

/* NCCL plumbing.  libnccl.so.2 is loaded on first use (dlopen; in a process that already loaded
 * PyTorch's NCCL that same library is used); MN_ERR_COMM if it cannot be.  Bootstrap: rank 0 calls
 * mn_nccl_get_unique_id, the caller broadcasts the 128 bytes (e.g. over a torch process group),
 * every rank calls mn_nccl_comm_init on its own (current) device. */
int mn_nccl_available(void);
mn_status mn_nccl_get_unique_id(void* id128);
mn_status mn_nccl_comm_init(const void* id128, int world, int rank, void** nccl_comm);
mn_status mn_nccl_comm_destroy(void* nccl_comm);
/* Fills *out with NCCL-backed exchange operations on nccl_comm (rank, world from the communicator). */
mn_status mn_comm_from_nccl(void* nccl_comm, mn_comm* out);

/* Host-only exchange plan of step 2 (used by mn_find_neighbors_dist; exported so the protocol can
 * be checked without a GPU).  gathered: world rows of (2 + 2 * world) int64 each, row g =
 * [error word of rank g, status of rank g, counts_g[0..world), aux_g[0..world)]
 * where counts_g[h] are the incidences rank g sends to rank h and aux_g[h] a per-destination
 * auxiliary count (mn_find_neighbors_dist stores rank g's locality flag in aux_g[0]).  Writes
 * recv_counts[g] = counts_g[rank] and recv_row_counts[g] = aux_g[rank] and returns the
 * global outcome: the first nonzero status in rank order, else the error of the lowest error word
 * (detail decoded into err), else MN_OK.  Error word: (global element << 5) | (repeated node << 4)
 * | position, all ones when the shard is valid — so the lowest word is the lowest element, and
 * within it a range error before a repeated node (reading R8). */
mn_status mn_dist_plan(int world, int rank, const int64_t* gathered, int64_t* recv_counts,
                       int64_t* recv_row_counts, mn_error_detail* err);

/* Stream-ordered copy between any two buffers (cudaMemcpyDefault), then a sync of `stream`
 * (host-staged exchange callbacks use it). */
mn_status mn_memcpy_sync(void* dst, const void* src, size_t bytes, mn_stream stream);

/* ---------------------------------------------------------------------------------------------
 * Algorithm selection for the element CSR (process-wide; results are identical either way).
 *   0 = auto: meshes of >= 2^20 elements whose consecutive elements share nodes (sampled: fewer
 *       than 0.5 distinct (slot, node) groups per incidence in windows of 32 elements) use the
 *       counting-sort transpose, all others the LSD radix sort.  Costs one extra blocking read.
 *   1 = LSD radix sort of (node, element) pairs (§2.2.2, "sort according to the
 *       first array of integers").
 *   2 = counting-sort transpose: per-node counts, scan, scatter, per-node sort of element ids
 *       (element CSR = transpose of the incidence matrix).
 *   3 = MSD: one stable onesweep pass buckets the (node, element) pairs by node range (512
 *       ranges), then one CTA per range counts, scans, scatters and sorts in shared memory
 *       (SURVEY.md §8(f) row 1).  Needs ceil(N / 512) <= 49152; otherwise the LSD sort runs.
 *       Not chosen by auto (measured slower than 1 on B200).
 * ------------------------------------------------------------------------------------------- */
mn_status mn_set_elem_path(int mode);
int mn_get_elem_path(void);

/* Test knob (process-wide): upper bound on the capacity, in entries, of the fixed-size 128-node
 * chunk buckets the transpose path scatters into in one read of conn (auto: twice the mean chunk
 * load, 2 * k * M / ceil(N / 128), rounded down to a multiple of 32).  0 restores auto.  When a
 * chunk overflows its bucket the counted path (count, scan, scatter) runs instead, so results never
 * depend on it; tests use a small cap to force that fallback.  MN_ERR_INVALID_ARG if cap < 0. */
mn_status mn_set_chunk_cap(int cap);

/* Small meshes (process-wide knob): with the automatic element path, fixed-type calls on meshes of
 * at most `max_incidences` (<= 8192, default 8192) element-node incidences and <= 4096 nodes run
 * in ONE CTA (validation, both transposes, the per-node sort + dedupe and both scans in shared
 * memory; the node lists are written straight into the output, whose allocation then has capacity
 * C * incidences >= nnz, at most 96 KB), then one blocking read (latency path, configs 1-like);
 * identical results.  0 disables it.  Not used for _shared, _host or forced element paths. */
mn_status mn_set_small_path(int64_t max_incidences);


/* ---------------------------------------------------------------------------------------------
 * Instrumentation (bench only; not thread-safe)
 * ------------------------------------------------------------------------------------------- */
/* Latency of the C-ABI call: runs mn_find_neighbors_both `reps` times back to back (after 2
 * warm-up calls) with the default allocator (cudaMallocAsync on `stream`; the current device's
 * default pool is set to keep freed blocks) and reports the median (and minimum) host wall time
 * per call in microseconds — from entry until `stream` has finished the call's last kernel (the
 * call itself returns with the node compaction still queued), the one blocking read included.
 * Outputs are released after each call. */
mn_status mn_time_both(mn_elem_type type, const int32_t* d_conn, int64_t num_elems, int64_t num_nodes, int reps,
                       mn_stream stream, double* median_us, double* min_us);

/* Count of kernels this library has launched since load. */
int64_t mn_launch_count(void);
/* When enabled, every kernel launch is bracketed by CUDA events on its stream. */
void mn_profile_enable(int on);
void mn_profile_reset(void);
/* Synchronises the recorded events and returns the number of distinct kernel names. */
int mn_profile_collect(void);
/* Entry i of the collected table: kernel name, launches, total device ms, algorithmic bytes
 * (sum over launches of the bytes the stage must move by definition, DESIGN.md §"Roofline"). */
mn_status mn_profile_entry(int i, const char** name, int64_t* launches, double* total_ms,
                           double* alg_bytes);

/* ------------------------------------------------------------------------------------------ *
 * Mesh ingestion (host; SURVEY.md §8(f) row 3 "OFF/OBJ ingestion"; SPEC.md mesh-io load_off /
 * load_obj; rules in csrc/meshio.cu and DESIGN.md R19).  The file image (bytes, len)
 * is parsed into the polygon CSR form of mn_find_poly_neighbors, in host memory owned by the
 * library (release with mn_host_mesh_free).  Vertex coordinates are checked to be numeric and
 * dropped (topology only).  The result is validated (R18); every failure is a typed status with
 * detail (line, token) for format errors and (face, position) for validation errors; the output
 * is zeroed on failure.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  int64_t num_nodes;      /* vertex count                                                 */
  int64_t num_elems;      /* face count M                                                 */
  int64_t conn_len;       /* off[M]                                                       */
  int64_t* off;           /* M + 1 ring offsets, off[0] = 0                               */
  int32_t* idx;           /* conn_len 0-based vertex ids                                  */
  int32_t uniform_arity;  /* k if every face has k nodes (3 -> TRI3, 4 -> QUAD4 conn), else 0 */
} mn_host_mesh;

mn_status mn_parse_off(const char* bytes, size_t len, mn_host_mesh* out, mn_error_detail* err);
mn_status mn_parse_obj(const char* bytes, size_t len, mn_host_mesh* out, mn_error_detail* err);
void mn_host_mesh_free(mn_host_mesh* mesh);

#ifdef __cplusplus
}
#endif

#endif /* MESHNBR_H_ */
