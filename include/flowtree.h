/*
 * flowtree.h — C ABI of the B200-native Flowtree query path (arXiv 1910.04126).
 *
 * Problem (§1): X ⊂ R^d is a finite ground set, μ_1..μ_n are distributions on X
 * with support ≤ s, and ν is a query distribution; find the k μ_i closest to ν in W1 (Eq. (1),
 * PAPER.md:21-26).  The library estimates W1(ν, μ_i) with
 *   - the Quadtree estimate   Σ_v 2^{ℓ(v)} |μ(v) − ν(v)|            (§2), and
 *   - the Flowtree estimate   Σ f(x,x') ||x − x'||, f = tree-optimal flow  (§3;
 *                              greedy bottom-up computation, App. A.1),
 * and ranks with the prefetch-and-prune pipeline Quadtree → top-m → Flowtree → top-k
 * (§4.4).  The readings of the paper that fix every unstated detail
 * (cell rule, node numbering, tie-break, integer masses) are DESIGN.md §3 R1-R18.
 *
 * Conventions (all entry points):
 *   - Every call returns ft_status; FT_OK = 0.  On failure ft_last_error() returns a
 *     thread-local message naming the argument or record at fault.  Nothing is written to the
 *     outputs of a call that fails on the host.
 *   - Distributions are CSR: offsets (int64, n+1, offsets[0] = 0), vocab ids (int32, in
 *     [0, N)) and integer masses (uint32 ≥ 1).  A distribution must be non-empty, have no
 *     duplicate id, and total mass ≤ 65535 (so W·U < 2^32, R13): FT_EINVAL /
 *     FT_ERANGE / FT_EOVERFLOW otherwise.  Estimates are in normalised W1 units (masses summing
 *     to 1), as doubles.
 *   - Build/load inputs are host arrays, copied; the caller keeps ownership.  Index and dataset
 *     are opaque, library-owned and device resident (current CUDA device at creation).  Free a
 *     dataset before its index.  Neither is safe for concurrent calls from several threads.
 *   - Query calls: q_off is a HOST array (the batch shape).  q_ids, q_w, docs and every output
 *     may be host or device pointers (detected with cudaPointerGetAttributes).  If every output
 *     is a device pointer the call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and device-side validation errors of the query payload are reported by
 *     the next ft_synchronize() (sticky); otherwise the call synchronises `stream` before
 *     returning and reports them itself.  Scratch is cached per dataset: no device allocation
 *     after the first call at a given size.
 *   - Limits: support ≤ 2048 per distribution; support × tree depth ≤ 8192; k and prefilter_m
 *     ≤ 8192; N < 2^30; nnz < 2^32.
 */
#ifndef FLOWTREE_H
#define FLOWTREE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FT_OK = 0,
    FT_EINVAL = 1,     /* invalid argument / record (empty, zero mass, duplicate id, bad k) */
    FT_ERANGE = 2,     /* vocab id outside [0, N), or a size limit exceeded */
    FT_EOVERFLOW = 3,  /* total mass > 65535, or a Quadtree numerator ≥ 2^53 */
    FT_ENOMEM = 4,     /* device or host allocation failed */
    FT_ECUDA = 5,      /* CUDA runtime error */
    FT_ESTATE = 6      /* object in an unusable state (e.g. NULL handle) */
} ft_status;

typedef struct ft_index ft_index;
typedef struct ft_dataset ft_dataset;

/* Build the randomly shifted quadtree over X (§2 "Generic Quadtree").
 *   X          host float32 [N × d], row-major; copied to the device.
 *   seed       σ_i = Φ · (SplitMix64(seed, i) >> 11) · 2^-53 (R3).
 *   max_depth  depth cap D (number of halvings), ≤ 0 → 32, must be ≤ 52 (R5).
 * Node ids are breadth first, children ordered by (parent id, child bit-vector, dim 0 first)
 * (R7); cells are half-open (R4); the cell rule is evaluated in FP64 exactly as the
 * oracle does, so the node ids match it bit for bit.  FT_EINVAL if N < 1, d < 1 or D > 52.   */
ft_status ft_build_quadtree(const float* X, int64_t N, int32_t d, uint64_t seed, int32_t max_depth,
                            ft_index** out);
/* Same with an explicit shift σ (host double [d], each in [0, Φ]) — test hook.               */
ft_status ft_build_quadtree_shift(const float* X, int64_t N, int32_t d, const double* sigma,
                                  int32_t max_depth, ft_index** out);
/* Φ (max coordinate range), ℓ_root = ⌈log2 Φ⌉+1, realised depth D*, number of nodes.  Any
 * output pointer may be NULL.                                                                */
ft_status ft_index_info(const ft_index* ix, double* phi, int32_t* l_root, int32_t* d_star, int64_t* n_nodes);
/* Parity hook: host int32 [N × (D*+1)], node id of point x at depth k, −1 below its leaf.      */
ft_status ft_index_paths(const ft_index* ix, int32_t* out);
/* Parity hook: host double [d], the shift σ actually used.                                    */
ft_status ft_index_sigma(const ft_index* ix, double* sigma);
/* Parity hook: host int32 [M] node depths and [M] ground-point counts (either may be NULL).   */
ft_status ft_index_nodes(const ft_index* ix, int32_t* depth, int32_t* count);

/* Load n documents (host CSR, copied) into the node-sorted device layout:
 * a vocab-sorted Flowtree record, the M-node lists, and the node-sorted Quadtree record
 * (the ℓ1 embedding of PAPER.md:131-134).  Errors name the first offending document.         */
ft_status ft_load_dataset(const ft_index* ix, const int64_t* doc_off, int64_t n, const int32_t* ids,
                          const uint32_t* w, ft_dataset** out);
/* n, nnz, number of Quadtree node records, max support.  Any pointer may be NULL.            */
ft_status ft_dataset_info(const ft_dataset* ds, int64_t* n, int64_t* nnz, int64_t* n_qt_records,
                          int32_t* max_support);

/* Quadtree estimates for every (query, doc) pair.
 *   q_off   HOST int64 [nq+1];  q_ids int32 / q_w uint32 [q_off[nq]] (host or device).
 *   docs    int64 [n_docs] doc indices, or NULL for all n docs (then n_docs is ignored).
 *   out     double [nq × n_docs] row-major (host or device).
 * Values are bit-identical to the oracle (exact integer numerator, two correctly rounded ops). */
ft_status ft_quadtree_estimate(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                               const uint32_t* q_w, const int64_t* docs, int64_t n_docs, double* out,
                               void* stream);
/* Flowtree estimates with the same signature.  The flow is integer exact.
 * Distances: for d ≤ 32 FP32 direct differences; for d > 32 a tensor-core table in exact integer
 * arithmetic on the points quantised to 24-bit fixed point (unit 2^-e, e the largest exponent with
 * max|x − mean|·2^e ≤ 2^23 − 2^16): |error| ≤ sqrt(d)·2^-e absolute plus ≈2^-22 relative, and
 * identical coordinates give exactly 0.  Accumulation FP64 across batches.  Tolerance of the
 * estimate: 1e-5 relative.  With candidate lists the call reads the per-query
 * table sizes back once (one stream synchronisation) before the distance stage.               */
ft_status ft_flowtree_estimate(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                               const uint32_t* q_w, const int64_t* docs, int64_t n_docs, double* out,
                               void* stream);
/* Parity hook: the Flowtree flow of one (query, doc) pair, HOST outputs, in canonical order
 * (node depth desc, node id asc, src asc, dst asc) — the oracle's emission order.  The flow comes
 * from the kernel that scores the pair in ft_knn / ft_flowtree_estimate: for d > 32 the
 * lane-per-pair kernel (k_ftd) unless the pair has a matching multi-point cell, else the warp
 * kernel (k_flowtree).
 *   src = doc vocab id, dst = query vocab id, mass in units of 1/(W·U), node where matched.
 *   FT_ERANGE if more than cap triples (n_out still receives the count).                     */
ft_status ft_flowtree_flow(const ft_dataset* ds, int32_t q_len, const int32_t* q_ids, const uint32_t* q_w,
                           int64_t doc, int32_t* src, int32_t* dst, uint64_t* mass, int32_t* node, int32_t cap,
                           int32_t* n_out);
/* k-NN: for each query the k docs with the smallest Flowtree estimate, ties by
 * doc id.  prefilter_m == 0 or ≥ n: exhaustive Flowtree; else Quadtree over all docs, keep
 * the m smallest (value, id), Flowtree on those, keep k.  FT_EINVAL if
 * k < 1 or 0 < prefilter_m < k.  If fewer than k candidates, pads with id −1 / value +inf.
 *   out_ids int64 [nq × k], out_val double [nq × k] (host or device).                        */
ft_status ft_knn(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                 const uint32_t* q_w, int32_t k, int64_t prefilter_m, int64_t* out_ids, double* out_val,
                 void* stream);
/* Doc-sharded k-NN building blocks: with the docs split across ranks, each rank
 * keeps its local top-m Quadtree candidates, the ranks exchange (value, global id) lists, merge
 * them with ft_topk, and each rank scores the merged candidates it owns with
 * ft_flowtree_estimate_lists; the result is identical to ft_knn on the whole collection.
 *
 * ft_topk: per row, the k smallest (value, id) pairs, ties by id, in ascending order — the
 * selection of ft_knn (reading R14).  DEVICE pointers only (FT_EINVAL else).
 *   vals double [rows × vals_ld] (L used per row; NaN sorts last);
 *   ids  int64 [rows × ids_ld], or NULL: the id of column c is id_base + c;
 *   out_ids int64 / out_val double [rows × k]; rows with fewer than k entries pad with −1 / +inf.
 * Asynchronous on `stream`.                                                                  */
ft_status ft_topk(const double* vals, int64_t vals_ld, const int64_t* ids, int64_t ids_ld, int64_t id_base,
                  int64_t L, int32_t rows, int32_t k, int64_t* out_ids, double* out_val, void* stream);
/* Flowtree estimates of per-query candidate lists:
 *   docs  int64 [nq × docs_ld] DEVICE: the first n_per_q entries of row q are doc indices of
 *         this dataset; a negative entry is skipped and scores +inf (so per-shard results
 *         combine with a MIN reduction); an index ≥ n scores NaN and sets FT_ERANGE.
 *   out   double [nq × n_per_q] DEVICE.  q_off is HOST; q_ids / q_w host or device.          */
ft_status ft_flowtree_estimate_lists(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                                     const uint32_t* q_w, const int64_t* docs, int64_t docs_ld, int64_t n_per_q,
                                     double* out, void* stream);
/* Exact W1 (Eq. (1)) of per-query candidate lists — the last stage of the
 * paper's Quadtree → Flowtree → Exact pipelines: the transportation simplex
 * on the cross-scaled integer masses, FP32 Euclidean costs, FP64 objective, one CTA per pair.
 * Same layout as ft_flowtree_estimate_lists (DEVICE docs [nq × docs_ld], out [nq × n_per_q];
 * negative entries score +inf).  Supports up to m + n ≤ 511 points whose m·n FP32 costs fit one CTA's shared memory (larger pairs:
 * NaN + FT_ERANGE via ft_synchronize); a pivot cap guards against cycling (NaN likewise).     */
ft_status ft_exact_w1_lists(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                            const uint32_t* q_w, const int64_t* docs, int64_t docs_ld, int64_t n_per_q, double* out,
                            void* stream);
/* Synchronise `stream` and report (then clear) any sticky device-side validation error.      */
ft_status ft_synchronize(const ft_dataset* ds, void* stream);

/* Diagnostics (used by bench.py for the live roofline numbers).  With profiling enabled, the
 * query calls on `ds` record a CUDA event pair around every stage on the call's stream; reading
 * synchronises the events and returns, per stage, the total device milliseconds and the number
 * of timed launches since the last reset.  Stages: 0 query prep (a2), 1 Quadtree (a3),
 * 2 top-m select (a4), 3 candidate vocabulary (a5 prep), 4 distance table (a5), 5 Flowtree (a6),
 * 6 top-k select (a7).  ft_launch_count() is the number of kernels this library has launched
 * in the process so far.                                                                      */
#define FT_NUM_STAGES 7
ft_status ft_profile_enable(ft_dataset* ds, int32_t enable);
ft_status ft_profile_reset(ft_dataset* ds);
ft_status ft_profile_read(ft_dataset* ds, int32_t stage, double* total_ms, int64_t* launches);
/* Algorithmic bytes the kernels of a stage moved since the last reset (SURVEY §8(d) units),
 * counted on the device while profiling is enabled: stage 4 (distance table) Σ rows·(4d + 4 s_q),
 * stage 5 (Flowtree) Σ pairs·(8 s_doc + 16).  The extra slot FT_PROF_DIST_FLOPS holds the
 * distance table's algorithmic flops Σ 2·rows·s_q·d (one product per entry; the
 * 3xTF32 kernel executes three).  Synchronises the device.                                     */
#define FT_PROF_DIST_FLOPS FT_NUM_STAGES
ft_status ft_profile_units(ft_dataset* ds, int32_t stage, uint64_t* bytes);
const char* ft_profile_stage_name(int32_t stage);
uint64_t ft_launch_count(void);

/* Process-wide tuning and test options (not part of the method; the defaults are the product
 * configuration).  Each is read by the library on every call that uses it; nothing is read from
 * the environment.  FT_EINVAL for an unknown option or a value out of range.
 *   FT_OPT_VOCAB_HASH      1: the warp Flowtree kernel looks vocab ids up in the query's hash
 *                          instead of the shared-memory bitmap (the path taken when N > 2^19).
 *   FT_OPT_WARP_ONLY       1: every Flowtree pair runs on the warp kernel (k_flowtree), not the
 *                          lane-per-pair kernel (k_ftd).
 *   FT_OPT_QT_HASH         1: the Quadtree scan uses the hash chunk structure, not the dense one.
 *   FT_OPT_SELECT_RADIX    1: selection uses the radix kernel for every row.
 *   FT_OPT_EXACT_START_NW  1: the exact-W1 simplex starts from the northwest corner.
 *   FT_OPT_TABLE_CHUNK     > 0: at most this many queries per distance-table chunk.
 *   FT_OPT_TABLE_BUDGET_MB > 0: distance-table bytes per chunk (default: 1/4 of free HBM at the
 *                          dataset's first Flowtree call, at most 48 GB).
 *   FT_OPT_QT_WAVES        > 0: CTA waves per SM slot of the Quadtree launch (default 4).
 *   FT_OPT_FTD_CARVEOUT    1..100: k_ftd shared-memory carveout percent (0: sized for the kernel's CTAs per SM: 3, or 2 with compact tables).
 *   FT_OPT_PREFILTER_UNFUSED 1: ft_knn's prefilter writes every Quadtree value and then selects
 *                          (the fused sample-threshold scan is the default when n ≥ 32·m).
 *   FT_OPT_QT_PAIR_OFF     1: the Quadtree scan serves 32 queries per record pass (no chunk pairs).
 *   FT_OPT_DIST_QMAJOR     1: exhaustive distance tables are built query by query (not tile-major
 *                          with the A tile shared by consecutive work items).
 *   FT_OPT_DEBUG           bit mask of diagnostics printed to stderr: 1 distance-table role
 *                          clocks, 2 exact-W1 pivots, 4 selection paths, 8 scratch growth; and
 *                          16: ft_flowtree_flow fails (FT_ESTATE) unless the lane-per-pair kernel
 *                          (the one scoring the pair in ft_knn) produced the flow.               */
typedef enum {
    FT_OPT_VOCAB_HASH = 0,
    FT_OPT_WARP_ONLY = 1,
    FT_OPT_QT_HASH = 2,
    FT_OPT_SELECT_RADIX = 3,
    FT_OPT_EXACT_START_NW = 4,
    FT_OPT_TABLE_CHUNK = 5,
    FT_OPT_TABLE_BUDGET_MB = 6,
    FT_OPT_QT_WAVES = 7,
    FT_OPT_FTD_CARVEOUT = 8,
    FT_OPT_DEBUG = 9,
    FT_OPT_PREFILTER_UNFUSED = 10,
    FT_OPT_QT_PAIR_OFF = 11,
    FT_OPT_DIST_QMAJOR = 12,
    FT_NUM_OPTIONS = 13
} ft_option;
ft_status ft_set_option(int32_t option, int64_t value);
ft_status ft_get_option(int32_t option, int64_t* value);

void ft_index_free(ft_index* ix);
void ft_dataset_free(ft_dataset* ds);
/* Thread-local message of the last failing call on this thread ("" if none).                 */
const char* ft_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FLOWTREE_H */
