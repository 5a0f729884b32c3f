// ft_internal.cuh — shared internals of the B200 Flowtree library (NOT part of the C ABI).
//
// Layouts are described in DESIGN.md §6.  Nothing here is shared with oracle/ (DESIGN.md §4).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/flowtree.h"

// ---------------------------------------------------------------------------------------------
// limits
// ---------------------------------------------------------------------------------------------
#define FTI_MAX_SUPPORT 2048        // max support size of one distribution (doc or query)
#define FTI_MAX_NODE_ENTRIES 8192   // max support * depth entries per distribution
#define FTI_MAX_SELECT 8192         // max k / prefilter_m handled by the selection kernel
#define FTI_PREFILTER_CAP 32768     // candidate-list capacity per query of the fused prefilter
#define FTI_MAX_WEIGHT_TOTAL 65535u // W, U <= 65535 keeps W*U < 2^32
#define FTI_VOCAB_MASK 0x3FFFFFFFu  // vocab ids < 2^30; bits 30/31 of an item word are flags
#define FTI_FLAG_MULTI_LEAF 0x80000000u  // the item's leaf holds >= 2 ground points
#define FTI_FLAG_DEEP 0x40000000u        // some non-root node on the item's path holds >= 2 points
#define FTI_SMALL_D 32              // d <= this: Flowtree prices distances on the fly (no table)
#define FTI_EMPTY 0xFFFFFFFFu

// device-side error bits (sticky, OR-ed into the dataset's mapped error word)
#define FTI_ERR_RANGE 1u
#define FTI_ERR_INVAL 2u
#define FTI_ERR_OVERFLOW 4u
#define FTI_ERR_CAP 8u

// ---------------------------------------------------------------------------------------------
// host-side error reporting
// ---------------------------------------------------------------------------------------------
ft_status fti_fail(ft_status st, const std::string& msg);
#define FTI_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t _e = (call);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return fti_fail(FT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
    } while (0)

// FTI_CHECKED builds (python -m paper_1910_04126_b200.build --checked) add device-side bounds
// assertions on the table gathers and stores, the per-lane queues and the row maps: the stand-in
// for compute-sanitizer, which this pool does not allow
#ifndef FTI_CHECKED
#define FTI_CHECKED 0
#endif
#if FTI_CHECKED
#include <cassert>
#define FTI_ASSERT(c) assert(c)
#else
#define FTI_ASSERT(c) ((void)0)
#endif

// process-wide options set through ft_set_option (include/flowtree.h); 0 = default
int64_t fti_opt(int option);
#define FTI_DBG_DIST 1
#define FTI_DBG_EXACT 2
#define FTI_DBG_SELECT 4
#define FTI_DBG_ALLOC 8
#define FTI_DBG_FLOW_FTD 16   // ft_flowtree_flow: fail unless the lane-per-pair kernel produced the flow

// grow-only device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(size_t b) {
        if (b <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t nb = b < 256 ? 256 : b;
        if (fti_opt(FT_OPT_DEBUG) & FTI_DBG_ALLOC) fprintf(stderr, "ft DevBuf grow -> %zu bytes\n", nb);
        cudaError_t e = cudaMalloc(&p, nb);
        if (e == cudaSuccess) bytes = nb;
        return e;
    }
    template <class T>
    T* as() const { return (T*)p; }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

// ---------------------------------------------------------------------------------------------
// index (a0): the quadtree, device resident
// ---------------------------------------------------------------------------------------------
struct ft_index {
    int64_t N = 0;
    int32_t d = 0;
    int32_t D = 0;        // depth cap
    int32_t d_star = 0;   // realised max leaf depth
    int32_t l_root = 0;
    double phi = 0.0;
    int64_t M = 0;        // nodes
    std::vector<double> sigma, mn;
    std::vector<int64_t> level_base;   // first node id of each depth, size d_star+2
    float* X = nullptr;               // [N*d]
    int32_t* path = nullptr;          // [N*(d_star+1)], -1 below the leaf
    uint8_t* leaf_depth = nullptr;    // [N]
    uint8_t* node_depth = nullptr;    // [M]
    int32_t* node_count = nullptr;    // [M] ground points in the cell
    uint32_t* vflags = nullptr;       // [N] FTI_FLAG_* per ground point
    // distance-table operand (built on first use, ft_dist.cu): the points translated by their FP64
    // mean and quantised to 24-bit fixed point v = rint((x − mean)·2^qexp), stored as three signed
    // 8-bit limbs per coordinate (v = a0 + 2^8 a1 + 2^16 a2), rows [nks][3 limbs][64 bytes] with
    // the coordinates zero padded to 64·nks and one extra all-zero row N; exact int64 norms Σ v²
    int8_t* Xq = nullptr;             // [(N+1) * nks * 192]
    long long* xnq = nullptr;         // [N+1]
    int32_t nks = 0;                  // 64-coordinate K stages
    int32_t qexp = 0;                 // quantisation exponent e
    int device = 0;
};

// ---------------------------------------------------------------------------------------------
// dataset (a1): node-sorted layout in HBM
// ---------------------------------------------------------------------------------------------
struct QueryLayout {           // per-query slot geometry (host computed)
    int32_t smax = 0;          // max support in the batch (rounded)
    int32_t vh_cap = 0;        // vocab hash capacity (pow2)
    int32_t nh_cap = 0;        // node hash capacity (pow2) — QT
    int32_t mh_cap = 0;        // M-node hash capacity (pow2) — FT
    int32_t ml_cap = 0;        // M-node list entries
    size_t off_items = 0, off_vh = 0, off_nh = 0, off_nd = 0, off_mh = 0, off_ml = 0;
    size_t stride = 0;         // bytes per query slot
};

struct QHeader {               // first 64 bytes of a query slot
    uint32_t s;                // support size
    uint32_t U;                // total weight
    unsigned long long B;      // Σ_v ω(v) m_ν(v) over non-root nodes
    uint32_t nh_mask;          // node hash mask (QT)
    uint32_t vh_mask;          // vocab hash mask
    uint32_t mh_mask;          // M-node hash mask (FT)
    uint32_t n_nodes;          // distinct non-root nodes
    uint32_t n_mn;             // M-nodes
    uint32_t n_ml;             // M-node list entries
    uint32_t err;              // FTI_ERR_* bits for this query
    uint32_t pad[5];
};
static_assert(sizeof(QHeader) == 64, "QHeader is 64 bytes");

struct ft_dataset {
    const ft_index* ix = nullptr;
    int64_t n = 0, nnz = 0;
    int32_t max_s = 0;
    int32_t max_mn = 0;        // max M-nodes per doc
    bool unit_w = false;       // every doc weight is 1
    // Flowtree record: items sorted by vocab id {vocab|flags, w}
    uint32_t* doc_off = nullptr;   // [n+1]
    uint2* items = nullptr;        // [nnz]
    uint32_t* W = nullptr;         // [n]
    // M-nodes (nodes holding >= 2 ground points) for the Flowtree phase B
    uint32_t* mn_off = nullptr;    // [n+1]
    uint4* mnodes = nullptr;       // {node, list_off(global), list_len, depth}, per doc (depth desc, node asc)
    uint16_t* mlists = nullptr;    // item indices (vocab order) under each M-node
    int64_t n_mn = 0, n_ml = 0;
    // Quadtree record: non-root nodes sorted by id {node, mass}
    uint32_t* qt_off = nullptr;    // [n+1]
    uint2* qt = nullptr;
    unsigned long long* A = nullptr;  // [n] Σ_v ω(v) m_μ(v)
    int64_t n_qt = 0;
    size_t table_budget = 0;       // a5 table bytes per query chunk (set at the first Flowtree call)
    // sticky device-side error word (FTI_ERR_* bits)
    uint32_t* err_dev = nullptr;
    // per-stage profiling (ft_profile_*)
    bool prof = false;
    struct EvPair { int stage; cudaEvent_t a, b; };
    std::vector<EvPair> prof_pending;
    std::vector<cudaEvent_t> prof_pool;
    double prof_ms[FT_NUM_STAGES] = {0};
    int64_t prof_n[FT_NUM_STAGES] = {0};
    unsigned long long* prof_units = nullptr;   // device [FT_NUM_STAGES] algorithmic bytes per stage
    unsigned long long* units_ptr(int stage) const { return prof ? prof_units + stage : nullptr; }
    // scratch (grow-only; reused across calls)
    DevBuf s_pitch, s_qoff, s_qids, s_qw, s_qblock, s_docs, s_vals, s_vals2, s_cand, s_outid, s_outval;
    DevBuf s_map, s_rows, s_rowcnt, s_table, s_flow, s_flowcnt, s_vlist, s_chunk, s_rowbase, s_bsplit, s_ny, s_tiles, s_qinfo, s_wdesc, s_wrow, s_sel, s_chunkd, s_fblist, s_fbcnt, s_topk;
    // fused prefilter (fti_launch_prefilter): sample doc ids, sample values, thresholds, lists
    DevBuf s_pf_samp, s_pf_sval, s_pf_tval, s_pf_cnt, s_pf_cval, s_pf_cid, s_pf_bad, s_pf_flag;
    DevBuf s_chunkd2;   // Quadtree chunk-pair dense structures (ft_qt.cu)
    DevBuf s_gbase;     // distance-table work list: per-query column-group prefix (ft_dist.cu)
    int64_t pf_ns = -1;
};

// ---------------------------------------------------------------------------------------------
// cross-file launch helpers (host)
// ---------------------------------------------------------------------------------------------
void fti_count_launches(int n);
enum { FTI_ST_PREP = 0, FTI_ST_QT, FTI_ST_SELM, FTI_ST_VMAP, FTI_ST_DIST, FTI_ST_FT, FTI_ST_SELK };
QueryLayout fti_query_layout(const ft_index* ix, int32_t smax);
cudaError_t fti_launch_query_prep(const ft_index* ix, const QueryLayout& L, const int64_t* d_qoff, int32_t nq,
                                  const int32_t* d_qids, const uint32_t* d_qw, uint8_t* d_qblock,
                                  uint32_t* d_err, cudaStream_t st);
// a3 + a4: per query the m smallest (Quadtree value, doc id) over all docs (fused when n ≥ 32·m)
cudaError_t fti_launch_prefilter(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq, int64_t m,
                                 int64_t* d_cand, double* d_cval, int* d_sel_scratch, cudaStream_t st);
cudaError_t fti_launch_qt(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                          const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, double* d_out, int64_t out_ld,
                          cudaStream_t st);
struct FtTable {
    const float* table = nullptr;      // query tables, or null (on-the-fly distances)
    const uint2* map = nullptr;        // [nq][ceil(N/32)] {bits, rank}: row = rank + popc(bits below), or null (row = vocab id)
    const int64_t* row_base = nullptr; // [nq] ELEMENT offset of each query's table
    const int32_t* pitch = nullptr;    // [nq] row pitch (floats) of each query's table
    const int32_t* rowcnt = nullptr;   // [nq] rows of each compact table (null: every vocab id is a row)
    int64_t rows_cap = 0;
};
// lane-per-pair Flowtree with a distance table (ft_flowd.cu), candidate lists or all docs; pairs it
// cannot score are listed per query in *fb_list / *fb_cnt (capacity n_docs per query) for the
// warp kernel's list mode.  Query supports up to FTD_MAX_SQ.
#define FTD_MAX_SQ 254
// With d_flow (the parity hook) it writes the pairs' flow triples {src, dst, η, node} instead of
// pricing them (no table needed).
cudaError_t fti_launch_ftd(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                           const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, const FtTable& tab, double* d_out,
                           int64_t out_ld, uint32_t** fb_list, uint32_t** fb_cnt, cudaStream_t st,
                           uint32_t* d_flow = nullptr, uint32_t* d_flowcnt = nullptr, int32_t flow_cap = 0);
// exact W1 of per-query candidate lists by the transportation simplex (ft_exact.cu)
cudaError_t fti_launch_exact(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                             const int64_t* d_docs, int64_t docs_ld, int64_t n_per_q, double* d_out, int64_t out_ld,
                             cudaStream_t st);
cudaError_t fti_launch_ft(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                          const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, const FtTable& tab,
                          double* d_out, int64_t out_ld, uint32_t* d_flow, uint32_t* d_flowcnt, int32_t flow_cap,
                          cudaStream_t st);
cudaError_t fti_launch_dist_table(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                                  const int32_t* d_rows, const int32_t* d_rowcnt, int64_t rows_cap,
                                  const int64_t* d_row_base, const int32_t* d_pitch, float* d_table, cudaStream_t st);
// the distance-table kernel's shared-memory geometry holds this index's dimension (d ≤ 576)
bool fti_dist_supported(const ft_index* ix);
cudaError_t fti_launch_vocab_map(const ft_dataset* ds, int32_t nq, const int64_t* d_cand, int64_t cand_ld,
                                 int64_t n_cand, uint2* d_map, int32_t* d_rows, int32_t* d_rowcnt, int64_t rows_cap,
                                 cudaStream_t st);
cudaError_t fti_launch_select(const double* d_vals, int64_t vals_ld, const int64_t* d_ids, int64_t ids_ld, int64_t L,
                              int32_t rows, int32_t k, int64_t* d_out_ids, double* d_out_val, int64_t out_ld,
                              int* d_scratch /* rows + 1 ints */, cudaStream_t st, int64_t id_base = 0,
                              const uint32_t* d_row_len = nullptr, const int* d_rows_list = nullptr,
                              const int* d_nrows_list = nullptr, int* d_bad = nullptr, bool nosort = false);
// per row, a value ≥ the r-th smallest (0-based) of L values within FP32 rounding (prefilter threshold)
cudaError_t fti_launch_row_threshold(const double* d_vals, int64_t ld, int64_t L, int32_t rows, int64_t r,
                                     double* d_thr, cudaStream_t st);
