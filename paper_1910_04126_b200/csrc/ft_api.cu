// ft_api.cu — the C ABI query entry points (include/flowtree.h): argument validation, host/device
// pointer handling, scratch management and the stage sequence of the hot path
//   a2 query prep → a3 Quadtree → a4 top-m → a5 distance table → a6 Flowtree → a7 top-k.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ft_device.cuh"

#include <atomic>

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

ft_status fti_fail(ft_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

void fti_count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

extern "C" const char* ft_last_error(void) { return g_last_error.c_str(); }
extern "C" uint64_t ft_launch_count(void) { return g_launches.load(); }

static std::atomic<int64_t> g_opts[FT_NUM_OPTIONS];

int64_t fti_opt(int option) { return g_opts[option].load(std::memory_order_relaxed); }

extern "C" ft_status ft_set_option(int32_t option, int64_t value) {
    if (option < 0 || option >= FT_NUM_OPTIONS) return fti_fail(FT_EINVAL, "ft_set_option: unknown option");
    if (value < 0) return fti_fail(FT_EINVAL, "ft_set_option: negative value");
    if (option == FT_OPT_FTD_CARVEOUT && value > 100) return fti_fail(FT_EINVAL, "ft_set_option: carveout > 100");
    g_opts[option].store(value, std::memory_order_relaxed);
    return FT_OK;
}

extern "C" ft_status ft_get_option(int32_t option, int64_t* value) {
    if (option < 0 || option >= FT_NUM_OPTIONS || !value) return fti_fail(FT_EINVAL, "ft_get_option: bad argument");
    *value = g_opts[option].load(std::memory_order_relaxed);
    return FT_OK;
}

namespace {

// records a CUDA event pair around one stage when profiling is enabled on the dataset
struct StageTimer {
    ft_dataset* ds;
    int stage;
    cudaStream_t st;
    cudaEvent_t b = nullptr;
    StageTimer(ft_dataset* d, int s, cudaStream_t t) : ds(d), stage(s), st(t) {
        if (!ds->prof) return;
        cudaEvent_t a = take();
        b = take();
        cudaEventRecord(a, st);
        ds->prof_pending.push_back({stage, a, b});
    }
    ~StageTimer() {
        if (b) cudaEventRecord(b, st);
    }
    cudaEvent_t take() {
        if (!ds->prof_pool.empty()) {
            cudaEvent_t e = ds->prof_pool.back();
            ds->prof_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

#define FTI_RES(buf, bytes)                                                                     \
    do {                                                                                        \
        cudaError_t _e = (buf).reserve(bytes);                                                  \
        if (_e != cudaSuccess) return fti_fail(FT_ENOMEM, std::string("scratch allocation: ") + \
                                                              cudaGetErrorString(_e));          \
    } while (0)

// a Flowtree launch; cudaErrorInvalidConfiguration means the supports do not fit the kernels'
// shared-memory geometry (a size limit, FT_ERANGE)
#define FTI_FT(call)                                                                                       \
    do {                                                                                                   \
        cudaError_t _e = (call);                                                                           \
        if (_e == cudaErrorInvalidConfiguration)                                                           \
            return fti_fail(FT_ERANGE, "Flowtree: doc/query supports too large for the kernel geometry");  \
        if (_e != cudaSuccess) return fti_fail(FT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// device error word (sticky) -> status
ft_status check_device_errors(const ft_dataset* ds, cudaStream_t st, const char* who) {
    uint32_t h = 0;
    FTI_CUDA(cudaMemcpyAsync(&h, ds->err_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    FTI_CUDA(cudaStreamSynchronize(st));
    if (h == 0) return FT_OK;
    FTI_CUDA(cudaMemsetAsync(ds->err_dev, 0, sizeof(uint32_t), st));
    FTI_CUDA(cudaStreamSynchronize(st));
    std::string w = std::string(who) + ": device-side validation failed: ";
    if (h & FTI_ERR_RANGE) return fti_fail(FT_ERANGE, w + "vocab or doc id out of range");
    if (h & FTI_ERR_OVERFLOW) return fti_fail(FT_EOVERFLOW, w + "total mass > 65535 or Quadtree numerator >= 2^53");
    return fti_fail(FT_EINVAL, w + "empty query, zero mass or duplicate vocab id");
}

struct Staged {
    QueryLayout L;
    const int32_t* qids = nullptr;
    const uint32_t* qw = nullptr;
    const int64_t* qoff_dev = nullptr;
    const int64_t* qoff_host = nullptr;
    uint8_t* qblock = nullptr;
};

// validate the batch shape (host q_off) and, for host payloads, the payload itself; stage to the
// device; run the a2 prep kernel.
ft_status stage_queries(ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids, const uint32_t* q_w,
                        cudaStream_t st, const char* who, Staged& S) {
    const ft_index* ix = ds->ix;
    if (!q_off || !q_ids || !q_w) return fti_fail(FT_EINVAL, std::string(who) + ": NULL query array");
    if (nq < 1) return fti_fail(FT_EINVAL, std::string(who) + ": need nq >= 1");
    if (is_device_ptr(q_off)) return fti_fail(FT_EINVAL, std::string(who) + ": q_off must be a host array");
    if (q_off[0] != 0) return fti_fail(FT_EINVAL, std::string(who) + ": q_off[0] must be 0");
    int32_t smax = 0;
    for (int32_t q = 0; q < nq; q++) {
        int64_t s = q_off[q + 1] - q_off[q];
        if (s < 1) return fti_fail(FT_EINVAL, std::string(who) + ": query " + std::to_string(q) + " is empty");
        if (s > FTI_MAX_SUPPORT)
            return fti_fail(FT_ERANGE, std::string(who) + ": query " + std::to_string(q) + " has support > 2048");
        smax = std::max<int32_t>(smax, (int32_t)s);
    }
    if ((int64_t)smax * std::max(1, ix->d_star) > FTI_MAX_NODE_ENTRIES)
        return fti_fail(FT_ERANGE, std::string(who) + ": query support x tree depth exceeds 8192 entries");
    const int64_t nnz = q_off[nq];
    const bool dev_ids = is_device_ptr(q_ids), dev_w = is_device_ptr(q_w);
    if (!dev_ids && !dev_w) {
        // full host validation with precise messages
        std::vector<int32_t> tmp;
        for (int32_t q = 0; q < nq; q++) {
            uint64_t U = 0;
            tmp.assign(q_ids + q_off[q], q_ids + q_off[q + 1]);
            for (int64_t t = q_off[q]; t < q_off[q + 1]; t++) {
                if (q_ids[t] < 0 || (int64_t)q_ids[t] >= ix->N)
                    return fti_fail(FT_ERANGE, std::string(who) + ": query " + std::to_string(q) + ": vocab id " +
                                                   std::to_string(q_ids[t]) + " outside [0, N)");
                if (q_w[t] == 0)
                    return fti_fail(FT_EINVAL, std::string(who) + ": query " + std::to_string(q) + ": zero mass");
                U += q_w[t];
            }
            if (U > FTI_MAX_WEIGHT_TOTAL)
                return fti_fail(FT_EOVERFLOW, std::string(who) + ": query " + std::to_string(q) + ": total mass > 65535");
            std::sort(tmp.begin(), tmp.end());
            if (std::adjacent_find(tmp.begin(), tmp.end()) != tmp.end())
                return fti_fail(FT_EINVAL, std::string(who) + ": query " + std::to_string(q) + ": duplicate vocab id");
        }
    }
    S.L = fti_query_layout(ix, smax);
    S.qoff_host = q_off;
    FTI_RES(ds->s_qoff, sizeof(int64_t) * (nq + 1));
    FTI_CUDA(cudaMemcpyAsync(ds->s_qoff.p, q_off, sizeof(int64_t) * (nq + 1), cudaMemcpyHostToDevice, st));
    S.qoff_dev = ds->s_qoff.as<int64_t>();
    if (dev_ids) S.qids = q_ids;
    else {
        FTI_RES(ds->s_qids, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
        FTI_CUDA(cudaMemcpyAsync(ds->s_qids.p, q_ids, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
        S.qids = ds->s_qids.as<int32_t>();
    }
    if (dev_w) S.qw = q_w;
    else {
        FTI_RES(ds->s_qw, sizeof(uint32_t) * std::max<int64_t>(nnz, 1));
        FTI_CUDA(cudaMemcpyAsync(ds->s_qw.p, q_w, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, st));
        S.qw = ds->s_qw.as<uint32_t>();
    }
    FTI_RES(ds->s_qblock, S.L.stride * (size_t)nq);
    S.qblock = ds->s_qblock.as<uint8_t>();
    StageTimer tm(ds, FTI_ST_PREP, st);
    FTI_CUDA(fti_launch_query_prep(ix, S.L, S.qoff_dev, nq, S.qids, S.qw, S.qblock, ds->err_dev, st));
    return FT_OK;
}

// docs argument: NULL = all; host arrays are validated and copied; device arrays are checked in-kernel.
ft_status stage_docs(ft_dataset* ds, const int64_t* docs, int64_t n_docs, cudaStream_t st, const char* who,
                     const int64_t** out, int64_t* n_out) {
    if (!docs) {
        *out = nullptr;
        *n_out = ds->n;
        return FT_OK;
    }
    if (n_docs < 1) return fti_fail(FT_EINVAL, std::string(who) + ": need n_docs >= 1");
    if (is_device_ptr(docs)) {
        *out = docs;
        *n_out = n_docs;
        return FT_OK;
    }
    for (int64_t i = 0; i < n_docs; i++)
        if (docs[i] < 0 || docs[i] >= ds->n)
            return fti_fail(FT_ERANGE, std::string(who) + ": docs[" + std::to_string(i) + "] outside [0, n)");
    FTI_RES(ds->s_docs, sizeof(int64_t) * n_docs);
    FTI_CUDA(cudaMemcpyAsync(ds->s_docs.p, docs, sizeof(int64_t) * n_docs, cudaMemcpyHostToDevice, st));
    *out = ds->s_docs.as<int64_t>();
    *n_out = n_docs;
    return FT_OK;
}

// the Flowtree stage prices from a distance table (d beyond the on-the-fly limit, within the table
// kernel's geometry)
bool ix_uses_table(const ft_index* ix) { return ix->d > FTI_SMALL_D && fti_dist_supported(ix); }

// a5 + a6 over a query batch, chunked so the distance tables stay within a memory budget.
ft_status flowtree_stage(ft_dataset* ds, const Staged& S, int32_t nq, const int64_t* d_docs, int64_t docs_ld,
                         int64_t n_docs, double* d_out, int64_t out_ld, cudaStream_t st) {
    const ft_index* ix = ds->ix;
    if (!ix_uses_table(ix)) {
        // small d: distances on the fly from shared memory; d beyond the distance-table kernel's
        // shared-memory geometry (> 576): on the fly from global memory (slow, any d)
        StageTimer tm(ds, FTI_ST_FT, st);
        FTI_FT(fti_launch_ft(ds, S.L, S.qblock, nq, d_docs, docs_ld, n_docs, FtTable{}, d_out, out_ld, nullptr,
                             nullptr, 0, st));
        return FT_OK;
    }
    // the budget is fixed at the dataset's first Flowtree call: cudaMemGetInfo on every call showed
    // as occasional multi-ms host stalls, and a stable budget keeps the allocation from changing
    if (ds->table_budget == 0) {
        size_t fr = 0, tot = 0;
        ds->table_budget = (size_t)3 << 30;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
            ds->table_budget = std::max(ds->table_budget, std::min(fr / 4, (size_t)48 << 30));
    }
    size_t budget = ds->table_budget;
    if (fti_opt(FT_OPT_TABLE_BUDGET_MB) > 0) budget = (size_t)fti_opt(FT_OPT_TABLE_BUDGET_MB) << 20;
    const int64_t qcap = fti_opt(FT_OPT_TABLE_CHUNK) > 0 ? fti_opt(FT_OPT_TABLE_CHUNK) : (int64_t)nq;
    // per query: table rows, row pitch (floats) and ELEMENT offset within its chunk.  (A
    // column-major table — the distance kernel's lanes storing whole 128-byte column segments —
    // was measured: distance table 4.46 → 4.82 ms, Flowtree 0.75 → 0.68 ms; not kept.)  With candidate
    // lists the rows are the candidates' vocabulary (compact, counted on the device by k_vocab and
    // read back once: the tables are then sized exactly); exhaustively every vocab id is a row.
    const bool use_map = d_docs != nullptr;
    const int64_t rows_cap = use_map ? std::min<int64_t>(ix->N, n_docs * (int64_t)ds->max_s) : ix->N;
    const size_t nwords = (size_t)(ix->N + 31) / 32;
    std::vector<int32_t> rowcnt((size_t)nq, (int32_t)ix->N);
    if (use_map) {
        FTI_RES(ds->s_map, (size_t)nq * nwords * 8);
        FTI_RES(ds->s_rows, (size_t)nq * rows_cap * 4);
        FTI_RES(ds->s_rowcnt, (size_t)nq * 4);
        StageTimer tm(ds, FTI_ST_VMAP, st);
        FTI_CUDA(fti_launch_vocab_map(ds, nq, d_docs, docs_ld, n_docs, ds->s_map.as<uint2>(), ds->s_rows.as<int32_t>(),
                                      ds->s_rowcnt.as<int32_t>(), rows_cap, st));
        FTI_CUDA(cudaMemcpyAsync(rowcnt.data(), ds->s_rowcnt.p, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
        FTI_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<int64_t> base((size_t)nq);
    std::vector<int32_t> pitch((size_t)nq);
    std::vector<int32_t> chunk_q0;       // first query of each chunk
    size_t chunk_max = 0, cur = 0;
    int64_t in_chunk = 0;
    for (int32_t q = 0; q < nq; q++) {
        const int64_t s = S.qoff_host[q + 1] - S.qoff_host[q];
        pitch[q] = (int32_t)((s + 7) & ~7);          // 32-byte rows
        if ((uint64_t)rowcnt[q] * (uint64_t)pitch[q] >= (1ull << 32))
            return fti_fail(FT_ERANGE, "Flowtree: a query's distance table exceeds 2^32 entries (N x support)");
        const size_t bytes = (size_t)rowcnt[q] * (size_t)pitch[q] * 4;
        if (q == 0 || in_chunk >= qcap || (cur > 0 && cur + bytes > budget)) {
            chunk_q0.push_back(q);
            cur = 0;
            in_chunk = 0;
        }
        base[q] = (int64_t)(cur / 4);
        cur += bytes;
        in_chunk++;
        chunk_max = std::max(chunk_max, cur);
    }
    chunk_q0.push_back(nq);
    FTI_RES(ds->s_table, std::max<size_t>(chunk_max, 4));
    FTI_RES(ds->s_rowbase, (size_t)nq * 8);
    FTI_RES(ds->s_pitch, (size_t)nq * 4);
    FTI_CUDA(cudaMemcpyAsync(ds->s_rowbase.p, base.data(), (size_t)nq * 8, cudaMemcpyHostToDevice, st));
    FTI_CUDA(cudaMemcpyAsync(ds->s_pitch.p, pitch.data(), (size_t)nq * 4, cudaMemcpyHostToDevice, st));
    for (size_t c = 0; c + 1 < chunk_q0.size(); c++) {
        const int32_t q0 = chunk_q0[c], nqc = chunk_q0[c + 1] - q0;
        const uint8_t* qb = S.qblock + (size_t)q0 * S.L.stride;
        const int64_t* dq = d_docs ? d_docs + (int64_t)q0 * docs_ld : nullptr;
        const int32_t* rows_c = use_map ? ds->s_rows.as<int32_t>() + (int64_t)q0 * rows_cap : nullptr;
        const int32_t* rowcnt_c = use_map ? ds->s_rowcnt.as<int32_t>() + q0 : nullptr;
        FtTable tab;
        tab.table = ds->s_table.as<float>();
        tab.rows_cap = rows_cap;
        tab.row_base = ds->s_rowbase.as<int64_t>() + q0;
        tab.pitch = ds->s_pitch.as<int32_t>() + q0;
        if (use_map) {
            tab.map = ds->s_map.as<uint2>() + (int64_t)q0 * nwords;
            tab.rowcnt = rowcnt_c;
        }
        {
            StageTimer tm(ds, FTI_ST_DIST, st);
            FTI_CUDA(fti_launch_dist_table(ds, S.L, qb, nqc, rows_c, rowcnt_c, rows_cap, tab.row_base, tab.pitch,
                                           ds->s_table.as<float>(), st));
        }
        StageTimer tm(ds, FTI_ST_FT, st);
        FTI_FT(fti_launch_ft(ds, S.L, qb, nqc, dq, docs_ld, n_docs, tab, d_out + (int64_t)q0 * out_ld, out_ld,
                             nullptr, nullptr, 0, st));
    }
    return FT_OK;
}

ft_status estimate_common(const ft_dataset* cds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                          const uint32_t* q_w, const int64_t* docs, int64_t n_docs, double* out, void* stream,
                          bool flowtree, const char* who) {
    if (!cds) return fti_fail(FT_ESTATE, std::string(who) + ": NULL dataset");
    if (!out) return fti_fail(FT_EINVAL, std::string(who) + ": out is NULL");
    ft_dataset* ds = const_cast<ft_dataset*>(cds);
    cudaStream_t st = (cudaStream_t)stream;
    Staged S;
    ft_status rc = stage_queries(ds, q_off, nq, q_ids, q_w, st, who, S);
    if (rc) return rc;
    const int64_t* d_docs;
    int64_t nd;
    rc = stage_docs(ds, docs, n_docs, st, who, &d_docs, &nd);
    if (rc) return rc;
    const bool dev_out = is_device_ptr(out);
    double* d_out = out;
    if (!dev_out) {
        FTI_RES(ds->s_vals, sizeof(double) * nq * nd);
        d_out = ds->s_vals.as<double>();
    }
    if (flowtree) {
        rc = flowtree_stage(ds, S, nq, d_docs, 0, nd, d_out, nd, st);
        if (rc) return rc;
    } else {
        StageTimer tm(ds, FTI_ST_QT, st);
        FTI_CUDA(fti_launch_qt(ds, S.L, S.qblock, nq, d_docs, 0, nd, d_out, nd, st));
    }
    if (!dev_out) {
        FTI_CUDA(cudaMemcpyAsync(out, d_out, sizeof(double) * nq * nd, cudaMemcpyDeviceToHost, st));
        return check_device_errors(ds, st, who);
    }
    return FT_OK;
}

}  // namespace

extern "C" ft_status ft_quadtree_estimate(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                                          const uint32_t* q_w, const int64_t* docs, int64_t n_docs, double* out,
                                          void* stream) {
    return estimate_common(ds, q_off, nq, q_ids, q_w, docs, n_docs, out, stream, false, "ft_quadtree_estimate");
}

extern "C" ft_status ft_flowtree_estimate(const ft_dataset* ds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                                          const uint32_t* q_w, const int64_t* docs, int64_t n_docs, double* out,
                                          void* stream) {
    return estimate_common(ds, q_off, nq, q_ids, q_w, docs, n_docs, out, stream, true, "ft_flowtree_estimate");
}

extern "C" ft_status ft_flowtree_flow(const ft_dataset* cds, int32_t q_len, const int32_t* q_ids, const uint32_t* q_w,
                                      int64_t doc, int32_t* src, int32_t* dst, uint64_t* mass, int32_t* node,
                                      int32_t cap, int32_t* n_out) {
    const char* who = "ft_flowtree_flow";
    if (!cds) return fti_fail(FT_ESTATE, "ft_flowtree_flow: NULL dataset");
    ft_dataset* ds = const_cast<ft_dataset*>(cds);
    if (doc < 0 || doc >= ds->n) return fti_fail(FT_ERANGE, "ft_flowtree_flow: doc outside [0, n)");
    if (cap < 0 || !n_out) return fti_fail(FT_EINVAL, "ft_flowtree_flow: bad cap / n_out");
    cudaStream_t st = 0;
    int64_t q_off[2] = {0, q_len};
    Staged S;
    ft_status rc = stage_queries(ds, q_off, 1, q_ids, q_w, st, who, S);
    if (rc) return rc;
    int64_t ndoc = doc;
    FTI_RES(ds->s_docs, sizeof(int64_t));
    FTI_CUDA(cudaMemcpyAsync(ds->s_docs.p, &ndoc, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    const int32_t fcap = ds->max_s + q_len + 8;
    FTI_RES(ds->s_flow, sizeof(uint32_t) * 4 * fcap);
    FTI_RES(ds->s_flowcnt, sizeof(uint32_t));
    FTI_CUDA(cudaMemsetAsync(ds->s_flowcnt.p, 0, sizeof(uint32_t), st));
    FTI_RES(ds->s_vals, sizeof(double));
    // the kernel that scores the pair in the product path exports it: with a distance table
    // (d > 32) that is the lane-per-pair kernel unless the pair has a matching M-node (or too many
    // shared ids), which it hands to the warp kernel
    bool done = false;
    if (ix_uses_table(ds->ix) && !fti_opt(FT_OPT_WARP_ONLY)) {
        uint32_t* fl = nullptr;
        uint32_t* fc = nullptr;
        const cudaError_t e = fti_launch_ftd(ds, S.L, S.qblock, 1, ds->s_docs.as<int64_t>(), 0, 1, FtTable{},
                                             ds->s_vals.as<double>(), 1, &fl, &fc, st, ds->s_flow.as<uint32_t>(),
                                             ds->s_flowcnt.as<uint32_t>(), fcap);
        if (e != cudaSuccess && e != cudaErrorNotSupported) FTI_CUDA(e);
        if (e == cudaSuccess) {
            uint32_t handed = 0;
            FTI_CUDA(cudaMemcpyAsync(&handed, fc, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            FTI_CUDA(cudaStreamSynchronize(st));
            done = handed == 0;
        }
    }
    if (!done && (fti_opt(FT_OPT_DEBUG) & FTI_DBG_FLOW_FTD))
        return fti_fail(FT_ESTATE, "ft_flowtree_flow: the pair is not scored by the lane-per-pair kernel");
    if (!done) {
        FTI_CUDA(cudaMemsetAsync(ds->s_flowcnt.p, 0, sizeof(uint32_t), st));
        FTI_FT(fti_launch_ft(ds, S.L, S.qblock, 1, ds->s_docs.as<int64_t>(), 0, 1, FtTable{}, ds->s_vals.as<double>(),
                             1, ds->s_flow.as<uint32_t>(), ds->s_flowcnt.as<uint32_t>(), fcap, st));
    }
    uint32_t cnt = 0;
    FTI_CUDA(cudaMemcpyAsync(&cnt, ds->s_flowcnt.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    rc = check_device_errors(ds, st, who);
    if (rc) return rc;
    const uint32_t nget = std::min<uint32_t>(cnt, (uint32_t)fcap);
    std::vector<uint32_t> f(4 * (size_t)nget);
    FTI_CUDA(cudaMemcpy(f.data(), ds->s_flow.p, sizeof(uint32_t) * 4 * nget, cudaMemcpyDeviceToHost));
    // canonical order (depth desc, node asc, src asc, dst asc) = the oracle's emission order
    const ft_index* ix = ds->ix;
    auto depth_of = [&](uint32_t v) {
        int k = (int)(std::upper_bound(ix->level_base.begin(), ix->level_base.end(), (int64_t)v) -
                      ix->level_base.begin()) - 1;
        return k;
    };
    std::vector<uint32_t> ord(nget);
    for (uint32_t i = 0; i < nget; i++) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
        int da = depth_of(f[4 * a + 3]), db = depth_of(f[4 * b + 3]);
        if (da != db) return da > db;
        for (int t : {3, 0, 1})
            if (f[4 * a + t] != f[4 * b + t]) return f[4 * a + t] < f[4 * b + t];
        return false;
    });
    *n_out = (int32_t)cnt;
    if ((int32_t)cnt > cap) return fti_fail(FT_ERANGE, "ft_flowtree_flow: more triples than cap");
    for (uint32_t i = 0; i < nget; i++) {
        const uint32_t* t = &f[4 * ord[i]];
        if (src) src[i] = (int32_t)t[0];
        if (dst) dst[i] = (int32_t)t[1];
        if (mass) mass[i] = t[2];
        if (node) node[i] = (int32_t)t[3];
    }
    return FT_OK;
}

extern "C" ft_status ft_knn(const ft_dataset* cds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                            const uint32_t* q_w, int32_t k, int64_t prefilter_m, int64_t* out_ids, double* out_val,
                            void* stream) {
    const char* who = "ft_knn";
    if (!cds) return fti_fail(FT_ESTATE, "ft_knn: NULL dataset");
    if (!out_ids || !out_val) return fti_fail(FT_EINVAL, "ft_knn: NULL output");
    if (k < 1) return fti_fail(FT_EINVAL, "ft_knn: need k >= 1");
    if (prefilter_m > 0 && prefilter_m < k) return fti_fail(FT_EINVAL, "ft_knn: need prefilter_m == 0 or >= k");
    if (k > FTI_MAX_SELECT) return fti_fail(FT_ERANGE, "ft_knn: k > 8192");
    ft_dataset* ds = const_cast<ft_dataset*>(cds);
    cudaStream_t st = (cudaStream_t)stream;
    const bool exhaustive = prefilter_m <= 0 || prefilter_m >= ds->n;
    if (!exhaustive && prefilter_m > FTI_MAX_SELECT) return fti_fail(FT_ERANGE, "ft_knn: prefilter_m > 8192");
    Staged S;
    ft_status rc = stage_queries(ds, q_off, nq, q_ids, q_w, st, who, S);
    if (rc) return rc;
    const bool dev_out = is_device_ptr(out_ids) && is_device_ptr(out_val);
    int64_t* d_ids = out_ids;
    double* d_val = out_val;
    if (!dev_out) {
        FTI_RES(ds->s_outid, sizeof(int64_t) * nq * k);
        FTI_RES(ds->s_outval, sizeof(double) * nq * k);
        d_ids = ds->s_outid.as<int64_t>();
        d_val = ds->s_outval.as<double>();
    }
    const int64_t n = ds->n;
    FTI_RES(ds->s_sel, sizeof(int) * ((size_t)nq + 1));
    int* sel_scratch = ds->s_sel.as<int>();
    if (exhaustive) {
        FTI_RES(ds->s_vals, sizeof(double) * nq * n);
        rc = flowtree_stage(ds, S, nq, nullptr, 0, n, ds->s_vals.as<double>(), n, st);
        if (rc) return rc;
        StageTimer tm(ds, FTI_ST_SELK, st);
        FTI_CUDA(fti_launch_select(ds->s_vals.as<double>(), n, nullptr, 0, n, nq, k, d_ids, d_val, k, sel_scratch,
                                   st));
    } else {
        const int64_t m = prefilter_m;
        FTI_RES(ds->s_cand, sizeof(int64_t) * nq * m);
        FTI_RES(ds->s_vals2, sizeof(double) * nq * m);
        {
            // Quadtree + top-m (fused: the stage time is reported under "quadtree")
            StageTimer tm(ds, FTI_ST_QT, st);
            FTI_CUDA(fti_launch_prefilter(ds, S.L, S.qblock, nq, m, ds->s_cand.as<int64_t>(), ds->s_vals2.as<double>(),
                                          sel_scratch, st));
        }
        rc = flowtree_stage(ds, S, nq, ds->s_cand.as<int64_t>(), m, m, ds->s_vals2.as<double>(), m, st);
        if (rc) return rc;
        StageTimer tm(ds, FTI_ST_SELK, st);
        FTI_CUDA(fti_launch_select(ds->s_vals2.as<double>(), m, ds->s_cand.as<int64_t>(), m, m, nq, k, d_ids, d_val,
                                   k, sel_scratch, st));
    }
    if (!dev_out) {
        FTI_CUDA(cudaMemcpyAsync(out_ids, d_ids, sizeof(int64_t) * nq * k, cudaMemcpyDeviceToHost, st));
        FTI_CUDA(cudaMemcpyAsync(out_val, d_val, sizeof(double) * nq * k, cudaMemcpyDeviceToHost, st));
        return check_device_errors(ds, st, who);
    }
    return FT_OK;
}

extern "C" ft_status ft_topk(const double* vals, int64_t vals_ld, const int64_t* ids, int64_t ids_ld, int64_t id_base,
                             int64_t L, int32_t rows, int32_t k, int64_t* out_ids, double* out_val, void* stream) {
    const char* who = "ft_topk";
    if (rows < 0 || L < 0 || k < 1) return fti_fail(FT_EINVAL, "ft_topk: need rows >= 0, L >= 0, k >= 1");
    if (k > FTI_MAX_SELECT) return fti_fail(FT_ERANGE, "ft_topk: k > 8192");
    if (rows == 0) return FT_OK;
    if (!vals || !out_ids || !out_val) return fti_fail(FT_EINVAL, "ft_topk: NULL pointer");
    if (!is_device_ptr(vals) || !is_device_ptr(out_ids) || !is_device_ptr(out_val) || (ids && !is_device_ptr(ids)))
        return fti_fail(FT_EINVAL, "ft_topk: device pointers required");
    if (vals_ld < L || (ids && ids_ld < L)) return fti_fail(FT_EINVAL, "ft_topk: leading dimension < L");
    cudaStream_t st = (cudaStream_t)stream;
    // the selection's scratch (redo counter + row list) is stream-ordered per call, so concurrent
    // calls on different streams or devices never share it
    int* scratch = nullptr;
    FTI_CUDA(cudaMallocAsync((void**)&scratch, sizeof(int) * ((size_t)rows + 1), st));
    const cudaError_t e = fti_launch_select(vals, vals_ld, ids, ids_ld, L, rows, k, out_ids, out_val, k, scratch, st,
                                            id_base);
    FTI_CUDA(cudaFreeAsync(scratch, st));
    if (e != cudaSuccess) return fti_fail(FT_ECUDA, std::string(who) + ": " + cudaGetErrorString(e));
    return FT_OK;
}

extern "C" ft_status ft_flowtree_estimate_lists(const ft_dataset* cds, const int64_t* q_off, int32_t nq,
                                                const int32_t* q_ids, const uint32_t* q_w, const int64_t* docs,
                                                int64_t docs_ld, int64_t n_per_q, double* out, void* stream) {
    const char* who = "ft_flowtree_estimate_lists";
    if (!cds) return fti_fail(FT_ESTATE, std::string(who) + ": NULL dataset");
    if (!docs || !out) return fti_fail(FT_EINVAL, std::string(who) + ": NULL docs or out");
    if (n_per_q < 1 || docs_ld < n_per_q) return fti_fail(FT_EINVAL, std::string(who) + ": need 1 <= n_per_q <= docs_ld");
    if (!is_device_ptr(docs) || !is_device_ptr(out)) return fti_fail(FT_EINVAL, std::string(who) + ": device docs / out required");
    ft_dataset* ds = const_cast<ft_dataset*>(cds);
    cudaStream_t st = (cudaStream_t)stream;
    Staged S;
    ft_status rc = stage_queries(ds, q_off, nq, q_ids, q_w, st, who, S);
    if (rc) return rc;
    return flowtree_stage(ds, S, nq, docs, docs_ld, n_per_q, out, n_per_q, st);
}

extern "C" ft_status ft_exact_w1_lists(const ft_dataset* cds, const int64_t* q_off, int32_t nq, const int32_t* q_ids,
                                       const uint32_t* q_w, const int64_t* docs, int64_t docs_ld, int64_t n_per_q,
                                       double* out, void* stream) {
    const char* who = "ft_exact_w1_lists";
    if (!cds) return fti_fail(FT_ESTATE, std::string(who) + ": NULL dataset");
    if (!docs || !out) return fti_fail(FT_EINVAL, std::string(who) + ": NULL docs or out");
    if (n_per_q < 1 || docs_ld < n_per_q) return fti_fail(FT_EINVAL, std::string(who) + ": need 1 <= n_per_q <= docs_ld");
    if (!is_device_ptr(docs) || !is_device_ptr(out)) return fti_fail(FT_EINVAL, std::string(who) + ": device docs / out required");
    ft_dataset* ds = const_cast<ft_dataset*>(cds);
    cudaStream_t st = (cudaStream_t)stream;
    Staged S;
    ft_status rc = stage_queries(ds, q_off, nq, q_ids, q_w, st, who, S);
    if (rc) return rc;
    FTI_CUDA(fti_launch_exact(ds, S.L, S.qblock, nq, docs, docs_ld, n_per_q, out, n_per_q, st));
    return FT_OK;
}

extern "C" ft_status ft_synchronize(const ft_dataset* ds, void* stream) {
    if (!ds) return fti_fail(FT_ESTATE, "ft_synchronize: NULL dataset");
    return check_device_errors(ds, (cudaStream_t)stream, "ft_synchronize");
}

extern "C" ft_status ft_profile_enable(ft_dataset* ds, int32_t enable) {
    if (!ds) return fti_fail(FT_ESTATE, "ft_profile_enable: NULL dataset");
    ds->prof = enable != 0;
    return FT_OK;
}

static ft_status profile_drain(ft_dataset* ds) {
    for (auto& p : ds->prof_pending) {
        FTI_CUDA(cudaEventSynchronize(p.b));
        float ms = 0.f;
        FTI_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        ds->prof_ms[p.stage] += ms;
        ds->prof_n[p.stage] += 1;
        ds->prof_pool.push_back(p.a);
        ds->prof_pool.push_back(p.b);
    }
    ds->prof_pending.clear();
    return FT_OK;
}

extern "C" ft_status ft_profile_reset(ft_dataset* ds) {
    if (!ds) return fti_fail(FT_ESTATE, "ft_profile_reset: NULL dataset");
    ft_status rc = profile_drain(ds);
    for (int s = 0; s < FT_NUM_STAGES; s++) { ds->prof_ms[s] = 0; ds->prof_n[s] = 0; }
    FTI_CUDA(cudaDeviceSynchronize());
    FTI_CUDA(cudaMemset(ds->prof_units, 0, sizeof(unsigned long long) * (FT_NUM_STAGES + 1)));
    return rc;
}

extern "C" ft_status ft_profile_units(ft_dataset* ds, int32_t stage, uint64_t* bytes) {
    if (!ds || !bytes) return fti_fail(FT_ESTATE, "ft_profile_units: NULL argument");
    if (stage < 0 || stage > FT_PROF_DIST_FLOPS) return fti_fail(FT_EINVAL, "ft_profile_units: bad stage");
    FTI_CUDA(cudaDeviceSynchronize());
    unsigned long long v = 0;
    FTI_CUDA(cudaMemcpy(&v, ds->prof_units + stage, sizeof(v), cudaMemcpyDeviceToHost));
    *bytes = v;
    return FT_OK;
}

extern "C" ft_status ft_profile_read(ft_dataset* ds, int32_t stage, double* total_ms, int64_t* launches) {
    if (!ds) return fti_fail(FT_ESTATE, "ft_profile_read: NULL dataset");
    if (stage < 0 || stage >= FT_NUM_STAGES) return fti_fail(FT_EINVAL, "ft_profile_read: bad stage");
    ft_status rc = profile_drain(ds);
    if (rc) return rc;
    if (total_ms) *total_ms = ds->prof_ms[stage];
    if (launches) *launches = ds->prof_n[stage];
    return FT_OK;
}

extern "C" const char* ft_profile_stage_name(int32_t stage) {
    static const char* names[FT_NUM_STAGES] = {"query_prep", "quadtree", "select_m", "vocab_map",
                                               "dist_table", "flowtree", "select_k"};
    return (stage >= 0 && stage < FT_NUM_STAGES) ? names[stage] : "";
}
