// ft_layout.cu — a1: node-sorted dataset layout in HBM.
//
// One CTA per document, two passes (count, fill):
//   * Flowtree record: support sorted by vocab id, {vocab | flags, w}; W = Σ w.
//   * Quadtree record: the non-root nodes on the support's paths, sorted by node id, with the
//     integer node mass m_μ(v) = Σ_{x under v} w_x — the sparse ℓ1 embedding of PAPER.md:131-134
//     (coordinate v = 2^{ℓ(v)} μ(v)); A = Σ_v ω(v) m_μ(v), ω(v) = 2^{D* − depth(v)}.
//   * M-nodes: the nodes holding ≥ 2 ground points, ordered (depth desc, node asc), each with the
//     list of the doc's item indices under it in vocab order — the only non-root places where
//     Flowtree can match distinct points.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "ft_device.cuh"

namespace {

struct LayoutArgs {
    const uint32_t* off;
    const int32_t* ids;
    const uint32_t* w;
    int64_t n, N;
    int cols, d_star;
    const int32_t* path;
    const uint8_t* leaf_depth;
    const uint8_t* node_depth;
    const int32_t* node_count;
    const uint32_t* vflags;
    int P_items, P_ent;
    uint32_t *cnt_qt, *cnt_mn, *cnt_ml;
    uint32_t* err;
    uint32_t* err_doc;
    const uint32_t *qt_off, *mn_off, *ml_off;
    uint2* items;
    uint32_t* W;
    uint2* qt;
    unsigned long long* A;
    uint4* mnodes;
    uint16_t* mlists;
    int fill;
};

__global__ void __launch_bounds__(256) k_layout(LayoutArgs a) {
    extern __shared__ unsigned long long sm[];
    unsigned long long* key_items = sm;                          // P_items
    unsigned long long* key_ent = key_items + a.P_items;         // P_ent
    int* seg_start = (int*)(key_ent + a.P_ent);                  // P_ent + 1
    int* seg_aux = seg_start + a.P_ent + 1;                      // P_ent (M-node output position)
    int* lens_pos = seg_aux + a.P_ent;                           // P_ent (list length by position)
    __shared__ int tmp[32];
    __shared__ int s_bad;
    __shared__ unsigned long long s_A;
    __shared__ unsigned int s_W;
    __shared__ int mn_hist[64];
    __shared__ int mn_lt[64], mn_gt[64];

    const int64_t doc = blockIdx.x;
    const uint32_t base = a.off[doc];
    const int s = (int)(a.off[doc + 1] - base);
    if (threadIdx.x == 0) { s_bad = 0; s_A = 0; s_W = 0; }
    if (threadIdx.x < 64) mn_hist[threadIdx.x] = 0;
    __syncthreads();
    unsigned int wsum = 0;
    for (int i = threadIdx.x; i < a.P_items; i += blockDim.x) {
        unsigned long long key = ~0ull;
        if (i < s) {
            int32_t x = a.ids[base + i];
            uint32_t wx = a.w[base + i];
            if (x < 0 || (int64_t)x >= a.N) { atomicOr((unsigned*)&s_bad, FTI_ERR_RANGE); x = 0; }
            if (wx == 0) atomicOr((unsigned*)&s_bad, FTI_ERR_INVAL);
            wsum += wx;
            key = ((unsigned long long)(uint32_t)x << 32) | wx;
        }
        key_items[i] = key;
    }
    if (s < 1) atomicOr((unsigned*)&s_bad, FTI_ERR_INVAL);
    atomicAdd(&s_W, wsum);    // W <= 2048 * 2^32 can wrap: check per-item bound below
    __syncthreads();
    fti_bitonic_sort_u64(key_items, a.P_items);
    for (int i = threadIdx.x + 1; i < s; i += blockDim.x)
        if ((key_items[i] >> 32) == (key_items[i - 1] >> 32)) atomicOr((unsigned*)&s_bad, FTI_ERR_INVAL);
    for (int i = threadIdx.x; i < s; i += blockDim.x)
        if ((uint32_t)key_items[i] > FTI_MAX_WEIGHT_TOTAL) atomicOr((unsigned*)&s_bad, FTI_ERR_OVERFLOW);
    __syncthreads();
    if (s_W > FTI_MAX_WEIGHT_TOTAL && !(s_bad & FTI_ERR_OVERFLOW)) {
        if (threadIdx.x == 0) s_bad |= FTI_ERR_OVERFLOW;
    }
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) {
            atomicOr(a.err, (unsigned)s_bad);
            atomicMin(a.err_doc, (unsigned)doc);
        }
        return;
    }
    // entries (node at depth k, item index) for k = 1..leafdepth(x)
    int run = 0;
    for (int c = 0; c < s; c += blockDim.x) {
        int i = c + threadIdx.x;
        int ld = 0;
        uint32_t x = 0;
        if (i < s) {
            x = (uint32_t)(key_items[i] >> 32);
            ld = a.leaf_depth[x];
        }
        int tot;
        int pos = run + fti_block_exclusive_sum(ld, tmp, &tot);
        for (int k = 1; k <= ld; k++)
            key_ent[pos + k - 1] = ((unsigned long long)(uint32_t)a.path[(int64_t)x * a.cols + k] << 32) | (unsigned)i;
        run += tot;
    }
    const int E = run;
    const int PE = fti_pow2_at_least(E < 1 ? 1 : E);
    for (int e = E + threadIdx.x; e < PE; e += blockDim.x) key_ent[e] = ~0ull;
    __syncthreads();
    fti_bitonic_sort_u64(key_ent, PE);
    // segments = distinct nodes
    int nseg_run = 0;
    for (int c = 0; c < E; c += blockDim.x) {
        int e = c + threadIdx.x;
        int f = 0;
        if (e < E) f = (e == 0) || ((key_ent[e] >> 32) != (key_ent[e - 1] >> 32));
        int tot;
        int r = nseg_run + fti_block_exclusive_sum(f, tmp, &tot);
        if (f) seg_start[r] = e;
        nseg_run += tot;
    }
    const int nseg = nseg_run;
    if (threadIdx.x == 0) seg_start[nseg] = E;
    __syncthreads();
    // per segment: mass, ω, M-node classification
    unsigned long long A_part = 0;
    int mn_run = 0;
    for (int c = 0; c < nseg; c += blockDim.x) {
        int g = c + threadIdx.x;
        int is_mn = 0, dep = 0;
        uint32_t node = 0, mass = 0;
        if (g < nseg) {
            int e0 = seg_start[g], e1 = seg_start[g + 1];
            node = (uint32_t)(key_ent[e0] >> 32);
            for (int e = e0; e < e1; e++) mass += (uint32_t)key_items[(uint32_t)key_ent[e]];
            dep = a.node_depth[node];
            int sh = a.d_star - dep;
            if (sh > 0 && ((unsigned long long)mass >> (64 - sh)) != 0) atomicOr((unsigned*)&s_bad, FTI_ERR_OVERFLOW);
            A_part += (unsigned long long)mass << sh;
            is_mn = a.node_count[node] >= 2;
            if (is_mn) atomicAdd(&mn_hist[dep], 1);
            if (a.fill) a.qt[a.qt_off[doc] + g] = make_uint2(node, mass | ((uint32_t)dep << 16));   // mass | depth << 16
        }
        int tot;
        int r = mn_run + fti_block_exclusive_sum(is_mn, tmp, &tot);
        if (g < nseg) seg_aux[g] = is_mn ? r : -1;   // rank among M-nodes (node order)
        mn_run += tot;
    }
    atomicAdd(&s_A, A_part);
    const int nmn = mn_run;
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) {
            atomicOr(a.err, (unsigned)s_bad);
            atomicMin(a.err_doc, (unsigned)doc);
        }
        return;
    }
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < 64; k++) { mn_lt[k] = acc; acc += mn_hist[k]; }
        acc = 0;
        for (int k = 63; k >= 0; k--) { mn_gt[k] = acc; acc += mn_hist[k]; }
    }
    __syncthreads();
    // output position of each M-node: (depth desc, node asc)
    for (int g = threadIdx.x; g < nseg; g += blockDim.x) {
        int r = seg_aux[g];
        if (r >= 0) {
            uint32_t node = (uint32_t)(key_ent[seg_start[g]] >> 32);
            int dep = a.node_depth[node];
            int pos = mn_gt[dep] + (r - mn_lt[dep]);
            seg_aux[g] = pos;
            lens_pos[pos] = seg_start[g + 1] - seg_start[g];
        }
    }
    __syncthreads();
    // exclusive scan of list lengths in output order
    int lrun = 0;
    for (int c = 0; c < nmn; c += blockDim.x) {
        int p = c + threadIdx.x;
        int v = p < nmn ? lens_pos[p] : 0;
        int tot;
        int ex = lrun + fti_block_exclusive_sum(v, tmp, &tot);
        if (p < nmn) lens_pos[p] = ex;   // becomes the local list offset
        lrun += tot;
    }
    const int nml = lrun;
    __syncthreads();
    if (!a.fill) {
        if (threadIdx.x == 0) {
            a.cnt_qt[doc] = nseg;
            a.cnt_mn[doc] = nmn;
            a.cnt_ml[doc] = nml;
        }
        return;
    }
    for (int i = threadIdx.x; i < s; i += blockDim.x) {
        uint32_t x = (uint32_t)(key_items[i] >> 32);
        a.items[base + i] = make_uint2(x | a.vflags[x], (uint32_t)key_items[i]);
    }
    if (threadIdx.x == 0) {
        a.W[doc] = s_W;
        a.A[doc] = s_A;
    }
    const uint32_t mo = a.mn_off[doc], lo = a.ml_off[doc];
    for (int g = threadIdx.x; g < nseg; g += blockDim.x) {
        int e0 = seg_start[g], e1 = seg_start[g + 1];
        uint32_t node = (uint32_t)(key_ent[e0] >> 32);
        if (a.node_count[node] < 2) continue;
        int pos = seg_aux[g];
        int lofs = lens_pos[pos];
        a.mnodes[mo + pos] = make_uint4(node, lo + lofs, (uint32_t)(e1 - e0), a.node_depth[node]);
        for (int e = e0; e < e1; e++) a.mlists[lo + lofs + (e - e0)] = (uint16_t)(uint32_t)key_ent[e];
    }
}

const char* err_name(uint32_t e) {
    if (e & FTI_ERR_RANGE) return "vocab id outside [0, N)";
    if (e & FTI_ERR_OVERFLOW) return "total mass W > 65535";
    return "empty document, zero mass or duplicate vocab id";
}
ft_status err_status(uint32_t e) {
    if (e & FTI_ERR_RANGE) return FT_ERANGE;
    if (e & FTI_ERR_OVERFLOW) return FT_EOVERFLOW;
    return FT_EINVAL;
}

}  // namespace

extern "C" ft_status ft_load_dataset(const ft_index* ix, const int64_t* doc_off, int64_t n, const int32_t* ids,
                                     const uint32_t* w, ft_dataset** out) {
    if (!out) return fti_fail(FT_EINVAL, "ft_load_dataset: out is NULL");
    *out = nullptr;
    if (!ix) return fti_fail(FT_ESTATE, "ft_load_dataset: NULL index");
    if (!doc_off || !ids || !w) return fti_fail(FT_EINVAL, "ft_load_dataset: NULL array");
    if (n < 1) return fti_fail(FT_EINVAL, "ft_load_dataset: need n >= 1");
    if (doc_off[0] != 0) return fti_fail(FT_EINVAL, "ft_load_dataset: doc_off[0] must be 0");
    int32_t max_s = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t s = doc_off[i + 1] - doc_off[i];
        if (s < 1) return fti_fail(FT_EINVAL, "ft_load_dataset: document " + std::to_string(i) + " is empty");
        if (s > FTI_MAX_SUPPORT)
            return fti_fail(FT_ERANGE, "ft_load_dataset: document " + std::to_string(i) + " has support > 2048");
        max_s = std::max<int32_t>(max_s, (int32_t)s);
    }
    int64_t nnz = doc_off[n];
    if (nnz >= (int64_t)0xFFFFFFFFll) return fti_fail(FT_ERANGE, "ft_load_dataset: nnz must be < 2^32");
    int P_items = fti_pow2_at_least(max_s);
    int P_ent = fti_pow2_at_least(std::max(1, max_s * std::max(1, ix->d_star)));
    if (P_ent > FTI_MAX_NODE_ENTRIES)
        return fti_fail(FT_ERANGE, "ft_load_dataset: support x tree depth exceeds 8192 entries");
    size_t smem = sizeof(unsigned long long) * (P_items + P_ent) + sizeof(int) * (3 * P_ent + 1);

    ft_dataset* ds = new ft_dataset();
    ds->ix = ix;
    ds->n = n;
    ds->nnz = nnz;
    ds->max_s = max_s;
    ds->unit_w = true;   // every doc weight 1: the lane-per-pair Flowtree kernel's uniform path
    for (int64_t t = 0; t < nnz && ds->unit_w; t++) ds->unit_w = w[t] == 1u;
    cudaStream_t st;
    FTI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<uint32_t> off32(n + 1);
    for (int64_t i = 0; i <= n; i++) off32[i] = (uint32_t)doc_off[i];
    int32_t* d_ids;
    uint32_t *d_w, *cnt, *offs, *err;
    FTI_CUDA(cudaMalloc(&ds->doc_off, sizeof(uint32_t) * (n + 1)));
    FTI_CUDA(cudaMalloc(&d_ids, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    FTI_CUDA(cudaMalloc(&d_w, sizeof(uint32_t) * std::max<int64_t>(nnz, 1)));
    FTI_CUDA(cudaMalloc(&cnt, sizeof(uint32_t) * 3 * (n + 1)));
    FTI_CUDA(cudaMalloc(&offs, sizeof(uint32_t) * 3 * (n + 1)));
    FTI_CUDA(cudaMalloc(&err, sizeof(uint32_t) * 2));
    FTI_CUDA(cudaMemcpyAsync(ds->doc_off, off32.data(), sizeof(uint32_t) * (n + 1), cudaMemcpyHostToDevice, st));
    FTI_CUDA(cudaMemcpyAsync(d_ids, ids, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
    FTI_CUDA(cudaMemcpyAsync(d_w, w, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, st));
    uint32_t err_init[2] = {0u, 0xFFFFFFFFu};
    FTI_CUDA(cudaMemcpyAsync(err, err_init, sizeof(err_init), cudaMemcpyHostToDevice, st));
    FTI_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * 3 * (n + 1), st));
    FTI_CUDA(cudaFuncSetAttribute(k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));

    LayoutArgs a{};
    a.off = ds->doc_off; a.ids = d_ids; a.w = d_w; a.n = n; a.N = ix->N;
    a.cols = ix->d_star + 1; a.d_star = ix->d_star;
    a.path = ix->path; a.leaf_depth = ix->leaf_depth; a.node_depth = ix->node_depth;
    a.node_count = ix->node_count; a.vflags = ix->vflags;
    a.P_items = P_items; a.P_ent = P_ent;
    a.cnt_qt = cnt; a.cnt_mn = cnt + (n + 1); a.cnt_ml = cnt + 2 * (n + 1);
    a.err = err; a.err_doc = err + 1;
    a.fill = 0;
    k_layout<<<(unsigned)n, 256, smem, st>>>(a);
    FTI_CUDA(cudaGetLastError());
    uint32_t herr[2];
    FTI_CUDA(cudaMemcpyAsync(herr, err, sizeof(herr), cudaMemcpyDeviceToHost, st));
    FTI_CUDA(cudaStreamSynchronize(st));
    if (herr[0]) {
        cudaFree(d_ids); cudaFree(d_w); cudaFree(cnt); cudaFree(offs); cudaFree(err);
        cudaStreamDestroy(st);
        ft_dataset_free(ds);
        return fti_fail(err_status(herr[0]), "ft_load_dataset: document " + std::to_string(herr[1]) + ": " +
                                                 err_name(herr[0]));
    }
    // exclusive scans of the three count arrays (n+1 entries each -> offsets with totals at [n])
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs, (int)(n + 1), st);
    void* tmp;
    FTI_CUDA(cudaMalloc(&tmp, tb));
    for (int t = 0; t < 3; t++) {
        size_t tb2 = tb;
        FTI_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb2, cnt + t * (n + 1), offs + t * (n + 1), (int)(n + 1), st));
    }
    uint32_t tot[3];
    for (int t = 0; t < 3; t++)
        FTI_CUDA(cudaMemcpyAsync(&tot[t], offs + t * (n + 1) + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    // max M-nodes per doc (for the Flowtree kernel's sizing)
    uint32_t* dmax;
    FTI_CUDA(cudaMalloc(&dmax, sizeof(uint32_t)));
    size_t tbm = 0;
    cub::DeviceReduce::Max(nullptr, tbm, cnt + (n + 1), dmax, (int)n, st);
    void* tmpm;
    FTI_CUDA(cudaMalloc(&tmpm, tbm));
    FTI_CUDA(cub::DeviceReduce::Max(tmpm, tbm, cnt + (n + 1), dmax, (int)n, st));
    uint32_t hmax = 0;
    FTI_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    FTI_CUDA(cudaStreamSynchronize(st));
    ds->n_qt = tot[0];
    ds->n_mn = tot[1];
    ds->n_ml = tot[2];
    ds->max_mn = (int32_t)hmax;
    // 8 zero records past the end: the Flowtree kernels prefetch a few items beyond a doc's last
    FTI_CUDA(cudaMalloc(&ds->items, sizeof(uint2) * (size_t)(nnz + 8)));
    FTI_CUDA(cudaMemset(ds->items + nnz, 0, sizeof(uint2) * 8));
    FTI_CUDA(cudaMalloc(&ds->W, sizeof(uint32_t) * n));
    FTI_CUDA(cudaMalloc(&ds->A, sizeof(unsigned long long) * n));
    FTI_CUDA(cudaMalloc(&ds->qt, sizeof(uint2) * std::max<int64_t>(ds->n_qt, 1)));
    FTI_CUDA(cudaMalloc(&ds->mnodes, sizeof(uint4) * std::max<int64_t>(ds->n_mn, 1)));
    FTI_CUDA(cudaMalloc(&ds->mlists, sizeof(uint16_t) * std::max<int64_t>(ds->n_ml, 1)));
    FTI_CUDA(cudaMalloc(&ds->qt_off, sizeof(uint32_t) * (n + 1)));
    FTI_CUDA(cudaMalloc(&ds->mn_off, sizeof(uint32_t) * (n + 1)));
    FTI_CUDA(cudaMemcpyAsync(ds->qt_off, offs, sizeof(uint32_t) * (n + 1), cudaMemcpyDeviceToDevice, st));
    FTI_CUDA(cudaMemcpyAsync(ds->mn_off, offs + (n + 1), sizeof(uint32_t) * (n + 1), cudaMemcpyDeviceToDevice, st));
    a.fill = 1;
    a.qt_off = ds->qt_off; a.mn_off = ds->mn_off; a.ml_off = offs + 2 * (n + 1);
    a.items = ds->items; a.W = ds->W; a.qt = ds->qt; a.A = ds->A; a.mnodes = ds->mnodes; a.mlists = ds->mlists;
    k_layout<<<(unsigned)n, 256, smem, st>>>(a);
    FTI_CUDA(cudaGetLastError());
    FTI_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_ids); cudaFree(d_w); cudaFree(cnt); cudaFree(offs); cudaFree(err); cudaFree(tmp);
    cudaFree(dmax); cudaFree(tmpm);
    cudaStreamDestroy(st);
    FTI_CUDA(cudaMalloc(&ds->err_dev, sizeof(uint32_t) * 4));
    FTI_CUDA(cudaMemset(ds->err_dev, 0, sizeof(uint32_t) * 4));
    FTI_CUDA(cudaMalloc(&ds->prof_units, sizeof(unsigned long long) * (FT_NUM_STAGES + 1)));
    FTI_CUDA(cudaMemset(ds->prof_units, 0, sizeof(unsigned long long) * (FT_NUM_STAGES + 1)));
    *out = ds;
    return FT_OK;
}

extern "C" ft_status ft_dataset_info(const ft_dataset* ds, int64_t* n, int64_t* nnz, int64_t* n_qt_records,
                                     int32_t* max_support) {
    if (!ds) return fti_fail(FT_ESTATE, "ft_dataset_info: NULL dataset");
    if (n) *n = ds->n;
    if (nnz) *nnz = ds->nnz;
    if (n_qt_records) *n_qt_records = ds->n_qt;
    if (max_support) *max_support = ds->max_s;
    return FT_OK;
}

extern "C" void ft_dataset_free(ft_dataset* ds) {
    if (!ds) return;
    cudaFree(ds->doc_off); cudaFree(ds->items); cudaFree(ds->W); cudaFree(ds->mn_off); cudaFree(ds->mnodes);
    cudaFree(ds->mlists); cudaFree(ds->qt_off); cudaFree(ds->qt); cudaFree(ds->A);
    if (ds->err_dev) cudaFree(ds->err_dev);
    if (ds->prof_units) cudaFree(ds->prof_units);
    DevBuf* bufs[] = {&ds->s_qoff, &ds->s_qids, &ds->s_qw, &ds->s_qblock, &ds->s_docs, &ds->s_vals, &ds->s_vals2,
                      &ds->s_cand, &ds->s_outid, &ds->s_outval, &ds->s_map, &ds->s_rows, &ds->s_rowcnt,
                      &ds->s_table, &ds->s_flow, &ds->s_flowcnt, &ds->s_vlist, &ds->s_chunk, &ds->s_rowbase, &ds->s_bsplit, &ds->s_ny, &ds->s_tiles, &ds->s_qinfo, &ds->s_wdesc, &ds->s_wrow, &ds->s_sel, &ds->s_chunkd, &ds->s_fblist, &ds->s_fbcnt, &ds->s_topk, &ds->s_pitch, &ds->s_chunkd2, &ds->s_gbase};
    for (DevBuf* b : bufs) b->release();
    delete ds;
}
