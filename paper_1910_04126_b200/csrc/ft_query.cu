// ft_query.cu — a2: query preparation, one CTA per query.
//
// Builds the query slot read by the estimate kernels:
//   items    support sorted by vocab id {vocab | flags, u}, U = Σ u
//   vhash    vocab id -> item index (Flowtree phase A: singleton-leaf self matches)
//   nhash    non-root node -> m_ν(v) and depth (Quadtree), B = Σ ω(v) m_ν(v)
//   mhash    M-node -> (list offset, length, depth) with the item lists in vocab order
//            (Flowtree phase B)
#include <algorithm>

#include "ft_device.cuh"

QueryLayout fti_query_layout(const ft_index* ix, int32_t smax) {
    QueryLayout L;
    L.smax = std::max(1, smax);
    L.vh_cap = fti_pow2_at_least(std::max(32, 2 * L.smax));
    int ent = L.smax * std::max(1, ix->d_star);
    L.nh_cap = fti_pow2_at_least(std::max(32, 2 * ent));
    L.mh_cap = L.nh_cap;
    L.ml_cap = ent;
    auto up = [](size_t x, size_t a) { return (x + a - 1) / a * a; };
    size_t o = sizeof(QHeader);
    L.off_items = o; o = up(o + 8ull * L.smax, 16);
    L.off_vh = o;    o = up(o + 8ull * L.vh_cap, 16);
    L.off_nh = o;    o = up(o + 8ull * L.nh_cap, 16);
    L.off_nd = o;    o = up(o + 1ull * L.nh_cap, 16);
    L.off_mh = o;    o = up(o + 16ull * L.mh_cap, 16);
    L.off_ml = o;    o = up(o + 2ull * L.ml_cap, 128);
    L.stride = o;
    return L;
}

namespace {

struct PrepArgs {
    const int64_t* qoff;
    const int32_t* qids;
    const uint32_t* qw;
    int32_t nq;
    int64_t N;
    int cols, d_star;
    const int32_t* path;
    const uint8_t* leaf_depth;
    const uint8_t* node_depth;
    const int32_t* node_count;
    const uint32_t* vflags;
    QueryLayout L;
    int P_items, P_ent;
    uint8_t* qblock;
    uint32_t* err;
};

__global__ void __launch_bounds__(256) k_query_prep(PrepArgs a) {
    extern __shared__ unsigned long long sm[];
    unsigned long long* key_items = sm;
    unsigned long long* key_ent = key_items + a.P_items;
    int* seg_start = (int*)(key_ent + a.P_ent);
    __shared__ int tmp[32];
    __shared__ unsigned s_bad;
    __shared__ unsigned s_U;
    __shared__ unsigned long long s_B;
    __shared__ int s_nmn_list;

    const int q = blockIdx.x;
    uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    QHeader* hdr = (QHeader*)slot;
    uint2* items = (uint2*)(slot + a.L.off_items);
    uint2* vh = (uint2*)(slot + a.L.off_vh);
    uint2* nh = (uint2*)(slot + a.L.off_nh);
    uint8_t* nd = slot + a.L.off_nd;
    uint4* mh = (uint4*)(slot + a.L.off_mh);
    uint16_t* ml = (uint16_t*)(slot + a.L.off_ml);

    const int64_t base = a.qoff[q];
    const int s = (int)(a.qoff[q + 1] - base);
    if (threadIdx.x == 0) { s_bad = 0; s_U = 0; s_B = 0; s_nmn_list = 0; }
    __syncthreads();
    if (s < 1 || s > a.L.smax) {
        if (threadIdx.x == 0) {
            hdr->s = 0; hdr->U = 0; hdr->err = FTI_ERR_INVAL;
            atomicOr(a.err, FTI_ERR_INVAL);
        }
        return;
    }
    unsigned usum = 0;
    for (int i = threadIdx.x; i < a.P_items; i += blockDim.x) {
        unsigned long long key = ~0ull;
        if (i < s) {
            int32_t x = a.qids[base + i];
            uint32_t u = a.qw[base + i];
            if (x < 0 || (int64_t)x >= a.N) { atomicOr(&s_bad, FTI_ERR_RANGE); x = 0; }
            if (u == 0) atomicOr(&s_bad, FTI_ERR_INVAL);
            if (u > FTI_MAX_WEIGHT_TOTAL) atomicOr(&s_bad, FTI_ERR_OVERFLOW);
            usum += u;
            key = ((unsigned long long)(uint32_t)x << 32) | u;
        }
        key_items[i] = key;
    }
    atomicAdd(&s_U, usum);
    __syncthreads();
    fti_bitonic_sort_u64(key_items, a.P_items);
    for (int i = threadIdx.x + 1; i < s; i += blockDim.x)
        if ((key_items[i] >> 32) == (key_items[i - 1] >> 32)) atomicOr(&s_bad, FTI_ERR_INVAL);
    __syncthreads();
    if (s_U > FTI_MAX_WEIGHT_TOTAL && threadIdx.x == 0) s_bad |= FTI_ERR_OVERFLOW;
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) {
            hdr->s = 0; hdr->U = 0; hdr->err = s_bad;
            atomicOr(a.err, s_bad);
        }
        return;
    }
    for (int i = threadIdx.x; i < s; i += blockDim.x) {
        uint32_t x = (uint32_t)(key_items[i] >> 32);
        items[i] = make_uint2(x | a.vflags[x], (uint32_t)key_items[i]);
    }
    // entries (node at depth k, item index) for k = 1..leafdepth
    int run = 0;
    for (int c = 0; c < s; c += blockDim.x) {
        int i = c + threadIdx.x;
        int ld = 0;
        uint32_t x = 0;
        if (i < s) { x = (uint32_t)(key_items[i] >> 32); ld = a.leaf_depth[x]; }
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
    // hash sizes for this query
    const uint32_t vh_n = (uint32_t)min(a.L.vh_cap, fti_pow2_at_least(max(32, 2 * s)));
    const uint32_t nh_n = (uint32_t)min(a.L.nh_cap, fti_pow2_at_least(max(32, 2 * nseg)));
    for (uint32_t i = threadIdx.x; i < vh_n; i += blockDim.x) vh[i] = make_uint2(FTI_EMPTY, 0);
    for (uint32_t i = threadIdx.x; i < nh_n; i += blockDim.x) { nh[i] = make_uint2(FTI_EMPTY, 0); nd[i] = 0; }
    // M-node count first (for the hash size)
    int mcount = 0;
    for (int c = 0; c < nseg; c += blockDim.x) {
        int g = c + threadIdx.x;
        int is_mn = 0;
        if (g < nseg) is_mn = a.node_count[(uint32_t)(key_ent[seg_start[g]] >> 32)] >= 2;
        int tot;
        fti_block_exclusive_sum(is_mn, tmp, &tot);
        mcount += tot;
    }
    const uint32_t mh_n = (uint32_t)min(a.L.mh_cap, fti_pow2_at_least(max(32, 2 * mcount)));
    for (uint32_t i = threadIdx.x; i < mh_n; i += blockDim.x) mh[i] = make_uint4(FTI_EMPTY, 0, 0, 0);
    __syncthreads();
    // vocab hash
    for (int i = threadIdx.x; i < s; i += blockDim.x) {
        uint32_t x = (uint32_t)(key_items[i] >> 32);
        uint32_t h = fti_hash(x) & (vh_n - 1);
        while (atomicCAS(&vh[h].x, FTI_EMPTY, x) != FTI_EMPTY) h = (h + 1) & (vh_n - 1);
        vh[h].y = (uint32_t)i;
    }
    // node hash, B, M-node lists
    unsigned long long Bp = 0;
    for (int c = 0; c < nseg; c += blockDim.x) {
        int g = c + threadIdx.x;
        int len = 0;
        uint32_t node = 0, mass = 0;
        int dep = 0, is_mn = 0;
        if (g < nseg) {
            int e0 = seg_start[g], e1 = seg_start[g + 1];
            node = (uint32_t)(key_ent[e0] >> 32);
            for (int e = e0; e < e1; e++) mass += (uint32_t)key_items[(uint32_t)key_ent[e]];
            dep = a.node_depth[node];
            Bp += (unsigned long long)mass << (a.d_star - dep);
            uint32_t h = fti_hash(node) & (nh_n - 1);
            while (atomicCAS(&nh[h].x, FTI_EMPTY, node) != FTI_EMPTY) h = (h + 1) & (nh_n - 1);
            nh[h].y = mass;
            nd[h] = (uint8_t)dep;
            is_mn = a.node_count[node] >= 2;
            if (is_mn) len = e1 - e0;
        }
        int tot;
        int lofs = s_nmn_list + fti_block_exclusive_sum(len, tmp, &tot);
        if (is_mn) {
            int e0 = seg_start[g];
            for (int t = 0; t < len; t++) ml[lofs + t] = (uint16_t)(uint32_t)key_ent[e0 + t];
            uint32_t h = fti_hash(node) & (mh_n - 1);
            while (atomicCAS(&mh[h].x, FTI_EMPTY, node) != FTI_EMPTY) h = (h + 1) & (mh_n - 1);
            mh[h].y = (uint32_t)lofs;
            mh[h].z = (uint32_t)len;
            mh[h].w = (uint32_t)dep;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_nmn_list += tot;
        __syncthreads();
    }
    atomicAdd(&s_B, Bp);
    __syncthreads();
    if (threadIdx.x == 0) {
        hdr->s = (uint32_t)s;
        hdr->U = s_U;
        hdr->B = s_B;
        hdr->nh_mask = nh_n - 1;
        hdr->vh_mask = vh_n - 1;
        hdr->mh_mask = mh_n - 1;
        hdr->n_nodes = (uint32_t)nseg;
        hdr->n_mn = (uint32_t)mcount;
        hdr->n_ml = (uint32_t)s_nmn_list;
        hdr->err = 0;
    }
}

}  // namespace

cudaError_t fti_launch_query_prep(const ft_index* ix, const QueryLayout& L, const int64_t* d_qoff, int32_t nq,
                                  const int32_t* d_qids, const uint32_t* d_qw, uint8_t* d_qblock, uint32_t* d_err,
                                  cudaStream_t st) {
    PrepArgs a{};
    a.qoff = d_qoff; a.qids = d_qids; a.qw = d_qw; a.nq = nq; a.N = ix->N;
    a.cols = ix->d_star + 1; a.d_star = ix->d_star;
    a.path = ix->path; a.leaf_depth = ix->leaf_depth; a.node_depth = ix->node_depth;
    a.node_count = ix->node_count; a.vflags = ix->vflags;
    a.L = L;
    a.P_items = fti_pow2_at_least(L.smax);
    a.P_ent = fti_pow2_at_least(std::max(1, L.ml_cap));
    a.qblock = d_qblock;
    a.err = d_err;
    size_t smem = sizeof(unsigned long long) * (a.P_items + a.P_ent) + sizeof(int) * (a.P_ent + 1);
    cudaError_t e = cudaFuncSetAttribute(k_query_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (nq > 0) k_query_prep<<<nq, 256, smem, st>>>(a);
    fti_count_launches(nq > 0 ? 1 : 0);
    return cudaGetLastError();
}
