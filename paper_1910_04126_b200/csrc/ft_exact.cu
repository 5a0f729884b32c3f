// ft_exact.cu — the exact-W1 stage of the paper's pipelines (Quadtree → Flowtree → Exact;
// PAPER.md:408-424, Table 5 :935-937): W1(μ, ν) of Eq. (1)
// for a few surviving (query, doc) pairs, by the transportation simplex (MODI / stepping stone) —
// one CTA per pair.
//
//   supplies  a_i = w_i · U  (doc items),  demands  b_j = u_j · W  (query items),  Σa = Σb = W·U
//   (the exact integer cross-scaling of reading R13), costs c_ij = ‖x_i − y_j‖₂ (FP32, in shared
//   memory), W1 = Σ f_ij c_ij / (W·U) accumulated in FP64.
//
// Start: the northwest-corner basis in vocab order (m + n − 1 basic cells, a spanning tree of the
// bipartite row/column graph; degenerate zero cells keep it spanning).  Each pivot:
//   1. potentials u_i + v_j = c_ij on the basic cells by a DFS over the basis tree (thread 0),
//      recording each node's parent edge;
//   2. reduced costs c_ij − u_i − v_j of every cell in parallel, block-wide argmin;
//   3. stop when the minimum is ≥ −tol; else the entering cell (p, q) closes the cycle
//      p → … → q through the tree; θ = the smallest flow on the cycle's odd (−) cells; the first
//      of them reaching 0 leaves the basis (thread 0).
// Flows stay exact integers (u32 < 2^32).  A pivot cap turns cycling into FTI_ERR_CAP + NaN.
#include <algorithm>
#include <cfloat>

#include "ft_device.cuh"

namespace {

constexpr int EX_THREADS = 256;
constexpr int EX_MAXS = 128;            // support cap per side for this stage

struct ExArgs {
    const uint32_t* doc_off;
    const uint2* items;
    const uint32_t* Wd;
    const float* X;
    int d;
    int64_t n;
    const uint8_t* qblock;
    QueryLayout L;
    const int64_t* docs;
    int64_t docs_ld, n_per_q;
    double* out;
    int64_t out_ld;
    uint32_t* err;
};

__global__ void __launch_bounds__(EX_THREADS) k_exact(ExArgs a) {
    extern __shared__ float cost[];        // [EX_MAXS][EX_MAXS] (dynamic: 64 KB)
    __shared__ uint32_t sup[EX_MAXS], dem[EX_MAXS];
    __shared__ uint32_t xid[EX_MAXS], yid[EX_MAXS];
    __shared__ double pu[EX_MAXS], pv[EX_MAXS];
    // basis: 2S − 1 cells {row, col, flow}; per node (rows 0..m−1, cols m..m+n−1) parent edge
    __shared__ int bi[2 * EX_MAXS], bj[2 * EX_MAXS];
    __shared__ uint32_t bf[2 * EX_MAXS];
    __shared__ int adj_off[2 * EX_MAXS + 1], adj[4 * EX_MAXS];
    __shared__ int par_edge[2 * EX_MAXS], par_node[2 * EX_MAXS], depth[2 * EX_MAXS], stk[2 * EX_MAXS];
    __shared__ int cyc_a[2 * EX_MAXS], cyc_b[2 * EX_MAXS];
    __shared__ double red_v[EX_THREADS / 32];
    __shared__ int red_i[EX_THREADS / 32];
    __shared__ int s_enter, s_done, s_m, s_n, s_nb;
    __shared__ float s_maxc;

    const int q = blockIdx.y;
    const int64_t slot_j = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    double* outp = a.out + (int64_t)q * a.out_ld + slot_j;
    const int64_t doc = a.docs[(int64_t)q * a.docs_ld + slot_j];
    if (hdr->err || hdr->s == 0) {
        if (t == 0) *outp = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    if (doc < 0) {
        if (t == 0) *outp = __longlong_as_double(0x7ff0000000000000ll);
        return;
    }
    if (doc >= a.n) {
        if (t == 0) { *outp = __longlong_as_double(0x7ff8000000000000ll); atomicOr(a.err, FTI_ERR_RANGE); }
        return;
    }
    const uint32_t i0 = a.doc_off[doc];
    const int m = (int)(a.doc_off[doc + 1] - i0), n = (int)hdr->s;
    if (m > EX_MAXS || n > EX_MAXS) {
        if (t == 0) { *outp = __longlong_as_double(0x7ff8000000000000ll); atomicOr(a.err, FTI_ERR_CAP); }
        return;
    }
    const uint32_t W = a.Wd[doc], U = hdr->U;
    const uint2* qitems = (const uint2*)(slot + a.L.off_items);
    for (int i = t; i < m; i += EX_THREADS) {
        const uint2 it = a.items[i0 + i];
        xid[i] = it.x & FTI_VOCAB_MASK;
        sup[i] = it.y * U;
    }
    for (int j = t; j < n; j += EX_THREADS) {
        const uint2 it = qitems[j];
        yid[j] = it.x & FTI_VOCAB_MASK;
        dem[j] = it.y * W;
    }
    __syncthreads();
    // cost matrix: a warp per (i, j) cell row-chunk, lanes over the coordinates
    float lmax = 0.f;
    for (int c = warp; c < m * n; c += EX_THREADS / 32) {
        const int i = c / n, j = c - i * n;
        const float* xr = a.X + (int64_t)xid[i] * a.d;
        const float* yr = a.X + (int64_t)yid[j] * a.d;
        float acc = 0.f;
        for (int e = lane; e < a.d; e += 32) {
            const float df = xr[e] - yr[e];
            acc = fmaf(df, df, acc);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const float cv = xid[i] == yid[j] ? 0.f : sqrtf(acc);
        if (lane == 0) cost[i * EX_MAXS + j] = cv;
        lmax = fmaxf(lmax, cv);
    }
    if (t == 0) s_maxc = 0.f;
    __syncthreads();
    if (lane == 0) atomicMax((int*)&s_maxc, __float_as_int(lmax));   // non-negative floats order as ints
    // northwest-corner basis (thread 0): m + n − 1 cells
    if (t == 0) {
        int i = 0, j = 0, k = 0;
        uint32_t ra = sup[0], rb = dem[0];
        while (true) {
            const uint32_t f = ra < rb ? ra : rb;
            bi[k] = i; bj[k] = j; bf[k] = f; k++;
            ra -= f; rb -= f;
            if (i == m - 1 && j == n - 1) break;
            if (ra == 0 && i < m - 1) { i++; ra = sup[i]; }
            else { j++; rb = dem[j]; }
        }
        s_nb = k;          // = m + n − 1
        s_m = m; s_n = n;
        s_done = 0;
    }
    __syncthreads();
    const int nb = s_nb;
    const double tol = 1e-9 * (double)s_maxc;
    const int max_pivots = 50 * (m + n) + 100;
    int piv = 0;
    while (true) {
        // ---- 1. potentials over the basis tree, rooted at row 0 (thread 0) ----
        if (t == 0) {
            const int V = m + n;
            for (int v = 0; v <= V; v++) adj_off[v] = 0;
            for (int e = 0; e < nb; e++) { adj_off[bi[e] + 1]++; adj_off[m + bj[e] + 1]++; }
            for (int v = 0; v < V; v++) adj_off[v + 1] += adj_off[v];
            for (int v = 0; v < V; v++) stk[v] = adj_off[v];
            for (int e = 0; e < nb; e++) { adj[stk[bi[e]]++] = e; adj[stk[m + bj[e]]++] = e; }
            for (int v = 0; v < V; v++) par_edge[v] = -2;
            int sp = 0;
            stk[sp++] = 0;
            par_edge[0] = -1; par_node[0] = -1; depth[0] = 0;
            pu[0] = 0.0;
            while (sp) {
                const int v = stk[--sp];
                for (int p = adj_off[v]; p < adj_off[v + 1]; p++) {
                    const int e = adj[p];
                    const int w = v < m ? m + bj[e] : bi[e];
                    if (par_edge[w] != -2) continue;
                    par_edge[w] = e; par_node[w] = v; depth[w] = depth[v] + 1;
                    const double c = (double)cost[bi[e] * EX_MAXS + bj[e]];
                    if (w >= m) pv[w - m] = c - pu[v];
                    else pu[w] = c - pv[v - m];
                    stk[sp++] = w;
                }
            }
        }
        __syncthreads();
        // ---- 2. most negative reduced cost ----
        double best = 0.0;
        int bidx = -1;
        for (int c = t; c < m * n; c += EX_THREADS) {
            const int i = c / n, j = c - i * n;
            const double r = (double)cost[i * EX_MAXS + j] - pu[i] - pv[j];
            if (r < best) { best = r; bidx = c; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
            if (ob < best || (ob == best && oi >= 0 && (bidx < 0 || oi < bidx))) { best = ob; bidx = oi; }
        }
        if (lane == 0) { red_v[warp] = best; red_i[warp] = bidx; }
        __syncthreads();
        if (t == 0) {
            double bv = 0.0;
            int bx = -1;
            for (int w = 0; w < EX_THREADS / 32; w++)
                if (red_v[w] < bv || (red_v[w] == bv && red_i[w] >= 0 && (bx < 0 || red_i[w] < bx))) {
                    bv = red_v[w];
                    bx = red_i[w];
                }
            s_enter = (bv < -tol) ? bx : -1;
            if (s_enter < 0) s_done = 1;
            else if (++piv > max_pivots) s_done = 2;
        }
        __syncthreads();
        if (s_done) break;
        // ---- 3. the cycle of the entering cell and the pivot (thread 0) ----
        if (t == 0) {
            const int p = s_enter / n, qq = s_enter - p * n;
            // path between row node p and column node m + qq in the tree: climb to the LCA
            int a0 = p, b0 = m + qq, na = 0, nbk = 0;
            int* pa = cyc_a;                     // edges climbing from p
            int* pbk = cyc_b;                    // edges climbing from q
            while (depth[a0] > depth[b0]) { pa[na++] = par_edge[a0]; a0 = par_node[a0]; }
            while (depth[b0] > depth[a0]) { pbk[nbk++] = par_edge[b0]; b0 = par_node[b0]; }
            while (a0 != b0) {
                pa[na++] = par_edge[a0]; a0 = par_node[a0];
                pbk[nbk++] = par_edge[b0]; b0 = par_node[b0];
            }
            // cycle order: (p, q)+ then from q down its climb to the LCA, then up p's climb
            // reversed; the cells alternate −, +, −, … starting at q's first edge
            uint32_t theta = 0xFFFFFFFFu;
            int leave = -1;
            int pos = 0;
            for (int k = 0; k < nbk; k++, pos++)
                if ((pos & 1) == 0 && bf[pbk[k]] < theta) { theta = bf[pbk[k]]; leave = pbk[k]; }
            for (int k = na - 1; k >= 0; k--, pos++)
                if ((pos & 1) == 0 && bf[pa[k]] < theta) { theta = bf[pa[k]]; leave = pa[k]; }
            pos = 0;
            for (int k = 0; k < nbk; k++, pos++) bf[pbk[k]] = (pos & 1) ? bf[pbk[k]] + theta : bf[pbk[k]] - theta;
            for (int k = na - 1; k >= 0; k--, pos++) bf[pa[k]] = (pos & 1) ? bf[pa[k]] + theta : bf[pa[k]] - theta;
            bi[leave] = p; bj[leave] = qq; bf[leave] = theta;
        }
        __syncthreads();
    }
    // ---- W1 = Σ f c / (W U) ----
    double part = 0.0;
    for (int e = t; e < nb; e += EX_THREADS) part += (double)bf[e] * (double)cost[bi[e] * EX_MAXS + bj[e]];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red_v[warp] = part;
    __syncthreads();
    if (t == 0) {
        double tot = 0.0;
        for (int w = 0; w < EX_THREADS / 32; w++) tot += red_v[w];
        if (s_done == 2) {
            atomicOr(a.err, FTI_ERR_CAP);
            *outp = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            *outp = tot / ((double)W * (double)U);
        }
    }
}

}  // namespace

cudaError_t fti_launch_exact(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                             const int64_t* d_docs, int64_t docs_ld, int64_t n_per_q, double* d_out, int64_t out_ld,
                             cudaStream_t st) {
    if (nq <= 0 || n_per_q <= 0) return cudaSuccess;
    ExArgs a{};
    a.doc_off = ds->doc_off; a.items = ds->items; a.Wd = ds->W;
    a.X = ds->ix->X; a.d = ds->ix->d; a.n = ds->n;
    a.qblock = d_qblock; a.L = L;
    a.docs = d_docs; a.docs_ld = docs_ld; a.n_per_q = n_per_q;
    a.out = d_out; a.out_ld = out_ld;
    a.err = ds->err_dev;
    const size_t smem = sizeof(float) * EX_MAXS * EX_MAXS;
    cudaError_t e = cudaFuncSetAttribute(k_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_exact<<<dim3((unsigned)n_per_q, (unsigned)nq), EX_THREADS, smem, st>>>(a);
    fti_count_launches(1);
    return cudaGetLastError();
}
