// ft_exact.cu — the exact-W1 stage of the paper's pipelines (Quadtree → Flowtree → Exact;
// PAPER.md:408-424, Table 5 :935-937): W1(μ, ν) of Eq. (1)
// for a few surviving (query, doc) pairs, by the transportation simplex (MODI / stepping stone) —
// one CTA per pair.
//
//   supplies  a_i = w_i · U  (doc items),  demands  b_j = u_j · W  (query items),  Σa = Σb = W·U
//   (the exact integer cross-scaling of reading R13), costs c_ij = ‖x_i − y_j‖₂ (FP32, in shared
//   memory), W1 = Σ f_ij c_ij / (W·U) accumulated in FP64.
//
// Costs: coordinates are staged 8 dimensions at a time (doc rows row-major, query rows transposed)
// and accumulated per cell in shared memory; a warp per row, lanes over the columns.
//
// Start (a basic feasible solution = m + n − 1 cells forming a spanning tree of the bipartite
// row/column graph): greedy "mutual minimum" rounds — every live row picks its cheapest live column
// and every live column its cheapest live row; each mutual pair is allocated min(supply, demand)
// and crosses out one exhausted line (the matrix-minimum method, several lines per round) — then
// the northwest corner over the remaining live lines.  Any sequence of "allocate at a live cell,
// cross out one exhausted line" gives a spanning tree; degenerate zero cells keep it spanning.
// The tree is rooted at row 0 (one DFS).  Nodes are rows 0..m−1 and columns m..m+n−1, one thread
// per node.  Each pivot is parallel over nodes and cells, O(log(m + n)) barriers:
//   1. pointer jumping over the parent links: depth, potentials (u_i + v_j = c_ij on basic cells,
//      pot = c_parent-edge − pot_parent, composed along the path to the root) and the
//      binary-lifting ancestor table;
//   2. reduced costs c_ij − u_i − v_j of every cell, block-wide argmin (Dantzig's rule, ties to the
//      smallest cell index); stop when the minimum is ≥ −tol;
//   3. the entering cell (p, q) closes a cycle with the tree paths p → LCA ← q; each node decides
//      from the lifting table whether its parent edge lies on it and at which position (cells
//      alternate −, +, … starting at q's parent edge); θ = the smallest flow on a − cell (first in
//      cycle order on ties) and that cell leaves;
//   4. flows ±θ around the cycle; the cut-off subtree is re-rooted at the entering cell's endpoint
//      by reversing the parent links on its path to the leaving edge.
// Flows stay exact integers (u32 < 2^32).  A pivot cap turns cycling into FTI_ERR_CAP + NaN.
//
// Shared memory is laid out per launch from the batch's largest supports (Mx doc points, Nx query
// points: Vx = Mx + Nx nodes, Mx·Nx cells): ≈ 99 B per node + 4 B per cell, so reviews-size pairs
// (≤ 90 × 90) run 4 CTAs per SM.
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ft_device.cuh"

namespace {

constexpr int EX_MAXV = 512;            // rows + columns per pair (one thread per node)
constexpr int EX_LOGX = 9;              // 2^EX_LOGX ≥ EX_MAXV
constexpr int EX_DC = 8;                // dimensions staged per cost chunk
constexpr int EX_GREEDY_ROUNDS = 48;    // mutual-minimum rounds before the NW-corner completion
constexpr size_t EX_SMEM_MAX = 226 * 1024;   // dynamic part; the static scalars fit in the rest

struct ExGeom {                          // byte offsets into the dynamic shared memory
    int Vx, cells;                       // a pair fits iff m + n ≤ Vx and m·n ≤ cells
    int o_pot, o_bf, o_sup, o_dem, o_xid, o_yid, o_bi, o_bj, o_pn, o_pe, o_anc, o_sgn, o_pdep, o_dep,
        o_alive, o_best, o_cost;
    size_t bytes;
};

__host__ __device__ inline int ex_align(int x, int a) { return (x + a - 1) / a * a; }

ExGeom ex_geom(int Vx, int cells) {
    ExGeom g{};
    g.Vx = Vx; g.cells = cells;
    const int V = Vx;
    int o = 32 * V;                       // [0, 32V): pacc[2][V] doubles, reused as cost staging / DFS scratch
    g.o_pot = o;   o += 8 * V;
    g.o_bf = o;    o += 4 * V;
    g.o_sup = o;   o += 4 * V;
    g.o_dem = o;   o += 4 * V;
    g.o_xid = o;   o += 4 * V;
    g.o_yid = o;   o += 4 * V;
    g.o_bi = o;    o += 2 * V;
    g.o_bj = o;    o += 2 * V;
    g.o_pn = o;    o += 2 * V;
    g.o_pe = o;    o += 2 * V;
    g.o_anc = o;   o += 2 * (EX_LOGX + 1) * V;
    g.o_pdep = o;  o += 4 * V;
    g.o_dep = o;   o += 2 * V;
    g.o_best = o;  o += 2 * V;
    g.o_sgn = o;   o += 2 * V;
    g.o_alive = o; o += V;
    o = ex_align(o, 16);
    g.o_cost = o;  o += 4 * cells;
    g.bytes = (size_t)ex_align(o, 16);
    return g;
}

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
    ExGeom g;
    int greedy;
    int q0;                     // first query of this launch (grid.y ≤ 65535)
};

__device__ unsigned long long g_exdbg[10];

#define EXT(slot) do { if (DBG && t == 0) { const long long c_ = clock64(); dbg[slot] += c_ - tlast; tlast = c_; } } while (0)

// argmin of (value, index) pairs within a warp; ties to the smaller index, index −1 = none
__device__ __forceinline__ void warp_argmin(float& v, int& ix) {
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
        if (oi >= 0 && (ix < 0 || ov < v || (ov == v && oi < ix))) { v = ov; ix = oi; }
    }
}

template <int NT, bool DBG>
__global__ void __launch_bounds__(NT) k_exact(ExArgs a) {
    long long tlast = DBG ? clock64() : 0;
    long long dbg[6] = {0, 0, 0, 0, 0, 0};
    int rounds = 0;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char sm[];
    const ExGeom& g = a.g;
    const int Vx = g.Vx;
    double* pacc = (double*)sm;                                  // [2][Vx]
    double* pot = (double*)(sm + g.o_pot);                       // u (rows 0..m−1), v (columns m..)
    uint32_t* bf = (uint32_t*)(sm + g.o_bf);                     // basic cell flows; slot = edge id
    uint32_t* sup = (uint32_t*)(sm + g.o_sup);
    uint32_t* dem = (uint32_t*)(sm + g.o_dem);
    uint32_t* xid = (uint32_t*)(sm + g.o_xid);
    uint32_t* yid = (uint32_t*)(sm + g.o_yid);
    int16_t* bi = (int16_t*)(sm + g.o_bi);                      // basic cells (row, col)
    int16_t* bj = (int16_t*)(sm + g.o_bj);
    int16_t* par_n = (int16_t*)(sm + g.o_pn);                   // parent node (root: itself)
    int16_t* par_e = (int16_t*)(sm + g.o_pe);                   // parent edge (root: −1)
    uint16_t* anc = (uint16_t*)(sm + g.o_anc);                  // [LOG+1][Vx] 2^k-th ancestor
    int16_t* pdep = (int16_t*)(sm + g.o_pdep);                  // [2][Vx]
    int16_t* dep = (int16_t*)(sm + g.o_dep);
    int16_t* best = (int16_t*)(sm + g.o_best);                  // greedy: best partner per line
    int8_t* psgn = (int8_t*)(sm + g.o_sgn);                     // [2][Vx]
    uint8_t* alive = sm + g.o_alive;                             // greedy: line not crossed out
    float* cost = (float*)(sm + g.o_cost);                       // [m][n]
    __shared__ double red_v[NW];
    __shared__ int red_i[NW];
    __shared__ unsigned long long s_key;
    __shared__ int s_enter, s_done, s_lca, s_x, s_ra, s_ca, s_k;
    __shared__ float s_maxc;

    const int q = a.q0 + (int)blockIdx.y;
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
    if (m + n > g.Vx || m * n > g.cells) { // outside the launch's geometry (host sized it from the maxima)
        if (t == 0) { *outp = __longlong_as_double(0x7ff8000000000000ll); atomicOr(a.err, FTI_ERR_CAP); }
        return;
    }
    const int V = m + n;
    const uint32_t W = a.Wd[doc], U = hdr->U;
    const uint2* qitems = (const uint2*)(slot + a.L.off_items);
    for (int i = t; i < m; i += NT) {
        const uint2 it = a.items[i0 + i];
        xid[i] = it.x & FTI_VOCAB_MASK;
        sup[i] = it.y * U;
    }
    for (int j = t; j < n; j += NT) {
        const uint2 it = qitems[j];
        yid[j] = it.x & FTI_VOCAB_MASK;
        dem[j] = it.y * W;
    }
    for (int c = t; c < m * n; c += NT) cost[c] = 0.f;
    if (t == 0) s_maxc = 0.f;
    __syncthreads();
    // ---- cost matrix: Σ (x − y)² over 8-dimension chunks staged in shared memory; each thread
    //      holds its share of the next chunk in registers while the current one is consumed ----
    {
        constexpr int PF = EX_DC;                      // (m + n) ≤ NT, so 8 (m + n) ≤ PF · NT
        float* xs = (float*)sm;                  // [m][EX_DC]
        float* yt = xs + m * EX_DC;              // [EX_DC][n]
        const int nel = (m + n) * EX_DC;
        float pre[PF];
        auto fetch = [&](int e0) {
#pragma unroll
            for (int r = 0; r < PF; r++) {
                const int k = t + r * NT;
                float v = 0.f;
                if (k < nel) {
                    const int row = k / EX_DC, e = k - row * EX_DC;
                    const uint32_t id = row < m ? xid[row] : yid[row - m];
                    if (e0 + e < a.d) v = __ldg(a.X + (int64_t)id * a.d + e0 + e);
                }
                pre[r] = v;
            }
        };
        fetch(0);
        for (int e0 = 0; e0 < a.d; e0 += EX_DC) {
#pragma unroll
            for (int r = 0; r < PF; r++) {
                const int k = t + r * NT;
                if (k < m * EX_DC) xs[k] = pre[r];
                else if (k < nel) {
                    const int kk = k - m * EX_DC, j = kk / EX_DC, e = kk - j * EX_DC;
                    yt[e * n + j] = pre[r];
                }
            }
            __syncthreads();
            if (e0 + EX_DC < a.d) fetch(e0 + EX_DC);
            for (int i = warp; i < m; i += NW) {
                float xv[EX_DC];
#pragma unroll
                for (int e = 0; e < EX_DC; e++) xv[e] = xs[i * EX_DC + e];
                for (int j = lane; j < n; j += 32) {
                    float acc = cost[i * n + j];
#pragma unroll
                    for (int e = 0; e < EX_DC; e++) {
                        const float df = xv[e] - yt[e * n + j];
                        acc = fmaf(df, df, acc);
                    }
                    cost[i * n + j] = acc;
                }
            }
            __syncthreads();
        }
        float lmax = 0.f;
        for (int c = t; c < m * n; c += NT) {
            const int i = c / n, j = c - i * n;
            const float cv = xid[i] == yid[j] ? 0.f : sqrtf(cost[c]);
            cost[c] = cv;
            lmax = fmaxf(lmax, cv);
        }
        for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        if (lane == 0) atomicMax((int*)&s_maxc, __float_as_int(lmax));   // non-negative floats order as ints
    }
    for (int v = t; v < V; v += NT) { alive[v] = 1; best[v] = -1; }
    if (t == 0) { s_ra = m; s_ca = n; s_k = 0; s_done = 0; }
    __syncthreads();
    EXT(0);
    // ---- start: mutual-minimum rounds.  best[] caches each live line's cheapest live partner; lines
    //      only die, so a cached partner that is still live is still the minimum ----
    for (int round = 0; a.greedy && round < EX_GREEDY_ROUNDS; round++) {
        if (s_ra <= 1 || s_ca <= 1) break;
        rounds++;
        for (int i = warp; i < m; i += NW) {
            const int c = best[i];
            if (!alive[i] || (c >= 0 && alive[m + c])) continue;
            float bv = FLT_MAX;
            int bx = -1;
            for (int j = lane; j < n; j += 32)
                if (alive[m + j] && (bx < 0 || cost[i * n + j] < bv)) { bv = cost[i * n + j]; bx = j; }
            warp_argmin(bv, bx);
            if (lane == 0) best[i] = (int16_t)bx;
        }
        for (int j = warp; j < n; j += NW) {
            const int c = best[m + j];
            if (!alive[m + j] || (c >= 0 && alive[c])) continue;
            float bv = FLT_MAX;
            int bx = -1;
            for (int i = lane; i < m; i += 32)
                if (alive[i] && (bx < 0 || cost[i * n + j] < bv)) { bv = cost[i * n + j]; bx = i; }
            warp_argmin(bv, bx);
            if (lane == 0) best[m + j] = (int16_t)bx;
        }
        __syncthreads();
        // mutual pairs (one thread per row, m ≤ NT): disjoint lines, so they commute
        bool mut = false, krow = false;
        int jj = -1;
        uint32_t f = 0;
        if (t < m && alive[t]) {
            jj = best[t];
            if (alive[m + jj] && best[m + jj] == t) {
                mut = true;
                f = sup[t] < dem[jj] ? sup[t] : dem[jj];
                krow = sup[t] == f;              // the row is exhausted (ties cross out the row)
            }
        }
        const int P = __syncthreads_count(mut);
        const int R = __syncthreads_count(mut && krow);
        const int ra = s_ra, ca = s_ca;
        if (ra - R >= 1 && ca - (P - R) >= 1) {  // no last row / column crossed out: all at once
            if (mut) {
                const int k = atomicAdd(&s_k, 1);
                bi[k] = (int16_t)t; bj[k] = (int16_t)jj; bf[k] = f;
                sup[t] -= f; dem[jj] -= f;
                if (krow) alive[t] = 0; else alive[m + jj] = 0;
            }
            __syncthreads();
            if (t == 0) { s_ra = ra - R; s_ca = ca - (P - R); }
        } else {
            __syncthreads();
            if (t == 0) {                        // in row order until one line of a kind is left
                int k = s_k, r2 = ra, c2 = ca;
                for (int i = 0; i < m && r2 > 1 && c2 > 1; i++) {
                    if (!alive[i]) continue;
                    const int j = best[i];
                    if (!alive[m + j] || best[m + j] != i) continue;
                    const uint32_t g2 = sup[i] < dem[j] ? sup[i] : dem[j];
                    bi[k] = (int16_t)i; bj[k] = (int16_t)j; bf[k] = g2; k++;
                    sup[i] -= g2; dem[j] -= g2;
                    if (sup[i] == 0) { alive[i] = 0; r2--; }
                    else { alive[m + j] = 0; c2--; }
                }
                s_k = k; s_ra = r2; s_ca = c2;
            }
        }
        __syncthreads();
    }
    EXT(4);
    // ---- northwest-corner completion over the live lines (thread 0) ----
    if (t == 0) {
        int k = s_k;
        int i = 0, j = 0;
        while (!alive[i]) i++;
        while (!alive[m + j]) j++;
        while (true) {
            const uint32_t f = sup[i] < dem[j] ? sup[i] : dem[j];
            bi[k] = (int16_t)i; bj[k] = (int16_t)j; bf[k] = f; k++;
            sup[i] -= f; dem[j] -= f;
            int ni = i + 1, nj = j + 1;
            while (ni < m && !alive[ni]) ni++;
            while (nj < n && !alive[m + nj]) nj++;
            if (ni >= m && nj >= n) break;
            if (nj >= n || (sup[i] == 0 && ni < m)) i = ni;
            else j = nj;
        }
        s_k = k;                                 // = m + n − 1
    }
    // ---- root the tree at row 0: adjacency lists (scratch in the pacc region), BFS by warp 0 ----
    int* adj_off = (int*)sm;                     // [V + 1]
    int* adj = adj_off + V + 1;                  // [2 (V − 1)]
    int* cur = adj + 2 * V;                      // [V]: degree, then fill cursor, then BFS queue
    for (int v = t; v < V; v += NT) cur[v] = 0;
    __syncthreads();
    const int nbasis = s_k;
    for (int e = t; e < nbasis; e += NT) { atomicAdd(&cur[bi[e]], 1); atomicAdd(&cur[m + bj[e]], 1); }
    __syncthreads();
    if (warp == 0) {
        const int per = (V + 31) / 32, lo = min(V, lane * per), hi = min(V, lo + per);
        int sum = 0;
        for (int v = lo; v < hi; v++) sum += cur[v];
        int incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int run = incl - sum;
        for (int v = lo; v < hi; v++) { const int dg = cur[v]; adj_off[v] = run; cur[v] = run; run += dg; }
        if (lane == 31) adj_off[V] = incl;
    }
    __syncthreads();
    for (int e = t; e < nbasis; e += NT) {
        adj[atomicAdd(&cur[bi[e]], 1)] = e;
        adj[atomicAdd(&cur[m + bj[e]], 1)] = e;
    }
    __syncthreads();
    if (warp == 0) {
        for (int v = lane; v < V; v += 32) par_e[v] = -2;
        __syncwarp();
        if (lane == 0) { par_e[0] = -1; par_n[0] = 0; cur[0] = 0; s_x = 1; }
        __syncwarp();
        int head = 0, tail = 1;
        while (head < tail) {                    // one tree level per step: each node has one parent
            for (int qi = head + lane; qi < tail; qi += 32) {
                const int v = cur[qi];
                for (int pp = adj_off[v]; pp < adj_off[v + 1]; pp++) {
                    const int e = adj[pp];
                    const int w = v < m ? m + bj[e] : bi[e];
                    if (par_e[w] != -2) continue;
                    par_e[w] = (int16_t)e; par_n[w] = (int16_t)v;
                    cur[atomicAdd(&s_x, 1)] = w;
                }
            }
            __syncwarp();
            head = tail;
            tail = *(volatile int*)&s_x;
            __syncwarp();
        }
    }
    __syncthreads();
    EXT(5);
    const int LOG = 32 - __clz(V - 1);           // 2^LOG ≥ V > any depth
    const double tol = 1e-9 * (double)s_maxc;
    const int max_pivots = 50 * V + 100;
    int piv = 0;
    while (true) {
        // ---- 1. pointer jumping: depth, potentials, ancestor table ----
        int cur = 0;
        if (t < V) {
            const int pn = par_n[t], pe = par_e[t];
            anc[t] = (uint16_t)pn;
            pacc[t] = pe < 0 ? 0.0 : (double)cost[bi[pe] * n + bj[pe]];
            psgn[t] = pe < 0 ? 1 : -1;
            pdep[t] = pe < 0 ? 0 : 1;
        }
        __syncthreads();
        for (int k = 0; k < LOG; k++) {
            if (t < V) {
                const int an = anc[k * Vx + t];
                const int o = cur * Vx, o2 = (cur ^ 1) * Vx;
                pacc[o2 + t] = pacc[o + t] + (double)psgn[o + t] * pacc[o + an];
                psgn[o2 + t] = (int8_t)(psgn[o + t] * psgn[o + an]);
                pdep[o2 + t] = (int16_t)(pdep[o + t] + pdep[o + an]);
                anc[(k + 1) * Vx + t] = anc[k * Vx + an];
            }
            cur ^= 1;
            __syncthreads();
        }
        if (t < V) { pot[t] = pacc[cur * Vx + t]; dep[t] = pdep[cur * Vx + t]; }
        __syncthreads();
        EXT(1);
        // ---- 2. most negative reduced cost: thread (column j, first row r0), rows r0, r0 + R, … ----
        {
            double bestr = 0.0;
            int bidx = -1;
            const int R = NT / n, j = t % n, r0 = t / n;
            if (r0 < R) {
                const double vj = pot[m + j];
                for (int i = r0; i < m; i += R) {
                    const double r = (double)cost[i * n + j] - pot[i] - vj;
                    if (r < bestr) { bestr = r; bidx = i * n + j; }
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, bestr, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
                if (ob < bestr || (ob == bestr && oi >= 0 && (bidx < 0 || oi < bidx))) { bestr = ob; bidx = oi; }
            }
            if (lane == 0) { red_v[warp] = bestr; red_i[warp] = bidx; }
        }
        __syncthreads();
        if (warp == 0) {                                   // across warps: warp 0, then lane 0 pivots
            double bv = lane < NW ? red_v[lane] : 0.0;
            int bx = lane < NW ? red_i[lane] : -1;
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bx, o);
                if (ob < bv || (ob == bv && oi >= 0 && (bx < 0 || oi < bx))) { bv = ob; bx = oi; }
            }
            const int enter = (bv < -tol) ? bx : -1;
            if (lane == 0) {
                s_enter = enter;
                if (enter < 0) s_done = 1;
                else if (++piv > max_pivots) s_done = 2;
                if (enter >= 0) {
                    // LCA of row p and column m + qq by binary lifting
                    int x = enter / n, y = m + (enter - (enter / n) * n);
                    if (dep[x] < dep[y]) { const int tt = x; x = y; y = tt; }
                    int diff = dep[x] - dep[y];
                    for (int k = 0; diff; k++, diff >>= 1)
                        if (diff & 1) x = anc[k * Vx + x];
                    if (x != y) {
                        for (int k = LOG; k >= 0; k--)
                            if (anc[k * Vx + x] != anc[k * Vx + y]) { x = anc[k * Vx + x]; y = anc[k * Vx + y]; }
                        x = anc[x];
                    }
                    s_lca = x;
                    s_key = ~0ull;
                }
            }
        }
        __syncthreads();
        EXT(2);
        if (s_done) break;
        // ---- 3. cycle membership and the leaving cell ----
        const int p = s_enter / n, qq = s_enter - (s_enter / n) * n, qn = m + qq;
        const int lca = s_lca, dl = dep[lca];
        const int nbk = dep[qn] - dl;                  // edges on q's side
        int pos = -1, side = 0;                        // side 1: q's path, 2: p's path
        if (t < V && t != lca && dep[t] > dl) {
            int x = qn, diff = dep[qn] - dep[t];
            if (diff >= 0) {
                for (int k = 0; diff; k++, diff >>= 1)
                    if (diff & 1) x = anc[k * Vx + x];
                if (x == t) { side = 1; pos = dep[qn] - dep[t]; }
            }
            if (!side) {
                x = p; diff = dep[p] - dep[t];
                if (diff >= 0) {
                    for (int k = 0; diff; k++, diff >>= 1)
                        if (diff & 1) x = anc[k * Vx + x];
                    if (x == t) { side = 2; pos = nbk + (dep[t] - dl - 1); }
                }
            }
            if (side && (pos & 1) == 0)
                atomicMin(&s_key, ((unsigned long long)bf[par_e[t]] << 32) | (unsigned)pos);
        }
        __syncthreads();
        const unsigned long long key = s_key;
        const uint32_t theta = (uint32_t)(key >> 32);
        const int lpos = (int)(key & 0xFFFFFFFFu);
        int my_pn = 0, my_pe = -1;
        if (side) {
            my_pn = par_n[t]; my_pe = par_e[t];
            bf[my_pe] = (pos & 1) ? bf[my_pe] + theta : bf[my_pe] - theta;
            if (pos == lpos) s_x = t;
        }
        __syncthreads();
        // ---- 4. re-root the cut-off subtree at the entering cell's endpoint ----
        const int x = s_x, leave = par_e[x];
        const int lside = lpos < nbk ? 1 : 2;
        __syncthreads();                               // everyone has read par_e[x]
        if (side == lside && dep[t] > dep[x]) {        // path node strictly below x: flip its link
            par_n[my_pn] = (int16_t)t;
            par_e[my_pn] = (int16_t)my_pe;
        }
        if (t == 0) {
            const int s = lside == 1 ? qn : p;
            par_n[s] = (int16_t)(lside == 1 ? p : qn);
            par_e[s] = (int16_t)leave;
            bi[leave] = (int16_t)p; bj[leave] = (int16_t)qq; bf[leave] = theta;
        }
        __syncthreads();
        EXT(3);
    }
    // ---- W1 = Σ f c / (W U) ----
    double part = 0.0;                           // over tree nodes: independent of edge-slot order
    for (int v = t; v < V; v += NT) {
        const int e = par_e[v];
        if (e >= 0) part += (double)bf[e] * (double)cost[bi[e] * n + bj[e]];
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red_v[warp] = part;
    __syncthreads();
    if (t == 0) {
        double tot = 0.0;
        for (int w = 0; w < NW; w++) tot += red_v[w];
        if (DBG) {
            for (int k = 0; k < 6; k++) atomicAdd(&g_exdbg[k], (unsigned long long)dbg[k]);
            atomicAdd(&g_exdbg[6], (unsigned long long)piv);
            atomicAdd(&g_exdbg[7], 1ull);
            atomicAdd(&g_exdbg[8], (unsigned long long)(m * n));
            atomicAdd(&g_exdbg[9], (unsigned long long)rounds);
        }
        if (s_done == 2) {
            atomicOr(a.err, FTI_ERR_CAP);
            *outp = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            *outp = tot / ((double)W * (double)U);
        }
    }
}

template <int NT>
cudaError_t ex_launch(const ExArgs& a, dim3 grid, cudaStream_t st, bool dbg) {
    auto kern = dbg ? k_exact<NT, true> : k_exact<NT, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.g.bytes);
    if (e != cudaSuccess) return e;
    ExArgs b = a;
    for (unsigned q0 = 0; q0 < grid.y; q0 += 65535) {
        b.q0 = (int)q0;
        kern<<<dim3(grid.x, std::min(65535u, grid.y - q0)), NT, a.g.bytes, st>>>(b);
    }
    return cudaSuccess;
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
    a.greedy = fti_opt(FT_OPT_EXACT_START_NW) ? 0 : 1;
    // geometry from the largest supports (doc side from the dataset, query side from the batch);
    // pairs beyond EX_MAXV − 1 nodes or the shared-memory budget fail alone (NaN + FTI_ERR_CAP)
    const int Mx = std::max(1, (int)ds->max_s), Nx = std::max(1, (int)L.smax);
    const int Vx = std::min(Mx + Nx, EX_MAXV - 1);
    const int64_t want = std::min<int64_t>((int64_t)Mx * Nx, (int64_t)(Vx / 2) * (Vx - Vx / 2));
    const int64_t room = ((int64_t)EX_SMEM_MAX - (int64_t)ex_geom(Vx, 0).bytes - 16) / 4;
    a.g = ex_geom(Vx, (int)std::min(want, room));
    const bool dbg = (fti_opt(FT_OPT_DEBUG) & FTI_DBG_EXACT) != 0;
    const dim3 grid((unsigned)n_per_q, (unsigned)nq);
    cudaError_t e = a.g.Vx <= 256 ? ex_launch<256>(a, grid, st, dbg) : ex_launch<512>(a, grid, st, dbg);
    if (e != cudaSuccess) return e;
    fti_count_launches(1);
    if (dbg) {
        unsigned long long h[10];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_exdbg, sizeof(h));
        const double c = h[7] ? (double)h[7] : 1.0;
        fprintf(stderr, "exact dbg per CTA (Vx %d cells %d smem %zu): cost %.1f greedy %.1f (%.1f rounds) nw+dfs %.1f kcyc | pivots %.1f: jump %.1f price %.1f cycle %.1f kcyc | m*n %.0f\n",
                a.g.Vx, a.g.cells, a.g.bytes, h[0] / c / 1e3, h[4] / c / 1e3, h[9] / c, h[5] / c / 1e3, h[6] / c,
                h[1] / c / 1e3, h[2] / c / 1e3, h[3] / c / 1e3, h[8] / c);
        memset(h, 0, sizeof(h));
        cudaMemcpyToSymbol(g_exdbg, h, sizeof(h));
    }
    return cudaGetLastError();
}
