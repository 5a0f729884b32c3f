// ft_flow.cu — a6: Flowtree estimate kernel (§3; greedy flow PAPER.md:495-504).
//
// One warp per (query, doc) pair.  Masses are cross-scaled integers (reading R13): μ'(x) = w_x·U,
// ν'(y) = u_y·W, both totalling W·U < 2^32, so every residual and prefix sum is an exact u32.
// The greedy bottom-up flow with the canonical tie-break (reading R10: at every node, residual
// lists in ascending vocab id, two-pointer northwest corner) is evaluated in three phases that
// visit exactly the nodes where matching can happen (C_μ(v), C_ν(v) ≠ ∅):
//   A  singleton leaves: a vocab id present on both sides self-matches min(μ', ν') at its leaf
//      (reading R8), distance 0;
//   B  M-nodes (cells holding ≥ 2 ground points) present on both sides, deepest first, each a
//      northwest corner over the vocab-ordered residual lists under it;
//   C  the root: northwest corner over all residuals in vocab order.
// Each northwest corner is computed in parallel: inclusive prefix sums S of both residual lists
// (warp scans), T = min of the totals, and every μ-item emits its overlaps with the ν-items
// whose cumulative intervals meet [S_{i−1}, min(S_i, T)) — the same set of triples the
// sequential two-pointer produces.  Leftovers: r_i ← max(0, S_i − max(S_{i−1}, T)).
// The flow is priced with FP32 Euclidean distances (on the fly for d ≤ 32, else from the a5
// table) and accumulated in FP64: FT = Σ η·dist / (W·U).
#include <algorithm>
#include <cstdlib>

#include "ft_device.cuh"

namespace {

struct FtArgs {
    const uint32_t* doc_off;
    const uint2* items;
    const uint32_t* Wd;
    const uint32_t* mn_off;
    const uint4* mnodes;
    const uint16_t* mlists;
    const float* X;
    int d;
    const int32_t* path;
    int cols;
    const uint8_t* leaf_depth;
    int64_t N;
    const uint8_t* qblock;
    QueryLayout L;
    int32_t nq;
    const int64_t* docs;
    int64_t docs_ld;
    int64_t n_docs;
    int64_t docs_per_cta;
    FtTable tab;
    double* out;
    int64_t out_ld;
    uint32_t* flow;
    uint32_t* flowcnt;
    int flow_cap;
    int Sd, Sq;
    int small_d;
    int64_t n;
    uint32_t* err;
    int use_bitmap;   // query vocab lookup by bitmap + rank (N small enough), else by hash
    int nwords;       // bitmap words = ceil(N / 32)
    unsigned long long* units;   // profiler: Σ pairs (8 s_doc + 16) algorithmic bytes, or null
    const uint32_t* fb_list;     // list mode: [nq][fb_cap] doc positions handed over by k_ftd
    const uint32_t* fb_cnt;      // [nq]
    int64_t fb_cap;
    int32_t q0;                  // first query of this launch (grid.y ≤ 65535)
};

#ifndef FT_BATCH_B
#define FT_BATCH_B 1       // phase B batched per depth (0: one warp northwest corner per node)
#endif
constexpr int64_t FT_BITMAP_MAX_N = 1 << 19;   // 16K words: 64 KB bitmap + 64 KB rank at most

constexpr int FT_WARPS = 8;                 // warps per CTA (fewer when the supports are large)

// per-warp shared words: dvoc, dres, dcum [Sd]; qres, qcum [Sq]; batched phase B: node table
// [8][32], u16 lists [Sd], [Sq], u8 node indices [Sd], [Sq]
__host__ __device__ __forceinline__ int ft_per_warp_words(int Sd, int Sq) {
    const int b16 = 2 * ((Sd + 1) & ~1) + 2 * ((Sq + 1) & ~1);
    const int b8 = ((Sd + 3) & ~3) + ((Sq + 3) & ~3);
    return 3 * Sd + 2 * Sq + 256 + (b16 + b8 + 3) / 4;
}
constexpr size_t FT_SMEM_MAX = 227 * 1024;

struct PairCtx {
    const FtArgs* a;
    int q;
    const uint2* qitem;     // smem
    const float* Y;         // smem (small d) or null
    uint32_t* dvoc;         // per-warp smem
    uint32_t* dres;
    uint32_t* dcum;
    uint32_t* qres;
    uint32_t* qcum;
    // batched phase B (one depth's common M-nodes at a time): concatenated item lists, their node
    // index in the batch, and per-node {doc start, query start, doc len, query len, doc base, query
    // base, T, node id}
    uint16_t* alst;
    uint16_t* blst;
    uint8_t* aseg;
    uint8_t* bseg;
    uint32_t* nb;           // [8][32]
    const float* trow_base; // table for this query or null
    uint32_t tld;           // its row pitch
    const uint2* map;       // candidate-vocabulary bitmap {bits, rank} per 32 ids, or null (row = vocab)
    const uint16_t* gml;    // the query's M-node item lists
};

__device__ __forceinline__ float pair_dist(const PairCtx& c, uint32_t x, uint32_t y, int jq) {
    const FtArgs& a = *c.a;
    if (c.trow_base) {
        int64_t row = (int64_t)x;
        if (c.map) {
            const uint2 m = c.map[x >> 5];
            row = (int64_t)(m.y + __popc(m.x & ((1u << (x & 31)) - 1u)));
        }
        FTI_ASSERT(jq < (int)c.tld && (!c.a->tab.rowcnt || row < c.a->tab.rowcnt[c.q]));
        return c.trow_base[row * c.tld + jq];
    }
    // on the fly, FP32 direct differences (the query row from shared memory when staged)
    const float* xr = a.X + (int64_t)x * a.d;
    const float* yr = c.Y ? c.Y + jq * a.d : a.X + (int64_t)y * a.d;
    if (a.d == 2) {   // planar ground sets (the image grid): the same FP32 operations, unrolled
        const float2 xv = *(const float2*)xr;
        const float d0 = xv.x - yr[0], d1 = xv.y - yr[1];
        return sqrtf(fmaf(d1, d1, fmaf(d0, d0, 0.f)));
    }
    float acc = 0.f;
    for (int t = 0; t < a.d; t++) {
        float df = xr[t] - yr[t];
        acc = fmaf(df, df, acc);
    }
    return sqrtf(acc);
}

template <bool EXPORT>
__device__ __forceinline__ void emit(const FtArgs& a, uint32_t x, uint32_t y, uint32_t eta, uint32_t node) {
    if (EXPORT) {
        uint32_t idx = atomicAdd(a.flowcnt, 1u);
        if ((int)idx < a.flow_cap) {
            a.flow[4 * idx + 0] = x;
            a.flow[4 * idx + 1] = y;
            a.flow[4 * idx + 2] = eta;
            a.flow[4 * idx + 3] = node;
        }
    }
}

// Northwest corner at one node.  A-list: doc item indices (a_list == null → identity 0..la),
// B-list: query item indices (b_list == null → identity).  Adds the priced flow to `cost`.
template <bool EXPORT>
__device__ void nw_corner(const PairCtx& c, const uint16_t* a_list, int la, const uint16_t* b_list, int lb,
                          uint32_t node, int lane, double& cost) {
    uint32_t carry = 0;
    for (int p0 = 0; p0 < la; p0 += 32) {
        int p = p0 + lane;
        uint32_t v = 0;
        if (p < la) v = c.dres[a_list ? a_list[p] : p];
        uint32_t incl = fti_warp_incl_u32(v, lane) + carry;
        if (p < la) c.dcum[p] = incl;
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    const uint32_t TA = carry;
    if (TA == 0) return;   // no doc mass left under the node: nothing matches, residuals unchanged
    carry = 0;
    for (int p0 = 0; p0 < lb; p0 += 32) {
        int p = p0 + lane;
        uint32_t v = 0;
        if (p < lb) v = c.qres[b_list ? b_list[p] : p];
        uint32_t incl = fti_warp_incl_u32(v, lane) + carry;
        if (p < lb) c.qcum[p] = incl;
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    const uint32_t TB = carry;
    __syncwarp();
    const uint32_t T = TA < TB ? TA : TB;
    if (T == 0) return;
    for (int p = lane; p < la; p += 32) {
        const uint32_t hi_a = c.dcum[p];
        const uint32_t lo_a = p ? c.dcum[p - 1] : 0u;
        const uint32_t end = hi_a < T ? hi_a : T;
        if (lo_a >= end) continue;
        // first j with qcum[j] > lo_a
        int lo = 0, hi = lb;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (c.qcum[mid] > lo_a) hi = mid; else lo = mid + 1;
        }
        const int ia = a_list ? a_list[p] : p;
        const uint32_t x = c.dvoc[ia] & FTI_VOCAB_MASK;
        for (int j = lo; j < lb; j++) {
            const uint32_t lo_b = j ? c.qcum[j - 1] : 0u;
            if (lo_b >= end) break;
            const uint32_t hi_b = c.qcum[j];
            const uint32_t s0 = lo_b > lo_a ? lo_b : lo_a;
            const uint32_t s1 = hi_b < end ? hi_b : end;
            if (s1 > s0) {
                const uint32_t eta = s1 - s0;
                const int jq = b_list ? b_list[j] : j;
                const uint32_t y = c.qitem[jq].x & FTI_VOCAB_MASK;
                if (x != y) cost += (double)eta * (double)pair_dist(c, x, y, jq);
                emit<EXPORT>(*c.a, x, y, eta, node);
            }
        }
    }
    __syncwarp();
    for (int p = lane; p < la; p += 32) {
        const uint32_t hi = c.dcum[p], lo = p ? c.dcum[p - 1] : 0u;
        c.dres[a_list ? a_list[p] : p] = hi <= T ? 0u : hi - (lo > T ? lo : T);
    }
    for (int p = lane; p < lb; p += 32) {
        const uint32_t hi = c.qcum[p], lo = p ? c.qcum[p - 1] : 0u;
        c.qres[b_list ? b_list[p] : p] = hi <= T ? 0u : hi - (lo > T ? lo : T);
    }
    __syncwarp();
}

// Phase B batched over the common M-nodes of ONE depth (≤ 32 records of the doc, lane l holds record
// l): the nodes are disjoint subtrees, so their northwest corners are independent (reading R11) and
// run as one segmented pass — the lists concatenated, one warp scan per side, per node
// T = min(totals), every doc item emitting its overlaps with the query items of its own node, the
// leftovers written back — instead of a warp pass per node.  The triples are those of nw_corner
// node by node.
template <bool EXPORT>
__device__ void batch_nw(const PairCtx& c, const uint4& rec, const uint4& qe, bool hit, int lane, double& cost) {
    const unsigned hm = __ballot_sync(0xffffffffu, hit);
    if (!hm) return;
    const int nh = __popc(hm);
    uint32_t* nDS = c.nb;
    uint32_t* nQS = c.nb + 32;
    uint32_t* nDL = c.nb + 64;
    uint32_t* nQL = c.nb + 96;
    uint32_t* nBA = c.nb + 128;
    uint32_t* nBB = c.nb + 160;
    uint32_t* nT = c.nb + 192;
    uint32_t* nID = c.nb + 224;
    const uint32_t dl = hit ? rec.z : 0u, ql = hit ? qe.z : 0u;
    const uint32_t dsi = fti_warp_incl_u32(dl, lane), qsi = fti_warp_incl_u32(ql, lane);
    const int LA = (int)__shfl_sync(0xffffffffu, dsi, 31), LB = (int)__shfl_sync(0xffffffffu, qsi, 31);
    const int ni = __popc(hm & ((1u << lane) - 1u));
    if (hit) {
        nDS[ni] = dsi - dl; nQS[ni] = qsi - ql; nDL[ni] = dl; nQL[ni] = ql;
    }
    // the concatenated lists (u16 item indices) and each element's node: element p of a side finds
    // its node by binary search over the node starts
    uint32_t* nDO = c.nb + 192;   // list offsets (nT / nID slots, rewritten below)
    uint32_t* nQO = c.nb + 224;
    if (hit) { nDO[ni] = rec.y; nQO[ni] = qe.y; }
    __syncwarp();
    auto seg_of = [&](const uint32_t* starts, int p) {
        int lo = 0, hi = nh - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (starts[mid] <= (uint32_t)p) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    for (int p = lane; p < LA; p += 32) {
        const int i = seg_of(nDS, p);
        c.alst[p] = c.a->mlists[nDO[i] + ((uint32_t)p - nDS[i])];
        c.aseg[p] = (uint8_t)i;
    }
    for (int p = lane; p < LB; p += 32) {
        const int i = seg_of(nQS, p);
        c.blst[p] = c.gml[nQO[i] + ((uint32_t)p - nQS[i])];
        c.bseg[p] = (uint8_t)i;
    }
    __syncwarp();
    if (hit) nID[ni] = rec.x;
    // global inclusive prefix sums over the concatenations
    uint32_t carry = 0;
    for (int p0 = 0; p0 < LA; p0 += 32) {
        const int p = p0 + lane;
        const uint32_t v = p < LA ? c.dres[c.alst[p]] : 0u;
        const uint32_t incl = fti_warp_incl_u32(v, lane) + carry;
        if (p < LA) c.dcum[p] = incl;
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    carry = 0;
    for (int p0 = 0; p0 < LB; p0 += 32) {
        const int p = p0 + lane;
        const uint32_t v = p < LB ? c.qres[c.blst[p]] : 0u;
        const uint32_t incl = fti_warp_incl_u32(v, lane) + carry;
        if (p < LB) c.qcum[p] = incl;
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    if (lane < nh) {   // per node: bases and T = min of the two totals under it
        const uint32_t ds = nDS[lane], qs = nQS[lane];
        const uint32_t ba = ds ? c.dcum[ds - 1] : 0u, bb = qs ? c.qcum[qs - 1] : 0u;
        const uint32_t ta = c.dcum[ds + nDL[lane] - 1] - ba, tb = c.qcum[qs + nQL[lane] - 1] - bb;
        nBA[lane] = ba; nBB[lane] = bb; nT[lane] = ta < tb ? ta : tb;
    }
    __syncwarp();
    for (int p = lane; p < LA; p += 32) {
        const int i = c.aseg[p];
        const uint32_t ba = nBA[i], T = nT[i], ds = nDS[i];
        const uint32_t hi_a = c.dcum[p] - ba;
        const uint32_t lo_a = (uint32_t)p > ds ? c.dcum[p - 1] - ba : 0u;
        const uint32_t end = hi_a < T ? hi_a : T;
        if (lo_a >= end) continue;
        const uint32_t bb = nBB[i], qs = nQS[i];
        int lo = (int)qs, hi = (int)(qs + nQL[i]);
        while (lo < hi) {   // first j of the node's query items with cum > lo_a
            const int mid = (lo + hi) >> 1;
            if (c.qcum[mid] - bb > lo_a) hi = mid; else lo = mid + 1;
        }
        const uint32_t x = c.dvoc[c.alst[p]] & FTI_VOCAB_MASK;
        const int jend = (int)(qs + nQL[i]);
        for (int j = lo; j < jend; j++) {
            const uint32_t lo_b = (uint32_t)j > qs ? c.qcum[j - 1] - bb : 0u;
            if (lo_b >= end) break;
            const uint32_t hi_b = c.qcum[j] - bb;
            const uint32_t s0 = lo_b > lo_a ? lo_b : lo_a;
            const uint32_t s1 = hi_b < end ? hi_b : end;
            if (s1 > s0) {
                const uint32_t eta = s1 - s0;
                const int jq = c.blst[j];
                const uint32_t y = c.qitem[jq].x & FTI_VOCAB_MASK;
                if (x != y) cost += (double)eta * (double)pair_dist(c, x, y, jq);
                emit<EXPORT>(*c.a, x, y, eta, nID[i]);
            }
        }
    }
    __syncwarp();
    for (int p = lane; p < LA; p += 32) {
        const int i = c.aseg[p];
        const uint32_t ba = nBA[i], T = nT[i];
        const uint32_t hi = c.dcum[p] - ba, lo = (uint32_t)p > nDS[i] ? c.dcum[p - 1] - ba : 0u;
        c.dres[c.alst[p]] = hi <= T ? 0u : hi - (lo > T ? lo : T);
    }
    for (int p = lane; p < LB; p += 32) {
        const int i = c.bseg[p];
        const uint32_t bb = nBB[i], T = nT[i];
        const uint32_t hi = c.qcum[p] - bb, lo = (uint32_t)p > nQS[i] ? c.qcum[p - 1] - bb : 0u;
        c.qres[c.blst[p]] = hi <= T ? 0u : hi - (lo > T ? lo : T);
    }
    __syncwarp();
}

// The root northwest corner as a warp-parallel stable merge ("merge path") of the two cumulative
// breakpoint lists SA (doc, vocab order) and SB (query, vocab order).  Walking the merged
// sequence, the segment between consecutive breakpoints [m_t, m_{t+1}) belongs to the doc item a
// and the query item b not yet consumed — exactly the triples of the sequential two-pointer
// (zero-residual items give empty segments).  Each lane walks a contiguous range of the merged
// sequence, found by one merge-path binary search; the flow is priced in FP32 per lane and
// accumulated in FP64.  No residual update is needed after the root.
template <bool EXPORT>
__device__ void root_merge(const PairCtx& c, int la, int lb, int lane, double& cost) {
    uint32_t carry = 0;
    for (int p0 = 0; p0 < la; p0 += 32) {
        int p = p0 + lane;
        uint32_t v = p < la ? c.dres[p] : 0u;
        uint32_t incl = fti_warp_incl_u32(v, lane) + carry;
        if (p < la) c.dcum[p] = incl;
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    carry = 0;
    for (int p0 = 0; p0 < lb; p0 += 32) {
        int p = p0 + lane;
        uint32_t v = p < lb ? c.qres[p] : 0u;
        uint32_t incl = fti_warp_incl_u32(v, lane) + carry;
        if (p < lb) c.qcum[p] = incl;
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const int L = la + lb;
    const int per = (L + 31) >> 5;
    const int t0 = min(L, lane * per), t1 = min(L, t0 + per);
    float acc = 0.f;
    if (t0 < t1) {
        int lo = max(0, t0 - lb), hi = min(t0, la);
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            const int b = t0 - mid;
            if (b == lb || c.dcum[mid - 1] <= c.qcum[b]) lo = mid; else hi = mid - 1;
        }
        int ai = lo, bi = t0 - lo;
        const uint32_t ma = ai ? c.dcum[ai - 1] : 0u, mb = bi ? c.qcum[bi - 1] : 0u;
        uint32_t m = ma > mb ? ma : mb;
        if (c.trow_base) {
            // table pricing in batches of RB triples: walk the merge (shared memory only), then issue
            // every vocab-map load, then every table load, so a batch pays two memory latencies
            // instead of two per triple; the FP32 accumulation order is the sequential one
            constexpr int RB = 4;
            const FtArgs& fa = *c.a;
            for (int tb = t0; tb < t1; tb += RB) {
                uint32_t ex[RB], xv[RB];
                int jv[RB];
#pragma unroll
                for (int u = 0; u < RB; u++) {
                    ex[u] = 0u; xv[u] = 0u; jv[u] = 0;
                    if (tb + u < t1) {
                        const uint32_t va = ai < la ? c.dcum[ai] : 0xFFFFFFFFu;
                        const uint32_t vb = bi < lb ? c.qcum[bi] : 0xFFFFFFFFu;
                        const bool takeA = va <= vb;
                        const uint32_t nxt = takeA ? va : vb;
                        if (nxt > m && ai < la && bi < lb) {
                            const uint32_t x = c.dvoc[ai] & FTI_VOCAB_MASK;
                            const uint32_t y = c.qitem[bi].x & FTI_VOCAB_MASK;
                            if (x != y) { ex[u] = nxt - m; xv[u] = x; jv[u] = bi; }
                            emit<EXPORT>(fa, x, y, nxt - m, 0u);
                        }
                        m = nxt;
                        if (takeA) ai++; else bi++;
                    }
                }
                uint32_t rv[RB];
                if (c.map) {
                    uint2 mw[RB];
#pragma unroll
                    for (int u = 0; u < RB; u++) mw[u] = ex[u] ? c.map[xv[u] >> 5] : make_uint2(0u, 0u);
#pragma unroll
                    for (int u = 0; u < RB; u++) rv[u] = mw[u].y + __popc(mw[u].x & ((1u << (xv[u] & 31)) - 1u));
                } else {
#pragma unroll
                    for (int u = 0; u < RB; u++) rv[u] = xv[u];
                }
                float dv[RB];
#pragma unroll
                for (int u = 0; u < RB; u++) {
                    FTI_ASSERT(!ex[u] || (jv[u] < (int)c.tld && (!fa.tab.rowcnt || (int)rv[u] < fa.tab.rowcnt[c.q])));
                    dv[u] = ex[u] ? c.trow_base[(int64_t)rv[u] * c.tld + jv[u]] : 0.f;
                }
#pragma unroll
                for (int u = 0; u < RB; u++)
                    if (ex[u]) acc = fmaf((float)ex[u], dv[u], acc);
            }
        } else
        for (int t = t0; t < t1; t++) {
            const uint32_t va = ai < la ? c.dcum[ai] : 0xFFFFFFFFu;
            const uint32_t vb = bi < lb ? c.qcum[bi] : 0xFFFFFFFFu;
            const bool takeA = va <= vb;
            const uint32_t nxt = takeA ? va : vb;
            if (nxt > m && ai < la && bi < lb) {
                const uint32_t eta = nxt - m;
                const uint32_t x = c.dvoc[ai] & FTI_VOCAB_MASK;
                const uint32_t y = c.qitem[bi].x & FTI_VOCAB_MASK;
                if (x != y) acc = fmaf((float)eta, pair_dist(c, x, y, bi), acc);
                emit<EXPORT>(*c.a, x, y, eta, 0u);
            }
            m = nxt;
            if (takeA) ai++; else bi++;
        }
    }
    cost += (double)acc;
}

template <bool EXPORT>
__global__ void __launch_bounds__(FT_WARPS * 32, 4) k_flowtree(FtArgs a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int q = a.q0 + (int)blockIdx.y;
    const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    // shared layout: qitem[Sq] uint2 | vocab lookup: bitmap[nw] + rank[nw] u32, or hash[vh_cap] uint2 |
    //                Y[Sq*d] f32 (small d) | per-warp u32 arrays
    uint2* qitem = (uint2*)smraw;
    uint32_t* bits = (uint32_t*)(qitem + a.Sq);
    uint32_t* rank = bits + a.nwords;
    uint2* vh = (uint2*)(qitem + a.Sq);
    float* Y = a.use_bitmap ? (float*)(rank + a.nwords) : (float*)(vh + a.L.vh_cap);
    uint32_t* wbase = (uint32_t*)(Y + (a.small_d ? a.Sq * a.d : 0));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per_warp = ft_per_warp_words(a.Sd, a.Sq);
    uint32_t* wsm = wbase + warp * per_warp;

    const uint32_t sq = hdr->s, U = hdr->U, vh_mask = hdr->vh_mask, mh_mask = hdr->mh_mask;
    const bool qok = hdr->err == 0 && sq > 0;
    const uint2* gitems = (const uint2*)(slot + a.L.off_items);
    const uint2* gvh = (const uint2*)(slot + a.L.off_vh);
    const uint4* gmh = (const uint4*)(slot + a.L.off_mh);
    const uint16_t* gml = (const uint16_t*)(slot + a.L.off_ml);
    for (int i = threadIdx.x; i < (int)sq; i += blockDim.x) qitem[i] = gitems[i];
    if (a.use_bitmap) {
        // query vocab bitmap with per-word rank: rank(x) = index of x among the sorted query ids
        for (int i = threadIdx.x; i < a.nwords; i += blockDim.x) bits[i] = 0u;
        __syncthreads();
        for (int i = threadIdx.x; i < (int)sq; i += blockDim.x) {
            const uint32_t x = gitems[i].x & FTI_VOCAB_MASK;
            atomicOr(&bits[x >> 5], 1u << (x & 31));
        }
        __syncthreads();
        __shared__ int tmp[32];
        int run = 0;
        for (int c0 = 0; c0 < a.nwords; c0 += blockDim.x) {
            const int w = c0 + threadIdx.x;
            const int v = w < a.nwords ? __popc(bits[w]) : 0;
            int tot;
            const int r = run + fti_block_exclusive_sum(v, tmp, &tot);
            if (w < a.nwords) rank[w] = (uint32_t)r;
            run += tot;
        }
    } else {
        for (int i = threadIdx.x; i <= (int)vh_mask; i += blockDim.x) vh[i] = gvh[i];
    }
    if (a.small_d) {
        for (int i = threadIdx.x; i < (int)sq * a.d; i += blockDim.x) {
            int j = i / a.d, t = i - j * a.d;
            Y[i] = a.X[(int64_t)(gitems[j].x & FTI_VOCAB_MASK) * a.d + t];
        }
    }
    __syncthreads();

    PairCtx c;
    c.a = &a;
    c.q = q;
    c.qitem = qitem;
    c.Y = a.small_d ? Y : nullptr;
    c.dvoc = wsm;
    c.dres = wsm + a.Sd;
    c.dcum = wsm + 2 * a.Sd;
    c.qres = wsm + 3 * a.Sd;
    c.qcum = wsm + 3 * a.Sd + a.Sq;
    c.nb = wsm + 3 * a.Sd + 2 * a.Sq;
    c.alst = (uint16_t*)(c.nb + 256);
    c.blst = c.alst + ((a.Sd + 1) & ~1);
    c.aseg = (uint8_t*)(c.blst + ((a.Sq + 1) & ~1));
    c.bseg = c.aseg + ((a.Sd + 3) & ~3);
    c.gml = (const uint16_t*)(slot + a.L.off_ml);
    c.trow_base = a.tab.table ? a.tab.table + a.tab.row_base[q] : nullptr;
    c.tld = a.tab.table ? (uint32_t)a.tab.pitch[q] : 0u;
    c.map = a.tab.map ? a.tab.map + (int64_t)q * ((a.N + 31) / 32) : nullptr;

    unsigned long long ubytes = 0;
    // range mode: this CTA's contiguous doc range; list mode: the pairs k_ftd handed over
    const bool list_mode = a.fb_list != nullptr;
    const int64_t d0 = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t d1 = min(a.n_docs, d0 + a.docs_per_cta);
    const int nwarp = (int)(blockDim.x >> 5);
    const int64_t e0 = list_mode ? (int64_t)blockIdx.x * nwarp + warp : d0 + warp;
    const int64_t e1 = list_mode ? (int64_t)a.fb_cnt[q] : d1;
    const int64_t estep = list_mode ? (int64_t)gridDim.x * nwarp : nwarp;
    for (int64_t e = e0; e < e1; e += estep) {
        const int64_t dp = list_mode ? (int64_t)a.fb_list[(int64_t)q * a.fb_cap + e] : e;
        const int64_t doc = a.docs ? a.docs[(int64_t)q * a.docs_ld + dp] : dp;
        double* outp = a.out ? a.out + (int64_t)q * a.out_ld + dp : nullptr;
        if (!qok || doc < 0 || doc >= a.n) {
            // a negative candidate (padding, or a doc another shard owns) scores +inf; an invalid
            // query or a doc index ≥ n scores NaN
            if (lane == 0 && outp)
                *outp = (qok && doc < 0) ? __longlong_as_double(0x7ff0000000000000ll)
                                         : __longlong_as_double(0x7ff8000000000000ll);
            if (lane == 0 && qok && doc >= a.n) atomicOr(a.err, FTI_ERR_RANGE);
            continue;
        }
        const uint32_t i0 = a.doc_off[doc];
        const int s = (int)(a.doc_off[doc + 1] - i0);
        const uint32_t W = a.Wd[doc];
        for (int i = lane; i < s; i += 32) {
            const uint2 it = a.items[i0 + i];
            c.dvoc[i] = it.x;
            c.dres[i] = it.y * U;
        }
        for (int j = lane; j < (int)sq; j += 32) c.qres[j] = qitem[j].y * W;
        __syncwarp();
        double cost = 0.0;
        // ---- phase A: self matches at singleton leaves ----
        for (int i = lane; i < s; i += 32) {
            const uint32_t v = c.dvoc[i];
            if (v & FTI_FLAG_MULTI_LEAF) continue;
            const uint32_t x = v & FTI_VOCAB_MASK;
            int jq = -1;
            if (a.use_bitmap) {
                const uint32_t w = bits[x >> 5], bm = 1u << (x & 31);
                if (w & bm) jq = (int)(rank[x >> 5] + __popc(w & (bm - 1u)));
            } else {
                uint32_t h = fti_hash(x) & vh_mask;
                while (true) {
                    const uint2 e = vh[h];
                    if (e.x == x) { jq = (int)e.y; break; }
                    if (e.x == FTI_EMPTY) break;
                    h = (h + 1) & vh_mask;
                }
            }
            if (jq >= 0) {
                const uint32_t dr = c.dres[i], qr = c.qres[jq];
                const uint32_t eta = dr < qr ? dr : qr;
                c.dres[i] = dr - eta;
                c.qres[jq] = qr - eta;
                if (EXPORT && eta) emit<EXPORT>(a, x, x, eta, (uint32_t)a.path[(int64_t)x * a.cols + a.leaf_depth[x]]);
            }
        }
        __syncwarp();
        // ---- phase B: common M-nodes, deepest first ----
        const uint32_t m0 = a.mn_off[doc], m1 = a.mn_off[doc + 1];
        if (m1 > m0 && hdr->n_mn > 0) {
            // records are ordered (depth desc, node asc): chunks of ≤ 32 records of one depth
            uint32_t cb = m0;
            while (cb < m1) {
                const uint32_t r = cb + lane;
                uint4 rec = make_uint4(0, 0, 0, 0xFFFFFFFFu), qe = make_uint4(0, 0, 0, 0);
                if (r < m1) rec = a.mnodes[r];
                const uint32_t dep0 = __shfl_sync(0xffffffffu, rec.w, 0);
                const int nrec = __popc(__ballot_sync(0xffffffffu, r < m1 && rec.w == dep0));
                bool hit = false;
                if (lane < nrec) {
                    uint32_t h = fti_hash(rec.x) & mh_mask;
                    while (true) {
                        const uint4 e = gmh[h];
                        if (e.x == rec.x) { qe = e; hit = true; break; }
                        if (e.x == FTI_EMPTY) break;
                        h = (h + 1) & mh_mask;
                    }
                }
                if (FT_BATCH_B) {
                    batch_nw<EXPORT>(c, rec, qe, hit, lane, cost);
                } else {
                    unsigned hm = __ballot_sync(0xffffffffu, hit);
                    while (hm) {
                        const int l = __ffs(hm) - 1;
                        hm &= hm - 1;
                        const uint32_t node = __shfl_sync(0xffffffffu, rec.x, l);
                        const uint32_t dlo = __shfl_sync(0xffffffffu, rec.y, l);
                        const uint32_t dln = __shfl_sync(0xffffffffu, rec.z, l);
                        const uint32_t qlo = __shfl_sync(0xffffffffu, qe.y, l);
                        const uint32_t qln = __shfl_sync(0xffffffffu, qe.z, l);
                        nw_corner<EXPORT>(c, a.mlists + dlo, (int)dln, gml + qlo, (int)qln, node, lane, cost);
                    }
                }
                cb += (uint32_t)nrec;
            }
        }
        // ---- phase C: the root ----
        root_merge<EXPORT>(c, s, (int)sq, lane, cost);
        cost = fti_warp_sum_f64(cost);
        ubytes += 8ull * (unsigned long long)s + 16ull;
        if (lane == 0 && outp) *outp = cost / (double)((unsigned long long)W * U);
        __syncwarp();
    }
    if (a.units && lane == 0 && ubytes) atomicAdd(a.units, ubytes);
}

}  // namespace

cudaError_t fti_launch_ft(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                          const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, const FtTable& tab, double* d_out,
                          int64_t out_ld, uint32_t* d_flow, uint32_t* d_flowcnt, int32_t flow_cap, cudaStream_t st) {
    if (nq <= 0 || n_docs <= 0) return cudaSuccess;
    const ft_index* ix = ds->ix;
    FtArgs a{};
    a.doc_off = ds->doc_off; a.items = ds->items; a.Wd = ds->W;
    a.mn_off = ds->mn_off; a.mnodes = ds->mnodes; a.mlists = ds->mlists;
    a.X = ix->X; a.d = ix->d; a.path = ix->path; a.cols = ix->d_star + 1; a.leaf_depth = ix->leaf_depth;
    a.N = ix->N;
    a.qblock = d_qblock; a.L = L; a.nq = nq;
    a.docs = d_docs; a.docs_ld = docs_ld; a.n_docs = n_docs;
    a.tab = tab;
    a.out = d_out; a.out_ld = out_ld;
    a.flow = d_flow; a.flowcnt = d_flowcnt; a.flow_cap = flow_cap;
    a.Sd = ds->max_s;
    a.Sq = L.smax;
    a.n = ds->n;
    a.err = ds->err_dev;
    a.units = d_flow ? nullptr : ds->units_ptr(FTI_ST_FT);
    a.small_d = (tab.table == nullptr && ix->d <= FTI_SMALL_D) ? 1 : 0;
    int64_t per_cta_target = std::max<int64_t>(FT_WARPS, (n_docs * nq + 148 * 16 - 1) / (148 * 16));
    int64_t bx = std::max<int64_t>(1, (n_docs + per_cta_target - 1) / per_cta_target);
    bx = std::max<int64_t>(bx, 1);
    a.docs_per_cta = (n_docs + bx - 1) / bx;
    bx = (n_docs + a.docs_per_cta - 1) / a.docs_per_cta;
    // FT_OPT_VOCAB_HASH (test option) forces the hash lookup used when N exceeds the bitmap limit
    a.use_bitmap = (ix->N <= FT_BITMAP_MAX_N && !fti_opt(FT_OPT_VOCAB_HASH)) ? 1 : 0;
    a.nwords = (int)((ix->N + 31) / 32);
    const size_t lookup = a.use_bitmap ? (size_t)a.nwords * 8 : (size_t)L.vh_cap * 8;
    const size_t ysm = a.small_d ? (size_t)a.Sq * a.d * 4 : 0;
    // per-warp residual arrays: fewer warps per CTA when large supports would exceed the
    // shared-memory limit (227 KB); FT_ERANGE-class failure when even one warp does not fit
    const size_t per_warp = (size_t)ft_per_warp_words(a.Sd, a.Sq) * 4;
    const size_t fixed = (size_t)a.Sq * 8 + lookup + ysm;
    int warps = FT_WARPS;
    while (warps > 1 && fixed + warps * per_warp > FT_SMEM_MAX) warps--;
    if (fixed + warps * per_warp > FT_SMEM_MAX) return cudaErrorInvalidConfiguration;
    const size_t smem = fixed + warps * per_warp;
    cudaError_t e;
    // with a distance table and a star-like tree, the lane-per-pair kernel (ft_flowd.cu) scores
    // every pair it can and lists the rest for this kernel (list mode)
    if (!d_flow && tab.table && a.use_bitmap && ds->n_mn <= 2 * ds->n && L.smax <= FTD_MAX_SQ &&
        !fti_opt(FT_OPT_WARP_ONLY)) {
        uint32_t* fl = nullptr;
        uint32_t* fc = nullptr;
        e = fti_launch_ftd(ds, L, d_qblock, nq, d_docs, docs_ld, n_docs, tab, d_out, out_ld, &fl, &fc, st);
        if (e == cudaSuccess) {
            a.fb_list = fl;
            a.fb_cnt = fc;
            a.fb_cap = n_docs;
            bx = std::max<int64_t>(1, std::min<int64_t>(32, (148 * 4 + nq - 1) / nq));
        } else if (e != cudaErrorNotSupported) {
            if (fti_opt(FT_OPT_DEBUG)) fprintf(stderr, "fti_launch_ft: k_ftd launch failed: %s\n", cudaGetErrorString(e));
            return e;
        }
    }
    auto kern = d_flow ? k_flowtree<true> : k_flowtree<false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    for (int32_t q0 = 0; q0 < nq; q0 += 65535) {          // grid.y ≤ 65535 queries per launch
        a.q0 = q0;
        kern<<<dim3((unsigned)bx, (unsigned)std::min(65535, nq - q0)), warps * 32, smem, st>>>(a);
        fti_count_launches(1);
    }
    return cudaGetLastError();
}
