// ft_flowd.cu — a6 with LANE = PAIR: the Flowtree estimate (§3; greedy flow
// PAPER.md:495-504) of 32 (query, doc) pairs per warp that share the query.
//
// A CTA works for one query over a strided range of candidate positions: the query's items and its
// vocab bitmap + per-word rank (query item index of an id) sit in shared memory; a compact
// candidate table's row map ({bits, rank} per 32 vocab ids) is read through L2.  Lane l of a warp
// scores the pair (q, docs[position l]) on its own:
//   * M-nodes: a cell with ≥ 2 ground points present on both sides where both keep residual mass
//     after the leaves' self matches (so phase B of the warp kernel would match there) hands the
//     pair to the warp kernel (list mode), as do pairs with more than DCAP shared ids;
//   * self matches (reading R8): one pass over the doc items tests the query bitmap and queues the
//     shared ids {doc index i, query index j} in increasing vocab order (sentinels end the queue);
//   * root: the northwest corner over the residuals in vocab order (reading R10) as a sequential
//     merge, branch free, one triple per step; the merge advances in warp-uniform batches of DRB
//     steps, after which every lane issues its DRB table gathers together (software pipelined one
//     batch deep).  Uniform weights (every doc and query mass 1: the text / reviews / stress
//     workloads) take a lean step over the two sides' cumulative residual boundaries E, F:
//     η = min(E, F) − previous boundary, the side(s) whose boundary was reached advance; each item
//     carries U (doc) or W (query), a shared id's leftover is U − min(U, W) or W − min(U, W); the
//     doc side reads its shared flag from the query bitmap while the next item is prepared, and
//     only the query side consumes the queue.
// All pairs of a CTA read one query's table, so the gathers of a warp hit one L2-resident table.
// Masses are exact u32 (reading R13), distances FP32 from the a5 table, sums FP32 per batch and FP64
// across batches.  EXPORT: the flow triples (src, dst, η, node) are written out instead of priced
// (ft_flowtree_flow's parity hook).
#include <algorithm>

#include "ft_device.cuh"

namespace {

// CTAs per SM the register budget allows: 3 (80 registers) when every vocab id is a table row
// (exhaustive scoring), 2 (111 registers) with a compact table's row map (the prefiltered
// pipeline: 0.72 → 0.67 ms per reviews batch; exhaustive scoring prefers 3: 2.88 vs 2.93 ms)
#ifndef FTD_MINB
#define FTD_MINB 3
#endif
#ifndef FTD_MINB_MAP
#define FTD_MINB_MAP 2
#endif
constexpr int DW = 8;      // warps per CTA
#ifndef FTD_DCAP
#define FTD_DCAP 48
#endif
constexpr int DCAP = FTD_DCAP;   // shared ids per pair held in the per-lane queue
constexpr int DQN = DCAP + 2;            // queue slots per lane: entries + two sentinels
#ifndef FTD_DRB
#define FTD_DRB 8
#endif
#ifndef FTD_PREV
#define FTD_PREV 1       // pre-pass reads the doc records with 32-byte loads (0: one 4-byte load per record)
#endif

constexpr int DRB = FTD_DRB;   // merge steps per gather batch
constexpr uint32_t DQ_END = 0xFFFFu;     // queue sentinel: i = j = 255 never matches (s, sq ≤ 254)

struct DArgs {
    const uint32_t* doc_off;
    const uint2* items;
    const uint32_t* Wd;
    int64_t nnz;               // records in items (followed by 8 zero records of padding)
    const uint32_t* mn_off;
    const uint4* mnodes;
    const uint16_t* mlists;
    const uint8_t* qblock;
    QueryLayout L;
    int32_t q0;
    const int64_t* docs;       // [nq][docs_ld] candidate docs, or null (position = doc)
    int64_t docs_ld, n_docs, n;
    const float* table;
    const uint2* map;          // [nq][nw] {bits, rank} rows of the compact table, or null (row = vocab id)
    const int64_t* row_base;   // [nq] ELEMENT offset of each query's table
    const int32_t* pitch;      // [nq] per-query row pitch (floats)
    const int32_t* rowcnt;     // [nq] table rows (compact tables), or null: n_rows (FTI_CHECKED bounds only)
    int64_t n_rows;
    int32_t nw, Sq;
    int unit_w;                // every doc weight is 1
    double* out;
    int64_t out_ld;
    uint32_t* fb_list;
    uint32_t* fb_cnt;
    int64_t fb_cap;
    uint32_t* err;
    unsigned long long* units;
    // EXPORT: flow triples {src, dst, η, node} and their count; path table for the leaf nodes
    uint32_t* flow;
    uint32_t* flowcnt;
    int32_t flow_cap;
    const int32_t* path;
    int32_t cols;
    const uint8_t* leaf_depth;
};

template <bool EXPORT>
__device__ __forceinline__ void ftd_emit(const DArgs& a, uint32_t x, uint32_t y, uint32_t eta, uint32_t node) {
    if (EXPORT) {
        const uint32_t idx = atomicAdd(a.flowcnt, 1u);
        if ((int)idx < a.flow_cap) {
            a.flow[4 * idx + 0] = x;
            a.flow[4 * idx + 1] = y;
            a.flow[4 * idx + 2] = eta;
            a.flow[4 * idx + 3] = node;
        }
    }
}

// MAP: the table is compact (rows = the candidates' vocabulary, looked up in the row map)
template <bool EXPORT, bool MAP>
__global__ void __launch_bounds__(DW * 32, MAP ? FTD_MINB_MAP : FTD_MINB) k_ftd(DArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int q = a.q0 + (int)blockIdx.y;
    const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    // shared: qitem[Sq] uint2 | qbits[nw] | qrank[nw] | queue[DW][DQN][32] u16
    uint2* qitem = (uint2*)sm;
    uint32_t* qbits = (uint32_t*)(qitem + a.Sq);
    uint32_t* qrank = qbits + a.nw;
    uint16_t* queue = (uint16_t*)(qrank + a.nw);
    const uint32_t sq = hdr->s, U = hdr->U, mh_mask = hdr->mh_mask;
    const bool qok = hdr->err == 0 && sq > 0;
    const uint2* gitems = (const uint2*)(slot + a.L.off_items);
    for (int i = threadIdx.x; i < (int)sq; i += blockDim.x) qitem[i] = gitems[i];
    for (int i = threadIdx.x; i < a.nw; i += blockDim.x) qbits[i] = 0u;
    __syncthreads();
    // bitmap of the query's ids; rank[w] = index of the first query item in word w (items are
    // sorted by id, so an id's item index is rank[w] + the bits below it).  Only words holding a
    // query id are ever ranked.
    for (int i = threadIdx.x; i < (int)sq; i += blockDim.x) {
        const uint32_t x = gitems[i].x & FTI_VOCAB_MASK;
        atomicOr(&qbits[x >> 5], 1u << (x & 31));
        if (i == 0 || ((gitems[i - 1].x & FTI_VOCAB_MASK) >> 5) != (x >> 5)) qrank[x >> 5] = (uint32_t)i;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint16_t* myq = queue + warp * DQN * 32 + lane;
    const float* trow = a.table ? a.table + a.row_base[q] : nullptr;
    const uint32_t ld = a.table ? (uint32_t)a.pitch[q] : 0u;   // row pitch
    const int64_t tab_elems = FTI_CHECKED && a.table ? (int64_t)ld * (a.rowcnt ? a.rowcnt[q] : a.n_rows) : 0;
    const uint2* gmapq = a.map ? a.map + (int64_t)q * a.nw : nullptr;
    const uint4* gmh = (const uint4*)(slot + a.L.off_mh);
    const uint16_t* gml = (const uint16_t*)(slot + a.L.off_ml);
    const bool qmn = hdr->n_mn > 0;
    // uniform weights on both sides (every mass 1): the lean merge
    const bool uni = a.unit_w && U == sq;
    unsigned ubytes = 0;
    __shared__ int shist[260];
    __shared__ uint16_t sperm[DW * 32];
    // table row offset of vocab id x (compact table: its candidate-vocabulary rank)
    auto row_off = [&](uint32_t x) -> uint32_t {
        uint32_t row = x;
        if (MAP) {
            const uint2 mw = __ldg(gmapq + (x >> 5));
            row = mw.y + __popc(mw.x & ((1u << (x & 31)) - 1u));
        }
        return row * ld;
    };
    const int64_t stride = (int64_t)gridDim.x * DW * 32;
    for (int64_t cbase = (int64_t)blockIdx.x * DW * 32; cbase < a.n_docs; cbase += stride) {
        // the CTA's DW*32 positions sorted by doc support size, so the lanes of a warp run merges
        // of similar length (the warp steps until its longest pair is done)
        // (a counting sort on the size: ≤ 254, 256 = past the end)
        int tpos;
        {
            const int64_t p = cbase + threadIdx.x;
            uint32_t key = 256u;
            if (p < a.n_docs) {
                const int64_t doc = a.docs ? a.docs[(int64_t)q * a.docs_ld + p] : p;
                key = (doc >= 0 && doc < a.n) ? a.doc_off[doc + 1] - a.doc_off[doc] : 0u;
            }
            tpos = fti_counting_rank(key, shist, sperm);
        }
        const int64_t dp = cbase + tpos;
        bool active = false;
        int s = 0;
        uint32_t i0 = 0, W = 0;
        double* outp = nullptr;
        int64_t doc = -1;
        if (dp < a.n_docs) {
            doc = a.docs ? a.docs[(int64_t)q * a.docs_ld + dp] : dp;
            outp = a.out ? a.out + (int64_t)q * a.out_ld + dp : nullptr;
            if (!qok || doc < 0 || doc >= a.n) {
                // a negative candidate (padding, or a doc another shard owns) scores +inf; an invalid
                // query or a doc index ≥ n scores NaN (as the warp kernel)
                if (outp)
                    *outp = (qok && doc < 0) ? __longlong_as_double(0x7ff0000000000000ll)
                                             : __longlong_as_double(0x7ff8000000000000ll);
                if (qok && doc >= a.n) atomicOr(a.err, FTI_ERR_RANGE);
            } else {
                i0 = a.doc_off[doc];
                s = (int)(a.doc_off[doc + 1] - i0);
                W = a.Wd[doc];
                active = true;
            }
        }
        // shared ids, in vocab order: {i | j << 8}, then two sentinels
        int nc = 0;
        if (active) {
#if FTD_PREV
            // 32-byte loads of four records each from the aligned-down start: a lane's request is one
            // sector whatever its width, and the L1 serves about one lane request per clock
            // (exhaustive reviews 2.88 -> 2.62 ms, text 0.537 -> 0.505, stress 6.00 -> 5.67)
            const int ia = -(int)(i0 & 3u);
            for (int i = ia; i < s; i += 8) {
                uint32_t xv[8];
                {
                    uint32_t r[16];
                    const uint2* p = a.items + i0 + i;
                    asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                                 : "l"(p));
                    asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                 : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                                 : "l"(p + 4));
#pragma unroll
                    for (int u = 0; u < 8; u++) xv[u] = r[2 * u];
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const uint32_t x = xv[u] & FTI_VOCAB_MASK;
                    const uint32_t bw = qbits[x >> 5], bm = 1u << (x & 31);
                    if (i + u >= 0 && i + u < s && (bw & bm)) {
                        const uint32_t j = qrank[x >> 5] + __popc(bw & (bm - 1u));
                        if (nc < DCAP) myq[nc * 32] = (uint16_t)((uint32_t)(i + u) | (j << 8));
                        nc++;
                    }
                }
            }
#else
            for (int i = 0; i < s; i += 8) {
                uint32_t xv[8];
#pragma unroll
                for (int u = 0; u < 8; u++) xv[u] = i + u < s ? a.items[i0 + i + u].x : 0u;
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const uint32_t x = xv[u] & FTI_VOCAB_MASK;
                    const uint32_t bw = qbits[x >> 5], bm = 1u << (x & 31);
                    if (i + u < s && (bw & bm)) {
                        const uint32_t j = qrank[x >> 5] + __popc(bw & (bm - 1u));
                        if (nc < DCAP) myq[nc * 32] = (uint16_t)((uint32_t)(i + u) | (j << 8));
                        nc++;
                    }
                }
            }
#endif
            if (nc <= DCAP) {
                myq[nc * 32] = (uint16_t)DQ_END;
                myq[(nc + 1) * 32] = (uint16_t)DQ_END;
            }
        }
        if (active && nc > DCAP) active = false;
        // M-nodes (cells holding ≥ 2 ground points) on both sides: matching happens at such a node v
        // only if, after the self matches at the leaves, both sides keep residual mass under v.  When
        // no common M-node does, phase B changes nothing and the pair is a leaves + root flow; else
        // the pair goes to the warp kernel.  (If no node matches, the residuals each node sees are
        // the self-match residuals, so testing every node against them is exact.)
        if (active && qmn) {
            const uint32_t m0 = a.mn_off[doc], m1 = a.mn_off[doc + 1];
            const uint32_t* dw = (const uint32_t*)(a.items + i0) + 1;
            bool general = false;
            for (uint32_t r = m0; r < m1 && !general; r++) {
                const uint4 rec = a.mnodes[r];
                uint32_t h = fti_hash(rec.x) & mh_mask;
                uint4 qe = make_uint4(FTI_EMPTY, 0u, 0u, 0u);
                while (true) {
                    const uint4 e = gmh[h];
                    if (e.x == rec.x || e.x == FTI_EMPTY) { qe = e; break; }
                    h = (h + 1) & mh_mask;
                }
                if (qe.x != rec.x) continue;
                uint32_t dsum = 0u, qsum = 0u;
                bool multi_shared = false;
                for (uint32_t t = 0; t < rec.z; t++) {
                    const uint32_t ii = a.mlists[rec.y + t];
                    FTI_ASSERT(ii < (uint32_t)s);
                    const uint32_t xv = a.items[i0 + ii].x;
                    const uint32_t x = xv & FTI_VOCAB_MASK;
                    uint32_t m = dw[2 * ii] * U;
                    const uint32_t bw = qbits[x >> 5], bm = 1u << (x & 31);
                    if (bw & bm) {
                        // a shared id whose leaf holds ≥ 2 points is matched by that leaf's northwest
                        // corner, not by a self match: always the warp kernel
                        multi_shared |= (xv & FTI_FLAG_MULTI_LEAF) != 0u;
                        const uint32_t qm = qitem[qrank[x >> 5] + __popc(bw & (bm - 1u))].y * W;
                        m -= (qm < m ? qm : m);
                    }
                    dsum += m;
                }
                for (uint32_t t = 0; t < qe.z && dsum && !multi_shared; t++) {
                    const uint32_t jj = gml[qe.y + t];
                    FTI_ASSERT(qe.y + t < hdr->n_ml && jj < sq);
                    uint32_t m = qitem[jj].y * W;
                    for (int c = 0; c < nc; c++) {
                        const uint32_t e = myq[c * 32];
                        if ((e >> 8) == jj) {
                            const uint32_t dm = dw[2 * (e & 0xFFu)] * U;
                            m -= (dm < m ? dm : m);
                            break;
                        }
                    }
                    qsum += m;
                }
                general = multi_shared || (dsum > 0u && qsum > 0u);
            }
            if (general) active = false;
        }
        const bool to_list = dp < a.n_docs && !active && s > 0 && qok && doc >= 0 && doc < a.n;
        if (to_list) {
            const uint32_t pos = atomicAdd(&a.fb_cnt[q], 1u);
            FTI_ASSERT((int64_t)pos < a.fb_cap);
            a.fb_list[(int64_t)q * a.fb_cap + pos] = (uint32_t)dp;
        }
        const bool scored = active;
        const uint2* dit = a.items + i0;
        const uint32_t* dw = (const uint32_t*)dit + 1;   // weights, stride 2 words
        if (EXPORT && active) {
            // the leaves' self matches (singleton leaves: the pair stayed here)
            for (int c = 0; c < nc; c++) {
                const uint32_t e = myq[c * 32];
                const uint32_t x = dit[e & 0xFFu].x & FTI_VOCAB_MASK;
                const uint32_t dm = dw[2 * (e & 0xFFu)] * U, qm = qitem[e >> 8].y * W;
                ftd_emit<EXPORT>(a, x, x, dm < qm ? dm : qm, (uint32_t)a.path[(int64_t)x * a.cols + a.leaf_depth[x]]);
            }
        }
        double acc = 0.0;
        float pdv[DRB];
        uint32_t pef[DRB];
#pragma unroll
        for (int u = 0; u < DRB; u++) { pdv[u] = 0.f; pef[u] = 0u; }
        if (uni) {
            // ---- root northwest corner, uniform weights ----
            // E / F: cumulative residual boundary of the current doc item i / query item j; o:
            // table-row offset of item i; (rn, on): residual and offset of item i+1; x2: vocab id of
            // item i+2, x3..x5: raw records of items i+3..i+5 (read through pn, which may run past the
            // doc's end into valid records: the items array carries 8 zero records of padding).  A
            // shared doc item's leftover is U − min(U, W) (its flag comes from the query bitmap); the
            // query side takes its shared items from the queue (qh = query index of the next one).
            // Both sides carry the same total residual, so the merge ends when either side's last
            // item is consumed (no overflow: W·U ≤ 65535²).
            const uint32_t mm = U < W ? U : W, Ud = U - mm, Wq = W - mm;
            auto dres = [&](uint32_t x) { return ((qbits[x >> 5] >> (x & 31)) & 1u) ? Ud : U; };
            int i = 0, j = 0;
            uint32_t E = 0, F = 0, o = 0, rn = 0, on = 0, x2 = 0, x3 = 0, x4 = 0, x5 = 0, prev = 0, qh = 0xFFu;
            uint32_t qaddr = (uint32_t)__cvta_generic_to_shared(myq);   // queue head (64 B per entry)
            uint32_t xc = 0, xn = 0;   // EXPORT: vocab ids of items i, i+1
            const uint2* pn = dit + 6;
            if (active) {
                const uint32_t x0 = dit[0].x & FTI_VOCAB_MASK;
                const uint32_t x1 = dit[1].x & FTI_VOCAB_MASK;
                x2 = dit[2].x & FTI_VOCAB_MASK;
                x3 = dit[3].x;
                x4 = dit[4].x;
                x5 = dit[5].x;
                E = dres(x0);
                rn = dres(x1);
                o = EXPORT ? 0u : row_off(x0);
                on = EXPORT ? 0u : row_off(x1);
                xc = x0;
                xn = x1;
                qh = (uint32_t)myq[0] >> 8;
                const bool h0 = qh == 0u;
                F = h0 ? Wq : W;
                if (h0) { qaddr += 64u; qh = (uint32_t)myq[32] >> 8; }
            }
            while (__any_sync(0xffffffffu, active)) {
                uint32_t off[DRB], ef[DRB];
#pragma unroll
                for (int u = 0; u < DRB; u++) {
                    const uint32_t cur = E < F ? E : F;
                    const uint32_t eta = active ? cur - prev : 0u;
                    off[u] = o + (uint32_t)j;
                    ef[u] = eta;
                    if (EXPORT && eta) ftd_emit<EXPORT>(a, xc, qitem[j].x & FTI_VOCAB_MASK, eta, 0u);
                    prev = cur;
                    const bool ad = active && E == cur, aq = active && F == cur;
                    // doc side: item i+1 becomes current, item i+2 is prepared
                    E = ad ? E + rn : E;
                    o = ad ? on : o;
                    // (every lane: predicating these lookups on `ad` measured slower, 0.79 vs 0.76 ms;
                    // taking the doc side's shared flags from the queue instead of the bitmap, 2%)
                    const uint32_t r2 = dres(x2), o2 = EXPORT ? 0u : row_off(x2);
                    rn = ad ? r2 : rn;
                    on = ad ? o2 : on;
                    if (EXPORT) { xc = ad ? xn : xc; xn = ad ? x2 : xn; }
                    // raw records loaded three advances before use (x3..x5: items i+3..i+5): the
                    // record load's latency had been the merge's largest stall
                    // (a predicated inline-PTX load straight into x5's register, to avoid the select
                    // on the fresh load: 2.89 -> 3.10 ms exhaustive, not kept; two records per 16-byte
                    // load on every other advance: 2.88 -> 3.55 ms, not kept)
                    if (ad) {
                        x2 = x3 & FTI_VOCAB_MASK;
                        x3 = x4;
                        x4 = x5;
                        FTI_ASSERT(pn - a.items < a.nnz + 8);
                        x5 = pn->x;
                    }
                    pn += ad;
                    i += ad;
                    // query side: item j+1 becomes current (queue entries hold j ≤ 253; the sentinel 255)
                    const bool hq = aq && qh == (uint32_t)(j + 1);
                    F = aq ? F + (hq ? Wq : W) : F;
                    uint32_t ne;
                    asm("ld.shared.u16 %0, [%1];" : "=r"(ne) : "r"(qaddr + 64u));
                    qh = hq ? ne >> 8 : qh;
                    qaddr += hq ? 64u : 0u;
                    j += aq;
                    // the two sides carry the same total residual, so when either runs out every
                    // unit is matched: stop.  (Stopping only when BOTH were done let a finished doc
                    // side keep stepping while the record after the doc's last was a shared id
                    // with leftover U − min(U, W) = 0 — its boundary never grew, `ad` fired on
                    // every remaining query step and pn ran up to s_q records past the doc: beyond
                    // the array's padding after the dataset's last doc.  All those steps had η = 0.)
                    active = active && i < s && j < (int)sq;
                }
                if (!EXPORT) {
                    float part = 0.f;
#pragma unroll
                    for (int u = 0; u < DRB; u++) part = fmaf((float)pef[u], pdv[u], part);
                    acc += (double)part;
#pragma unroll
                    for (int u = 0; u < DRB; u++) {
                        FTI_ASSERT(!ef[u] || (int64_t)off[u] < tab_elems);
                        pdv[u] = ef[u] ? __ldg(trow + off[u]) : 0.f;
                        pef[u] = ef[u];
                    }
                }
            }
        } else {
            // ---- root northwest corner, general weights, lane-sequential, branch-free ----
            // (ra, ro): residual and table-row offset of doc item i; (ran, ron) item i+1; p2 / p3 the raw
            // records of items i+2 / i+3 (loaded two advances before use).  rb / rbn: residuals of query
            // items j / j+1.  ed / eq: the next queued shared id {i | j << 8} for the doc / query side;
            // eqw the doc weight of eq's item (loaded when eq is set, used at the query side's next hit).
            int i = 0, j = 0, cd = 0, cq = 0;
            uint32_t ed = nc > 0 ? (uint32_t)myq[0] : DQ_END, eq = ed, eqw = 0u;
            if (nc > 0) eqw = dw[2 * (eq & 0xFFu)];
            uint32_t ra = 0, ro = 0, ran = 0, ron = 0, rb = 0, rbn = 0, rx = 0, rxn = 0;
            uint2 p2 = make_uint2(0u, 0u), p3 = make_uint2(0u, 0u);
            // doc item ii from its record it: residual after its self match, and its table-row offset
            auto doc_prep = [&](const uint2 it, int ii, bool take, uint32_t& r_, uint32_t& o_, uint32_t& x_) {
                const uint32_t x = it.x & FTI_VOCAB_MASK;
                const uint32_t m = it.y * U;
                const bool hit = take && (ed & 0xFFu) == (uint32_t)ii;
                const uint32_t qm = qitem[(ed >> 8) & 0xFFu].y * W;
                const uint32_t adj = hit ? (qm < m ? qm : m) : 0u;
                cd += hit;
                const uint32_t ne = myq[cd * 32];
                ed = hit ? ne : ed;
                r_ = m - adj;
                o_ = EXPORT ? 0u : row_off(x);
                x_ = x;
            };
            // query item jj: residual after its self match
            auto q_prep = [&](int jj, bool take) {
                const uint32_t m = qitem[jj].y * W;
                const bool hit = take && ((eq >> 8) & 0xFFu) == (uint32_t)jj;
                const uint32_t dm = eqw * U;
                const uint32_t adj = hit ? (dm < m ? dm : m) : 0u;
                cq += hit;
                const uint32_t ne = myq[cq * 32];
                eq = hit ? ne : eq;
                if (hit && eq != DQ_END) eqw = dw[2 * (eq & 0xFFu)];
                return m - adj;
            };
            if (active) {
                const uint2 t0 = dit[0];
                const uint2 t1 = s > 1 ? dit[1] : t0;
                if (s > 2) p2 = dit[2];
                if (s > 3) p3 = dit[3];
                doc_prep(t0, 0, true, ra, ro, rx);
                doc_prep(t1, 1, s > 1, ran, ron, rxn);
                rb = q_prep(0, true);
                rbn = q_prep(sq > 1 ? 1 : 0, sq > 1);
            }
            const int sqm1 = (int)sq - 1;
            while (__any_sync(0xffffffffu, active)) {
                uint32_t off[DRB];
                uint32_t ef[DRB];
#pragma unroll
                for (int u = 0; u < DRB; u++) {
                    const uint32_t eta = active ? (ra < rb ? ra : rb) : 0u;
                    off[u] = ro + (uint32_t)j;
                    ef[u] = eta;
                    if (EXPORT && eta) ftd_emit<EXPORT>(a, rx, qitem[j].x & FTI_VOCAB_MASK, eta, 0u);
                    ra -= eta;
                    rb -= eta;
                    const bool ad = active && ra == 0u, aq = active && rb == 0u;
                    // doc side: item i+2 (record p2) becomes the prepared next item
                    uint32_t r2, o2, xx2;
                    doc_prep(p2, i + 2, ad && i + 2 < s, r2, o2, xx2);
                    ra = ad ? ran : ra;
                    ro = ad ? ron : ro;
                    rx = ad ? rxn : rx;
                    ran = ad ? r2 : ran;
                    ron = ad ? o2 : ron;
                    rxn = ad ? xx2 : rxn;
                    p2 = ad ? p3 : p2;
                    if (ad && i + 4 < s) p3 = dit[i + 4];
                    i += ad;
                    // query side: item j+2
                    const int j2 = j + 2 < (int)sq ? j + 2 : sqm1;
                    const uint32_t q2 = q_prep(j2, aq && j + 2 < (int)sq);
                    rb = aq ? rbn : rb;
                    rbn = aq ? q2 : rbn;
                    j += aq;
                    active = active && i < s && j < (int)sq;
                }
                if (!EXPORT) {
                    float part = 0.f;
#pragma unroll
                    for (int u = 0; u < DRB; u++) part = fmaf((float)pef[u], pdv[u], part);
                    acc += (double)part;
#pragma unroll
                    for (int u = 0; u < DRB; u++) {
                        FTI_ASSERT(!ef[u] || (int64_t)off[u] < tab_elems);
                        pdv[u] = ef[u] ? __ldg(trow + off[u]) : 0.f;
                        pef[u] = ef[u];
                    }
                }
            }
        }
        if (!EXPORT) {
            float part = 0.f;
#pragma unroll
            for (int u = 0; u < DRB; u++) part = fmaf((float)pef[u], pdv[u], part);
            acc += (double)part;
        }
        if (scored) {
            if (outp) *outp = EXPORT ? 0.0 : acc / (double)((unsigned long long)W * U);
            ubytes += 8u * (unsigned)s + 16u;
        }
    }
    if (a.units) {
        const unsigned tot = __reduce_add_sync(0xffffffffu, ubytes);
        if (lane == 0 && tot) atomicAdd(a.units, (unsigned long long)tot);
    }
}

}  // namespace

// Lane-per-pair Flowtree over n_docs candidate positions per query (d_docs, or all docs when
// null) with a distance table (or, with d_flow, exporting the flow triples instead of pricing).
// Pairs it cannot score are listed per query in fb_list / fb_cnt (capacity n_docs per query) for
// the warp kernel's list mode.  cudaErrorNotSupported when the geometry does not fit (supports >
// 255, N beyond the shared-memory bitmap).
cudaError_t fti_launch_ftd(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                           const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, const FtTable& tab, double* d_out,
                           int64_t out_ld, uint32_t** fb_list, uint32_t** fb_cnt, cudaStream_t st,
                           uint32_t* d_flow, uint32_t* d_flowcnt, int32_t flow_cap) {
    const ft_index* ix = ds->ix;
    const bool exp = d_flow != nullptr;
    if ((!tab.table && !exp) || ds->max_s > FTD_MAX_SQ || L.smax > FTD_MAX_SQ) return cudaErrorNotSupported;
    DArgs a{};
    a.nw = (int)((ix->N + 31) / 32);
    a.Sq = std::max(1, L.smax);
    const size_t smem = 8ull * a.Sq + 8ull * a.nw + 2ull * DW * DQN * 32;
    if (smem > 200 * 1024) return cudaErrorNotSupported;
    cudaError_t e;
    if ((e = ds->s_fblist.reserve((size_t)nq * n_docs * 4)) != cudaSuccess) return e;
    if ((e = ds->s_fbcnt.reserve((size_t)nq * 4)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ds->s_fbcnt.p, 0, (size_t)nq * 4, st)) != cudaSuccess) return e;
    a.doc_off = ds->doc_off; a.items = ds->items; a.Wd = ds->W;
    a.nnz = ds->nnz;
    a.mn_off = ds->mn_off; a.mnodes = ds->mnodes; a.mlists = ds->mlists;
    a.qblock = d_qblock; a.L = L;
    a.docs = d_docs; a.docs_ld = docs_ld; a.n_docs = n_docs; a.n = ds->n;
    a.table = exp ? nullptr : tab.table;
    a.map = exp ? nullptr : tab.map;
    a.row_base = tab.row_base; a.pitch = tab.pitch;
    a.rowcnt = tab.rowcnt; a.n_rows = ix->N;
    a.unit_w = ds->unit_w ? 1 : 0;
    a.out = d_out; a.out_ld = out_ld;
    a.fb_list = ds->s_fblist.as<uint32_t>(); a.fb_cnt = ds->s_fbcnt.as<uint32_t>(); a.fb_cap = n_docs;
    a.err = ds->err_dev;
    a.units = exp ? nullptr : ds->units_ptr(FTI_ST_FT);
    a.flow = d_flow; a.flowcnt = d_flowcnt; a.flow_cap = flow_cap;
    a.path = ix->path; a.cols = ix->d_star + 1; a.leaf_depth = ix->leaf_depth;
    auto kern = exp ? k_ftd<true, false> : (a.map ? k_ftd<false, true> : k_ftd<false, false>);
    // function attributes are per device; they are set only when they change
    constexpr int MAXDEV = 64;
    static thread_local int cur_smem[3][MAXDEV], cur_pct[3][MAXDEV];
    static thread_local bool init = false;
    if (!init) {
        for (int k = 0; k < 3; k++)
            for (int i = 0; i < MAXDEV; i++) cur_smem[k][i] = cur_pct[k][i] = -1;
        init = true;
    }
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if (dev >= MAXDEV) return cudaErrorInvalidDevice;
    const int ki = exp ? 2 : (a.map ? 1 : 0);
    if ((int)smem > cur_smem[ki][dev]) {
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
            return e;
        cur_smem[ki][dev] = (int)smem;
    }
    // the L1 caches the lanes' doc records between the pre-pass and the merge: give shared memory
    // only what the target CTAs per SM need
    {
        const size_t need = (size_t)(a.map ? FTD_MINB_MAP : FTD_MINB) * (smem + 2176 + 1024);
        int pct = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
        if (fti_opt(FT_OPT_FTD_CARVEOUT) > 0) pct = (int)fti_opt(FT_OPT_FTD_CARVEOUT);
        pct = std::min(100, pct);
        if (pct != cur_pct[ki][dev]) {
            if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct)) != cudaSuccess)
                return e;
            cur_pct[ki][dev] = pct;
        }
    }
    // one CTA per 256 positions, x fastest: the resident CTAs then cover one or two queries at a
    // time, so the table gathers of an exhaustive scan stay in L2 (a strided assignment spreading
    // the resident CTAs over ~32 queries took 7.7 GB of DRAM instead of 1.4 GB for 64 × 100k pairs)
    const int64_t gx = (n_docs + DW * 32 - 1) / (DW * 32);
    for (int32_t q0 = 0; q0 < nq; q0 += 65535) {
        a.q0 = q0;
        kern<<<dim3((unsigned)gx, (unsigned)std::min(65535, nq - q0)), DW * 32, smem, st>>>(a);
        fti_count_launches(1);
    }
    *fb_list = a.fb_list;
    *fb_cnt = a.fb_cnt;
    return cudaGetLastError();
}
