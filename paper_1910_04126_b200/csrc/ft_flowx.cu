// ft_flowx.cu — a6 for exhaustive scoring: the Flowtree estimate (§3; greedy flow
// PAPER.md:495-504) with LANE = QUERY over a chunk of 32 queries, every doc read once per chunk.
//
// The warp kernel (ft_flow.cu) spends a warp on each (query, doc) pair, so its time per pair is a
// chain of dependent shared/L2 accesses.  When every query scores every doc, a warp can instead
// take one doc for 32 queries at once: the doc's items are staged in shared memory once, and lane q
// runs the pair (q, doc) as a sequential two-pointer merge — the canonical flow of reading R10:
//   * self matches (phase A): an id present on both sides matches min(w U, u W) at its singleton
//     leaf.  Doc side: the chunk's union of query ids (bitmap + rank) gives each doc item a
//     {query mask, posting offset} entry; lane q tests its bit and reads u.  Query side: a
//     monotone pointer over the staged doc items finds the doc weight of y_j;
//   * root (phase C): the northwest corner over the residuals in vocab order; η = min of the two
//     current residuals, exactly the triples of the warp kernel.
// Pairs that share an M-node (a cell with ≥ 2 ground points, phase B) are listed for the warp
// kernel.  The merge advances in warp-uniform batches of 8 steps: each lane queues the table
// offsets of its (up to 8) triples, then all lanes issue their gathers together, so one L2 latency
// is paid per batch rather than per triple.  Masses are exact u32 (reading R13), distances FP32
// from the a5 table, the sum FP32 per batch and FP64 across batches.
#include <algorithm>

#include "ft_device.cuh"

namespace {

constexpr int QC = 32;     // queries per chunk = lanes
constexpr int XW = 32;     // warps per CTA, one doc each, sharing the chunk structure
constexpr int RB = 8;      // merge steps per gather batch
constexpr int FTX_CM = 8;  // per-lane common-item masks: docs of ≤ 256 items

struct XGeom {
    int nw;                // vocab bitmap words = ceil(N / 32)
    int umax, pmax;        // union / posting capacity
    int sq;                // query items per query slot in the chunk copy (≥ max support)
    size_t off_bits, off_rank, off_ent, off_post, off_qy, off_qu, stride;
};

struct XHdr {
    uint32_t nU, nP, nq, pad;
    uint32_t U[QC], s[QC], ok[QC], nmn[QC];
};

// one CTA per chunk: the union of the chunk's query ids (bitmap + per-word rank), per union id the
// mask of the queries holding it and an offset into u16 postings of their weights (query order),
// and the queries' items transposed [j][lane] (ids u32, weights u16)
__global__ void __launch_bounds__(1024) k_ftx_chunk(const uint8_t* __restrict__ qblock, QueryLayout L, int32_t nq,
                                                    XGeom g, uint8_t* __restrict__ chunks, uint32_t* err) {
    extern __shared__ uint32_t sx[];
    uint32_t* bits = sx;                 // nw
    uint32_t* rank = bits + g.nw;        // nw
    uint32_t* emask = rank + g.nw;       // umax
    __shared__ int tmp[32];
    const int c = blockIdx.x;
    const int q0 = c * QC;
    const int nqc = min(QC, nq - q0);
    uint8_t* out = chunks + (size_t)c * g.stride;
    XHdr* hdr = (XHdr*)out;
    for (int i = threadIdx.x; i < g.nw; i += blockDim.x) bits[i] = 0u;
    for (int i = threadIdx.x; i < g.umax; i += blockDim.x) emask[i] = 0u;
    __syncthreads();
    auto qslot = [&](int ql) { return qblock + (size_t)(q0 + ql) * L.stride; };
    for (int t = threadIdx.x; t < nqc * g.sq; t += blockDim.x) {
        const int ql = t / g.sq, j = t - ql * g.sq;
        const QHeader* qh = (const QHeader*)qslot(ql);
        if (qh->err || j >= (int)qh->s) continue;
        const uint32_t x = ((const uint2*)(qslot(ql) + L.off_items))[j].x & FTI_VOCAB_MASK;
        atomicOr(&bits[x >> 5], 1u << (x & 31));
    }
    __syncthreads();
    int run = 0;
    for (int b0 = 0; b0 < g.nw; b0 += blockDim.x) {
        const int w = b0 + threadIdx.x;
        const int v = w < g.nw ? __popc(bits[w]) : 0;
        int tot;
        const int r = run + fti_block_exclusive_sum(v, tmp, &tot);
        if (w < g.nw) rank[w] = (uint32_t)r;
        run += tot;
    }
    const int nU = run;
    __syncthreads();
    auto uid = [&](uint32_t x) { return rank[x >> 5] + __popc(bits[x >> 5] & ((1u << (x & 31)) - 1u)); };
    for (int t = threadIdx.x; t < nqc * g.sq; t += blockDim.x) {
        const int ql = t / g.sq, j = t - ql * g.sq;
        const QHeader* qh = (const QHeader*)qslot(ql);
        if (qh->err || j >= (int)qh->s) continue;
        const uint32_t x = ((const uint2*)(qslot(ql) + L.off_items))[j].x & FTI_VOCAB_MASK;
        atomicOr(&emask[uid(x)], 1u << ql);
    }
    __syncthreads();
    uint2* gent = (uint2*)(out + g.off_ent);
    int prun = 0;
    for (int b0 = 0; b0 < nU; b0 += blockDim.x) {
        const int i = b0 + threadIdx.x;
        const int v = i < nU ? __popc(emask[i]) : 0;
        int tot;
        const int r = prun + fti_block_exclusive_sum(v, tmp, &tot);
        if (i < nU) gent[i] = make_uint2(emask[i], (uint32_t)r);
        prun += tot;
    }
    __syncthreads();
    uint16_t* gpost = (uint16_t*)(out + g.off_post);
    uint32_t* gqy = (uint32_t*)(out + g.off_qy);
    uint16_t* gqu = (uint16_t*)(out + g.off_qu);
    for (int t = threadIdx.x; t < QC * g.sq; t += blockDim.x) {
        const int ql = t / g.sq, j = t - ql * g.sq;
        uint32_t x = 0xFFFFFFFFu, u = 0;
        if (ql < nqc) {
            const QHeader* qh = (const QHeader*)qslot(ql);
            if (!qh->err && j < (int)qh->s) {
                const uint2 it = ((const uint2*)(qslot(ql) + L.off_items))[j];
                x = it.x & FTI_VOCAB_MASK;
                u = it.y;
                const uint32_t id = uid(x);
                const uint32_t m = gent[id].x;
                gpost[gent[id].y + __popc(m & ((1u << ql) - 1u))] = (uint16_t)u;
            }
        }
        gqy[j * QC + ql] = x;
        gqu[j * QC + ql] = (uint16_t)u;
    }
    uint32_t* gb = (uint32_t*)(out + g.off_bits);
    uint32_t* gr = (uint32_t*)(out + g.off_rank);
    for (int i = threadIdx.x; i < g.nw; i += blockDim.x) { gb[i] = bits[i]; gr[i] = rank[i]; }
    if (threadIdx.x < QC) {
        const int ql = threadIdx.x;
        uint32_t U = 0, s = 0, ok = 0, nmn = 0;
        if (ql < nqc) {
            const QHeader* qh = (const QHeader*)qslot(ql);
            U = qh->U;
            s = qh->s;
            nmn = qh->n_mn;
            ok = (qh->err == 0 && qh->s > 0) ? 1u : 0u;
        }
        hdr->U[ql] = U; hdr->s[ql] = s; hdr->ok[ql] = ok; hdr->nmn[ql] = nmn;
    }
    if (threadIdx.x == 0) {
        hdr->nU = (uint32_t)nU; hdr->nP = (uint32_t)prun; hdr->nq = (uint32_t)nqc;
        if (nU > g.umax || prun > g.pmax) atomicOr(err, FTI_ERR_CAP);
    }
}

struct XArgs {
    const uint32_t* doc_off;
    const uint2* items;
    const uint32_t* Wd;
    const uint32_t* mn_off;
    const uint4* mnodes;
    const uint8_t* qblock;
    QueryLayout L;
    int32_t nq;
    int64_t n_docs, docs_per_cta;
    const uint8_t* chunks;
    XGeom g;
    const float* table;
    int64_t rows_cap;
    int32_t ld;
    double* out;
    int64_t out_ld;
    int Sd;
    uint32_t* fb_list;
    uint32_t* fb_cnt;
    int64_t fb_cap;
    unsigned long long* units;
};

__global__ void __launch_bounds__(XW * 32) k_ftx(XArgs a) {
    extern __shared__ __align__(16) unsigned char smx[];
    __shared__ XHdr sh;
    const XGeom& g = a.g;
    const uint8_t* src = a.chunks + (size_t)blockIdx.y * g.stride;
    if (threadIdx.x == 0) sh = *(const XHdr*)src;
    __syncthreads();
    const int nU = min((int)sh.nU, g.umax), nP = min((int)sh.nP, g.pmax);
    // shared: bits[nw] | rank[nw] | ent[umax] | qy[sq][32] | post[pmax] u16 | qu[sq][32] u16 |
    //         per warp: dx[Sd] u32, dent[Sd] i32, dw[Sd] u16
    uint32_t* bits = (uint32_t*)smx;
    uint32_t* rank = bits + g.nw;
    uint2* ent = (uint2*)(rank + g.nw);
    uint32_t* qy = (uint32_t*)(ent + g.umax);
    uint16_t* post = (uint16_t*)(qy + g.sq * QC);
    uint16_t* qu = post + ((g.pmax + 1) & ~1);
    uint32_t* wbase = (uint32_t*)(qu + g.sq * QC);
    {
        const uint32_t* gb = (const uint32_t*)(src + g.off_bits);
        const uint32_t* gr = (const uint32_t*)(src + g.off_rank);
        for (int i = threadIdx.x; i < g.nw; i += blockDim.x) { bits[i] = gb[i]; rank[i] = gr[i]; }
        const uint2* ge = (const uint2*)(src + g.off_ent);
        for (int i = threadIdx.x; i < nU; i += blockDim.x) ent[i] = ge[i];
        const uint16_t* gp = (const uint16_t*)(src + g.off_post);
        for (int i = threadIdx.x; i < nP; i += blockDim.x) post[i] = gp[i];
        const uint32_t* gy = (const uint32_t*)(src + g.off_qy);
        const uint16_t* gu = (const uint16_t*)(src + g.off_qu);
        for (int i = threadIdx.x; i < g.sq * QC; i += blockDim.x) { qy[i] = gy[i]; qu[i] = gu[i]; }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* dx = wbase + warp * (2 * a.Sd + (a.Sd + 1) / 2 + FTX_CM * 32);
    int* dent = (int*)(dx + a.Sd);
    uint16_t* dw = (uint16_t*)(dent + a.Sd);
    uint32_t* cm = (uint32_t*)(dw + 2 * ((a.Sd + 1) / 2));    // [FTX_CM][32]: lane's common doc items
    const uint32_t lt = (1u << lane) - 1u;
    const int q = blockIdx.y * QC + lane;
    const bool qok = lane < (int)sh.nq && sh.ok[lane];
    const uint32_t U = sh.U[lane];
    const int sq = (int)sh.s[lane];
    const bool qmn = sh.nmn[lane] > 0;
    const float* trow = a.table + (int64_t)(q < a.nq ? q : 0) * a.rows_cap * a.ld;
    const uint32_t ld = (uint32_t)a.ld;
    const uint8_t* slot = a.qblock + (size_t)(q < a.nq ? q : 0) * a.L.stride;
    const uint4* gmh = (const uint4*)(slot + a.L.off_mh);
    const uint32_t mh_mask = ((const QHeader*)slot)->mh_mask;
    unsigned long long ubytes = 0;
    const int64_t d0 = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t d1 = min(a.n_docs, d0 + a.docs_per_cta);
    for (int64_t dp = d0 + warp; dp < d1; dp += XW) {
        const int64_t doc = dp;
        const uint32_t i0 = a.doc_off[doc];
        const int s = (int)(a.doc_off[doc + 1] - i0);
        const uint32_t W = a.Wd[doc];
        __syncwarp();
        // stage the doc: ids, weights, union entries; per lane the bitmask of the doc items its query
        // holds (a 32×32 bit transpose per 32-item chunk via ballots)
        for (int c0 = 0; c0 < s; c0 += 32) {
            const int i = c0 + lane;
            uint32_t em = 0u;
            if (i < s) {
                const uint2 it = a.items[i0 + i];
                const uint32_t x = it.x & FTI_VOCAB_MASK;
                dx[i] = x;
                dw[i] = (uint16_t)it.y;
                const uint32_t bw = bits[x >> 5], bm = 1u << (x & 31);
                const int e = (bw & bm) ? (int)(rank[x >> 5] + __popc(bw & (bm - 1u))) : -1;
                dent[i] = e;
                if (e >= 0) em = ent[e].x;
            }
            uint32_t mine = 0u;
            if (__any_sync(0xffffffffu, em != 0u)) {
#pragma unroll 4
                for (int qq = 0; qq < 32; qq++) {
                    const uint32_t b = __ballot_sync(0xffffffffu, (em >> qq) & 1u);
                    if (lane == qq) mine = b;
                }
            }
            cm[(c0 >> 5) * 32 + lane] = mine;
        }
        __syncwarp();
        // a common M-node hands the pair to the warp kernel
        bool active = qok;
        const uint32_t m0 = a.mn_off[doc], m1 = a.mn_off[doc + 1];
        if (active && qmn && m1 > m0) {
            bool general = false;
            for (uint32_t r = m0; r < m1 && !general; r++) {
                const uint32_t node = a.mnodes[r].x;
                uint32_t h = fti_hash(node) & mh_mask;
                while (true) {
                    const uint32_t kk = gmh[h].x;
                    if (kk == node) { general = true; break; }
                    if (kk == FTI_EMPTY) break;
                    h = (h + 1) & mh_mask;
                }
            }
            if (general) {
                const uint32_t pos = atomicAdd(&a.fb_cnt[q], 1u);
                a.fb_list[(int64_t)q * a.fb_cap + pos] = (uint32_t)dp;
                active = false;
            }
        }
        if (!qok && lane < (int)sh.nq) a.out[(int64_t)q * a.out_ld + dp] = __longlong_as_double(0x7ff8000000000000ll);
        const bool scored = active;
        // ---- per-lane merge, branch-free: (x, ra) / (y, rb) are the current doc / query item and
        // its residual, (xn, ran) / (yn, rbn) the next ones, recomputed every step so all lanes
        // stay converged; c is the next doc item this lane's query holds (its set mask bits) ----
        int c = s;
        uint32_t xc = 0xFFFFFFFFu;          // dx[c] (the id the next query-side self match needs)
        uint32_t cbits = 0u;
        int cchunk = -1;
#define FTX_NEXT_COMMON()                                                              \
    do {                                                                               \
        while (cbits == 0u && ++cchunk < (s + 31) / 32) cbits = cm[cchunk * 32 + lane]; \
        if (cbits) {                                                                   \
            c = cchunk * 32 + __ffs(cbits) - 1;                                        \
            cbits &= cbits - 1u;                                                       \
            xc = dx[c];                                                                \
        } else {                                                                       \
            c = s;                                                                     \
            xc = 0xFFFFFFFFu;                                                          \
        }                                                                              \
    } while (0)
        if (active) FTX_NEXT_COMMON();
        // residual of doc item ii for this lane: w U − min(w U, u W) when the query holds its id
#define FTX_DOC(ii, xo, ro)                                                             \
    do {                                                                                \
        const int ii_ = (ii) < s ? (ii) : s - 1;                                        \
        xo = dx[ii_];                                                                   \
        uint32_t m_ = (uint32_t)dw[ii_] * U;                                            \
        if ((cm[(ii_ >> 5) * 32 + lane] >> (ii_ & 31)) & 1u) {                          \
            const uint2 en_ = ent[dent[ii_]];                                           \
            const uint32_t qm_ = (uint32_t)post[en_.y + __popc(en_.x & lt)] * W;        \
            m_ -= (qm_ < m_ ? qm_ : m_);                                                \
        }                                                                               \
        ro = m_;                                                                        \
    } while (0)
        // residual of query item jj: u W − min(u W, w U) when it is the doc's next common item
#define FTX_Q(jj, yo, ro, hit)                                                          \
    do {                                                                                \
        const int jj_ = (jj) < sq ? (jj) : sq - 1;                                      \
        yo = qy[jj_ * QC + lane];                                                       \
        uint32_t m_ = (uint32_t)qu[jj_ * QC + lane] * W;                                \
        hit = xc == yo;                                                                 \
        if (hit) {                                                                      \
            const uint32_t dm_ = (uint32_t)dw[c] * U;                                   \
            m_ -= (dm_ < m_ ? dm_ : m_);                                                \
        }                                                                               \
        ro = m_;                                                                        \
    } while (0)
        int i = 0, j = 0;
        uint32_t x = 0, ra = 0, y = 0, rb = 0, xn = 0, ran = 0, yn = 0, rbn = 0;
        bool hit = false, hitn = false;
        if (active) {
            FTX_DOC(0, x, ra);
            FTX_Q(0, y, rb, hit);
            if (hit) FTX_NEXT_COMMON();
            FTX_DOC(1, xn, ran);
            FTX_Q(1, yn, rbn, hitn);
        }
        double acc = 0.0;
        while (__any_sync(0xffffffffu, active)) {
            uint32_t off[RB];
            float ef[RB];
#pragma unroll
            for (int u = 0; u < RB; u++) {
                const uint32_t eta = active ? (ra < rb ? ra : rb) : 0u;
                off[u] = x * ld + (uint32_t)j;
                ef[u] = (eta && x != y) ? (float)eta : 0.f;
                ra -= eta;
                rb -= eta;
                const bool ad = active && ra == 0u, aq = active && rb == 0u;
                i += ad;
                j += aq;
                if (ad) { x = xn; ra = ran; }
                if (aq) {
                    y = yn; rb = rbn;
                    if (hitn) FTX_NEXT_COMMON();
                }
                active = active && i < s && j < sq;
                if (ad) FTX_DOC(i + 1, xn, ran);
                if (aq) FTX_Q(j + 1, yn, rbn, hitn);
            }
            float dv[RB];
#pragma unroll
            for (int u = 0; u < RB; u++) dv[u] = ef[u] != 0.f ? trow[off[u]] : 0.f;
            float part = 0.f;
#pragma unroll
            for (int u = 0; u < RB; u++) part = fmaf(ef[u], dv[u], part);
            acc += (double)part;
        }
#undef FTX_NEXT_COMMON
#undef FTX_DOC
#undef FTX_Q
        if (scored) {
            a.out[(int64_t)q * a.out_ld + dp] = acc / (double)((unsigned long long)W * U);
            ubytes += 8ull * (unsigned long long)s + 16ull;
        }
    }
    if (a.units && ubytes) atomicAdd(a.units, ubytes);
}

}  // namespace

cudaError_t fti_launch_ftx(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq, int64_t n_docs,
                           const FtTable& tab, double* d_out, int64_t out_ld, uint32_t** fb_list, uint32_t** fb_cnt,
                           cudaStream_t st) {
    const ft_index* ix = ds->ix;
    const int nchunks = (nq + QC - 1) / QC;
    XGeom g{};
    g.nw = (int)((ix->N + 31) / 32);
    g.sq = std::max(1, L.smax);
    g.umax = (int)std::min<int64_t>(ix->N, (int64_t)QC * g.sq);
    g.pmax = QC * g.sq;
    auto up = [](size_t x) { return (x + 15) / 16 * 16; };
    size_t o = up(sizeof(XHdr));
    g.off_bits = o; o = up(o + 4ull * g.nw);
    g.off_rank = o; o = up(o + 4ull * g.nw);
    g.off_ent = o;  o = up(o + 8ull * g.umax);
    g.off_post = o; o = up(o + 2ull * g.pmax);
    g.off_qy = o;   o = up(o + 4ull * g.sq * QC);
    g.off_qu = o;   o = up(o + 2ull * g.sq * QC);
    g.stride = o;
    const size_t smem_c = 4ull * (2 * g.nw + g.umax);
    const size_t per_warp = 4ull * (2 * ds->max_s + 2 * ((ds->max_s + 1) / 2) + FTX_CM * 32);
    const size_t smem = 8ull * g.nw + 8ull * g.umax + 4ull * g.sq * QC + 2ull * ((g.pmax + 1) & ~1) +
                        2ull * g.sq * QC + (size_t)XW * per_warp + 16;
    if (smem_c > 200 * 1024 || smem > 220 * 1024 || ds->max_s > 32 * FTX_CM)
        return cudaErrorNotSupported;   // caller: warp kernel only
    cudaError_t e;
    if ((e = ds->s_ftxchunk.reserve(g.stride * (size_t)nchunks)) != cudaSuccess) return e;
    if ((e = ds->s_fblist.reserve((size_t)nq * n_docs * 4)) != cudaSuccess) return e;
    if ((e = ds->s_fbcnt.reserve((size_t)nq * 4)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ds->s_fbcnt.p, 0, (size_t)nq * 4, st)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_ftx_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c)) != cudaSuccess)
        return e;
    k_ftx_chunk<<<nchunks, 1024, smem_c, st>>>(d_qblock, L, nq, g, ds->s_ftxchunk.as<uint8_t>(), ds->err_dev);
    XArgs a{};
    a.doc_off = ds->doc_off; a.items = ds->items; a.Wd = ds->W;
    a.mn_off = ds->mn_off; a.mnodes = ds->mnodes;
    a.qblock = d_qblock; a.L = L; a.nq = nq; a.n_docs = n_docs;
    a.chunks = ds->s_ftxchunk.as<uint8_t>(); a.g = g;
    a.table = tab.table; a.rows_cap = tab.rows_cap; a.ld = tab.ld;
    a.out = d_out; a.out_ld = out_ld;
    a.Sd = ds->max_s;
    a.fb_list = ds->s_fblist.as<uint32_t>(); a.fb_cnt = ds->s_fbcnt.as<uint32_t>(); a.fb_cap = n_docs;
    a.units = ds->units_ptr(FTI_ST_FT);
    if ((e = cudaFuncSetAttribute(k_ftx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((n_docs + XW - 1) / XW, (296 + nchunks - 1) / nchunks));
    a.docs_per_cta = (n_docs + bx - 1) / bx;
    const int64_t gx = (n_docs + a.docs_per_cta - 1) / a.docs_per_cta;
    k_ftx<<<dim3((unsigned)gx, (unsigned)nchunks), XW * 32, smem, st>>>(a);
    fti_count_launches(2);
    *fb_list = ds->s_fblist.as<uint32_t>();
    *fb_cnt = ds->s_fbcnt.as<uint32_t>();
    return cudaGetLastError();
}
