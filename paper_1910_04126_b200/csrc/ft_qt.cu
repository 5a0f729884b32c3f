// ft_qt.cu — a3: Quadtree estimate kernel (§2 "Wasserstein-1 on Quadtree").
//
// For a (query ν, doc μ) pair with cross-scaled masses (reading R13):
//   num = Σ_{v≠root} ω(v) |U m_μ(v) − W m_ν(v)|
//       = U·A + W·B − 2 Σ_{v ∈ nodes(μ) ∩ nodes(ν)} ω(v) min(U m_μ(v), W m_ν(v))
//   QT  = (num · 2^{ℓ_root − D*}) / (W·U)
// so the kernel streams each doc's node-sorted record (the sparse ℓ1 embedding,
// PAPER.md:131-134) once per chunk of 32 queries and only the common nodes contribute.  The
// numerator is an exact u64; the value takes two correctly rounded FP64 operations, so it is
// bit-identical to the oracle.
//
// Query-chunk structure (k_qt_chunk, one CTA per chunk of ≤ 32 queries): one open-addressing hash
// over the union of the chunk's query nodes; each distinct node carries a 32-bit mask of the
// chunk queries that contain it and an offset into a posting array of packed
// (m_ν(v) | depth << 16 | query << 24) words ordered by query.
//
// Doc scan (k_qt, grid = doc tiles × chunks): the chunk structure is staged in shared memory;
// one warp per doc, lane-strided 8-byte records (coalesced), one probe per record; for every hit
// the warp visits the node once with LANE = QUERY: lane q tests bit q of the mask, reads its
// posting and accumulates ω·min(U m_μ, W m_ν) in a u64 register — no atomics, no per-query
// probing.  Lane q then finalises the value of (q, doc).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ft_device.cuh"

namespace {

constexpr int QT_WARPS = 32;   // 1024 threads share one staged chunk structure
constexpr int QT_QC = 32;   // queries per chunk (= lanes)

constexpr int QT_UCAP_S = 4096;   // distinct nodes staged in shared memory (else read from L2)
constexpr int QT_PCAP_S = 8192;   // postings staged in shared memory (else read from L2)

struct ChunkGeom {
    int cap;        // hash capacity (pow2 > 1.25 umax)
    int umax;       // max distinct nodes per chunk
    int pmax;       // max postings per chunk
    int ucap_s, pcap_s;
    size_t off_keys, off_idx, off_mask, off_off, off_post, stride;
};

struct ChunkHdr {
    uint32_t nU, nP, nq, pad;
    uint32_t U[QT_QC];
    uint32_t ok[QT_QC];
    unsigned long long B[QT_QC];
};

// geometry of a chunk that holds up to qc (≤ QT_QC) queries
ChunkGeom chunk_geom(const ft_dataset* ds, const QueryLayout& L, int qc) {
    ChunkGeom g;
    const int64_t per_q = std::min<int64_t>((int64_t)L.smax * std::max(1, ds->ix->d_star), ds->ix->M);
    g.umax = (int)std::min<int64_t>(std::min<int64_t>((int64_t)qc * per_q, ds->ix->M), 65535);
    g.pmax = (int)((int64_t)qc * per_q);
    g.cap = fti_pow2_at_least(std::max(64, g.umax + g.umax / 4 + 1));
    g.ucap_s = (std::min(g.umax, QT_UCAP_S) + 7) & ~7;   // multiples of 8 keep the u16 idx array 16-B aligned
    g.pcap_s = (std::min(g.pmax, QT_PCAP_S) + 7) & ~7;
    auto up = [](size_t x) { return (x + 15) / 16 * 16; };
    size_t o = up(sizeof(ChunkHdr));
    g.off_keys = o; o = up(o + 4ull * g.cap);
    g.off_idx = o;  o = up(o + 2ull * g.cap);
    g.off_mask = o; o = up(o + 8ull * g.umax);   // {query mask, posting offset} per distinct node
    g.off_off = 0;
    g.off_post = o; o = up(o + 4ull * g.pmax);
    g.stride = o;
    return g;
}

// the chunk's node hash (keys + dense indices, 6 bytes per slot) is always staged in shared memory,
// by the builder next to the masks/offsets and by the scan next to the staged postings
constexpr int QT_CAP_MAX = 16384;
bool chunk_fits(const ChunkGeom& g) {
    return g.cap <= QT_CAP_MAX && 6ull * g.cap + 8ull * g.umax <= 220 * 1024;
}

// queries per chunk for this batch: QT_QC unless the worst-case node union of 32 large-support
// queries on a deep tree would not fit the shared-memory hash; then the largest power of two that
// does (the batch is scored in sub-batches of that many queries, one partly filled chunk each).
// Within the documented limits (support × depth ≤ 8192) one query always fits.
int qt_fit_queries(const ft_dataset* ds, const QueryLayout& L) {
    for (int qc = QT_QC; qc >= 1; qc >>= 1)
        if (chunk_fits(chunk_geom(ds, L, qc))) return qc;
    return 0;
}

__device__ __forceinline__ int probe_slot(const uint32_t* keys, uint32_t mask, uint32_t node) {
    uint32_t h = fti_hash(node) & mask;
    while (true) {
        uint32_t k = keys[h];
        if (k == node) return (int)h;
        if (k == FTI_EMPTY) return -1;
        h = (h + 1) & mask;
    }
}

// one CTA per chunk: union hash of the chunk's query nodes with query masks and postings
__global__ void __launch_bounds__(1024) k_qt_chunk(const uint8_t* __restrict__ qblock, QueryLayout L, int32_t nq,
                                                   ChunkGeom g, uint8_t* __restrict__ chunks, uint32_t* err) {
    extern __shared__ uint32_t smq[];
    uint32_t* keys = smq;                         // cap
    uint32_t* emask = keys + g.cap;               // umax
    uint32_t* eoff = emask + g.umax;              // umax
    uint16_t* idxs = (uint16_t*)(eoff + g.umax);  // cap
    __shared__ int tmp[32];
    __shared__ int s_overflow;
    const int c = blockIdx.x;
    const int q0 = c * QT_QC;
    const int nqc = min(QT_QC, nq - q0);
    uint8_t* out = chunks + (size_t)c * g.stride;
    ChunkHdr* hdr = (ChunkHdr*)out;
    const uint32_t cmask = (uint32_t)g.cap - 1;
    for (int i = threadIdx.x; i < g.cap; i += blockDim.x) keys[i] = FTI_EMPTY;
    if (threadIdx.x == 0) s_overflow = 0;
    __syncthreads();
    // flattened (query, slot) iteration over the chunk's node hashes
    const int slots = L.nh_cap;
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        uint32_t h = fti_hash(e.x) & cmask;
        while (true) {
            uint32_t prev = atomicCAS(&keys[h], FTI_EMPTY, e.x);
            if (prev == FTI_EMPTY || prev == e.x) break;
            h = (h + 1) & cmask;
        }
    }
    __syncthreads();
    // dense ids of the distinct nodes (slot order)
    int run = 0;
    for (int b0 = 0; b0 < g.cap; b0 += blockDim.x) {
        int i = b0 + threadIdx.x;
        int f = (i < g.cap) ? (keys[i] != FTI_EMPTY) : 0;
        int tot;
        int r = run + fti_block_exclusive_sum(f, tmp, &tot);
        if (f) {
            if (r < g.umax) { idxs[i] = (uint16_t)r; emask[r] = 0; }
            else s_overflow = 1;
        }
        run += tot;
    }
    const int nU = min(run, g.umax);
    __syncthreads();
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        int h = probe_slot(keys, cmask, e.x);
        atomicOr(&emask[idxs[h]], 1u << ql);
    }
    __syncthreads();
    int prun = 0;
    for (int b0 = 0; b0 < nU; b0 += blockDim.x) {
        int i = b0 + threadIdx.x;
        int v = (i < nU) ? __popc(emask[i]) : 0;
        int tot;
        int r = prun + fti_block_exclusive_sum(v, tmp, &tot);
        if (i < nU) eoff[i] = (uint32_t)r;
        prun += tot;
    }
    const int nP = prun;
    __syncthreads();
    uint32_t* post = (uint32_t*)(out + g.off_post);
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        const uint32_t dep = (slot + L.off_nd)[s];
        const int id = idxs[probe_slot(keys, cmask, e.x)];
        const uint32_t mk = emask[id];
        const uint32_t pos = eoff[id] + __popc(mk & ((1u << ql) - 1u));
        if (pos < (uint32_t)g.pmax) post[pos] = (e.y & 0xFFFFu) | (dep << 16) | ((uint32_t)ql << 24);
    }
    // publish
    uint32_t* gk = (uint32_t*)(out + g.off_keys);
    uint16_t* gi = (uint16_t*)(out + g.off_idx);
    uint2* ge = (uint2*)(out + g.off_mask);
    for (int i = threadIdx.x; i < g.cap; i += blockDim.x) { gk[i] = keys[i]; gi[i] = idxs[i]; }
    for (int i = threadIdx.x; i < nU; i += blockDim.x) ge[i] = make_uint2(emask[i], eoff[i]);
    if (threadIdx.x < QT_QC) {
        const int ql = threadIdx.x;
        uint32_t U = 0, ok = 0;
        unsigned long long B = 0;
        if (ql < nqc) {
            const QHeader* qh = (const QHeader*)(qblock + (size_t)(q0 + ql) * L.stride);
            U = qh->U;
            B = qh->B;
            ok = (qh->err == 0 && qh->s > 0) ? 1u : 0u;
        }
        hdr->U[ql] = U;
        hdr->ok[ql] = ok && !s_overflow;
        hdr->B[ql] = B;
    }
    if (threadIdx.x == 0) {
        hdr->nU = nU; hdr->nP = nP; hdr->nq = nqc;
        if (s_overflow || nP > g.pmax) atomicOr(err, FTI_ERR_CAP);
    }
}

// Dense chunk structure, one CTA per chunk: the union of the chunk's query nodes as a bitmap over
// all node ids with per-word ranks, and a dense [union][32 lanes] u16 mass array.  Chunks whose
// union exceeds the capacity keep flag 0 and are scanned with the hash structure.
struct DenseGeom {
    int mw;          // bitmap words = ceil(M / 32)
    int cap;         // max union size (0: dense path disabled)
    size_t stride;   // bytes per chunk: header | bits[mw] | rank[mw] | post[cap][32]
    // chunk PAIRS (64 queries, lane l = queries l and 32 + l of the pair): the union of both
    // chunks' nodes, and per union node a u16 per lane packing the two queries' masses as bytes
    // (only when every mass < 256, e.g. unit weights); one record pass then serves 64 queries
    int cap2;        // max union size of a pair (0: pair path disabled)
    size_t stride2;  // bytes per pair: header | bits[mw] | rank[mw] | post2[cap2][32] u16
};

struct DenseHdr {
    uint32_t flag, nU, pad0, pad1;
};

__global__ void __launch_bounds__(1024) k_qt_dense(const uint8_t* __restrict__ qblock, QueryLayout L, int32_t nq,
                                                   DenseGeom dg, uint8_t* __restrict__ dchunks) {
    extern __shared__ uint32_t sd[];
    uint32_t* bits = sd;              // mw
    uint32_t* rank = sd + dg.mw;      // mw
    __shared__ int tmp[32];
    const int c = blockIdx.x;
    const int q0 = c * QT_QC;
    const int nqc = min(QT_QC, nq - q0);
    uint8_t* out = dchunks + (size_t)c * dg.stride;
    DenseHdr* hdr = (DenseHdr*)out;
    for (int i = threadIdx.x; i < dg.mw; i += blockDim.x) bits[i] = 0u;
    __syncthreads();
    const int slots = L.nh_cap;
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        atomicOr(&bits[e.x >> 5], 1u << (e.x & 31u));
    }
    __syncthreads();
    int run = 0;
    for (int b0 = 0; b0 < dg.mw; b0 += blockDim.x) {
        const int w = b0 + threadIdx.x;
        const int v = w < dg.mw ? __popc(bits[w]) : 0;
        int tot;
        const int r = run + fti_block_exclusive_sum(v, tmp, &tot);
        if (w < dg.mw) rank[w] = (uint32_t)r;
        run += tot;
    }
    __syncthreads();
    const int nU = run;
    if (nU > dg.cap) {
        if (threadIdx.x == 0) { hdr->flag = 0u; hdr->nU = (uint32_t)nU; }
        return;
    }
    uint32_t* gbits = (uint32_t*)(out + sizeof(DenseHdr));
    uint32_t* grank = gbits + dg.mw;
    uint16_t* gpost = (uint16_t*)(grank + dg.mw);
    for (int i = threadIdx.x; i < dg.mw; i += blockDim.x) { gbits[i] = bits[i]; grank[i] = rank[i]; }
    for (int i = threadIdx.x; i < nU * QT_QC / 2; i += blockDim.x) ((uint32_t*)gpost)[i] = 0u;
    __syncthreads();
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        const uint32_t bw = bits[e.x >> 5], bpos = e.x & 31u;
        const uint32_t id = rank[e.x >> 5] + __popc(bw & ((1u << bpos) - 1u));
        gpost[id * QT_QC + ql] = (uint16_t)(e.y & 0xFFFFu);
    }
    if (threadIdx.x == 0) { hdr->flag = 1u; hdr->nU = (uint32_t)nU; }
}

// Dense structure of a chunk PAIR (queries 64c .. 64c + 63): flag 0 when the union exceeds cap2 or
// a query node mass does not fit a byte (those pairs are scanned chunk by chunk).
__global__ void __launch_bounds__(1024) k_qt_dense2(const uint8_t* __restrict__ qblock, QueryLayout L, int32_t nq,
                                                    DenseGeom dg, uint8_t* __restrict__ dchunks) {
    extern __shared__ uint32_t sd[];
    uint32_t* bits = sd;              // mw
    uint32_t* rank = sd + dg.mw;      // mw
    __shared__ int tmp[32];
    __shared__ int s_big;
    const int c = blockIdx.x;
    const int q0 = c * 2 * QT_QC;
    const int nqc = min(2 * QT_QC, nq - q0);
    uint8_t* out = dchunks + (size_t)c * dg.stride2;
    DenseHdr* hdr = (DenseHdr*)out;
    for (int i = threadIdx.x; i < dg.mw; i += blockDim.x) bits[i] = 0u;
    if (threadIdx.x == 0) s_big = 0;
    __syncthreads();
    const int slots = L.nh_cap;
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        atomicOr(&bits[e.x >> 5], 1u << (e.x & 31u));
        if ((e.y & 0xFFFFu) > 255u) s_big = 1;
    }
    __syncthreads();
    int run = 0;
    for (int b0 = 0; b0 < dg.mw; b0 += blockDim.x) {
        const int w = b0 + threadIdx.x;
        const int v = w < dg.mw ? __popc(bits[w]) : 0;
        int tot;
        const int r = run + fti_block_exclusive_sum(v, tmp, &tot);
        if (w < dg.mw) rank[w] = (uint32_t)r;
        run += tot;
    }
    __syncthreads();
    const int nU = run;
    if (nU > dg.cap2 || s_big) {
        if (threadIdx.x == 0) { hdr->flag = 0u; hdr->nU = (uint32_t)nU; }
        return;
    }
    uint32_t* gbits = (uint32_t*)(out + sizeof(DenseHdr));
    uint32_t* grank = gbits + dg.mw;
    uint32_t* gpost = grank + dg.mw;                       // [nU][32] u16, as u32 pairs of lanes
    for (int i = threadIdx.x; i < dg.mw; i += blockDim.x) { gbits[i] = bits[i]; grank[i] = rank[i]; }
    for (int i = threadIdx.x; i < nU * QT_QC / 2; i += blockDim.x) gpost[i] = 0u;
    __syncthreads();
    for (int t = threadIdx.x; t < nqc * slots; t += blockDim.x) {
        const int ql = t / slots, s = t - ql * slots;
        const uint8_t* slot = qblock + (size_t)(q0 + ql) * L.stride;
        const QHeader* qh = (const QHeader*)slot;
        if (qh->err || s > (int)qh->nh_mask) continue;
        const uint2 e = ((const uint2*)(slot + L.off_nh))[s];
        if (e.x == FTI_EMPTY) continue;
        const uint32_t bw = bits[e.x >> 5], bpos = e.x & 31u;
        const uint32_t id = rank[e.x >> 5] + __popc(bw & ((1u << bpos) - 1u));
        const uint32_t ln = (uint32_t)ql & 31u, hi = (uint32_t)ql >> 5;   // lane, which chunk of the pair
        const uint32_t v = (e.y & 0xFFu) << (8u * hi + 16u * (ln & 1u));
        atomicOr(&gpost[(id * QT_QC + ln) >> 1], v);
    }
    if (threadIdx.x == 0) { hdr->flag = 1u; hdr->nU = (uint32_t)nU; }
}

struct QtArgs {
    const uint32_t* qt_off;
    const uint2* qt;
    const uint32_t* W;
    const unsigned long long* A;
    const uint8_t* chunks;
    ChunkGeom g;
    const uint8_t* dchunks;
    DenseGeom dg;
    int32_t nq;
    const int64_t* docs;
    int64_t n_docs;
    int64_t n;
    int64_t docs_per_cta;
    double* out;
    int64_t out_ld;
    int d_star, l_root;
    double pow2;                // 2^{ℓ_root − D*} when it is a normal double (0: use scalbn)
    float pow2f;                // the same as a normal float (0: the threshold screen is off)
    int wide;                   // D* > 31: the U·A and W·B products can overflow 64 bits
    uint32_t* err;
    // threshold mode (the fused prefilter): instead of writing out, append (value, doc) to query q's
    // candidate list when value ≤ thr[q·thr_ld]; ccnt counts every passing doc (also past ccap)
    const double* thr;
    int64_t thr_ld;
    uint32_t* ccnt;
    double* cval;
    int64_t* cid;
    int64_t ccap;
    // fallback mode: only the chunks holding a flagged query run, and only flagged rows are written
    const uint32_t* qflag;
    // pair mode: each CTA row (blockIdx.y) covers chunks 2y and 2y + 1
    int pair;
    int nchunks;
    const uint8_t* dchunks2;
};

// lane q: QT(q, doc) = (U A + W B_q − 2 acc) · 2^{ℓ_root − D*} / (W U), exact u64 numerator, two
// correctly rounded FP64 operations (NaN for an invalid query or an overflowing numerator)
// Threshold mode: thr_l is the lane's threshold, thr_hi an FP32 bound above it — a value whose FP32
// estimate exceeds thr_hi is certainly above thr_l (the estimate is within 2^-21 relative of the
// exact quotient), so most docs skip the FP64 division; the rest take the exact path.
struct QtThr {
    double t;
    float hi;
    float cu;   // 2^{ℓ_root − D*} / U of the lane's query
};
__device__ __forceinline__ QtThr qt_thr(const QtArgs& a, int nqc, int cy, uint32_t U) {
    const int lane = threadIdx.x & 31;
    QtThr r{0.0, 0.f, 0.f};
    if (a.thr && lane < nqc) {
        r.t = a.thr[(int64_t)(cy * QT_QC + lane) * a.thr_ld];
        r.cu = U ? __fdiv_rn(a.pow2f, (float)U) : 0.f;
        r.hi = a.pow2f != 0.f ? __fmul_ru(__double2float_ru(r.t), 1.0f + 0x1p-18f) : __int_as_float(0x7f800000);
        if (r.t != r.t) r.hi = -1.f;   // NaN threshold: nothing passes (and the exact path agrees)
    }
    return r;
}

__device__ __forceinline__ void qt_store(const QtArgs& a, const ChunkHdr& sh, int nqc, int cy, int64_t dp,
                                         int64_t doc, unsigned long long acc, uint32_t W32, unsigned long long A,
                                         const QtThr& th) {
    const int lane = threadIdx.x & 31;
    if (lane >= nqc) return;
    const int q = cy * QT_QC + lane;
    const unsigned long long Uq = sh.U[lane], Bq = sh.B[lane], W = W32;
    double val;
    bool bad = !sh.ok[lane];
    const unsigned long long ua = Uq * A, wb = W * Bq;
    const unsigned long long tot = ua + wb;
    // A, B < 2^16·2^{D*} (masses ≤ 65535 per level): with D* ≤ 31 neither product nor the sum
    // can overflow
    if (a.wide) bad |= __umul64hi(Uq, A) != 0ull || __umul64hi(W, Bq) != 0ull || tot < ua;
    const unsigned long long num = tot - (acc << 1);
    if (!bad && num >= (1ull << 53)) {
        bad = true;
        atomicOr(a.err, FTI_ERR_OVERFLOW);
    }
    if (a.thr && !bad) {
        // FP32 screen: (float)num, 2^k / U, the approximate reciprocal of W and two products each
        // round by ≤ 2 ulp (≤ 2^-20 relative in all), inside the 2^-18 margin of th.hi
        float rw;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rw) : "f"((float)W32));
        const float est = __fmul_rn(__fmul_rn(__ull2float_rn(num), th.cu), rw);
        if (est > th.hi) return;
    }
    if (bad) {
        val = __longlong_as_double(0x7ff8000000000000ll);
    } else {
        // exact: num < 2^53 and a power-of-two factor
        const double scaled = a.pow2 != 0.0 ? (double)num * a.pow2 : scalbn((double)num, a.l_root - a.d_star);
        val = __ddiv_rn(scaled, (double)(Uq * W));
    }
    if (a.thr) {
        if (!bad && val <= th.t) {
            const uint32_t pos = atomicAdd(&a.ccnt[q], 1u);
            if ((int64_t)pos < a.ccap) {
                a.cval[(int64_t)q * a.ccap + pos] = val;
                a.cid[(int64_t)q * a.ccap + pos] = doc;
            }
        }
        return;
    }
    if (a.qflag && !a.qflag[q]) return;
    a.out[(int64_t)q * a.out_ld + dp] = val;
}

// Dense chunk structure (when the chunk's node union is small and the tree's node ids fit a
// shared-memory bitmap): membership of a doc node is one bit test, its union index a rank
// (per-word prefix + popc), and the chunk's masses are a dense [union][32 lanes] u16 array — a
// query without the node reads 0 — so every hit costs one conflict-free LDS per lane, no mask
// test, no posting search.  The node's depth rides in the doc record (mass | depth << 16).
template <bool WIDE>
__device__ __forceinline__ void qt_scan_dense(const QtArgs& a, const uint32_t* __restrict__ bits,
                                              const uint32_t* __restrict__ rank, const uint16_t* __restrict__ post,
                                              uint4* __restrict__ hq, const ChunkHdr& sh, int nqc, int cy) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const QtThr th = qt_thr(a, nqc, cy, sh.U[threadIdx.x & 31]);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t U32 = sh.U[lane];
    const int64_t d0 = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t d1 = min(a.n_docs, d0 + a.docs_per_cta);
    for (int64_t dp = d0 + warp; dp < d1; dp += QT_WARPS) {
        const int64_t doc = a.docs ? a.docs[dp] : dp;
        if (doc < 0 || doc >= a.n) {
            if (lane < nqc && !a.thr)
                a.out[(int64_t)(cy * QT_QC + lane) * a.out_ld + dp] = __longlong_as_double(0x7ff8000000000000ll);
            if (lane == 0) atomicOr(a.err, FTI_ERR_RANGE);
            continue;
        }
        const uint32_t r0 = a.qt_off[doc], r1 = a.qt_off[doc + 1];
        const uint32_t W32 = a.W[doc];
        const unsigned long long A = a.A[doc];
        unsigned long long acc = 0;
        auto term = [&](uint32_t mnu, uint32_t mmu, uint32_t f_) {
            // U·m_μ and W·m_ν are < 2^32 (W, U ≤ 65535): 32-bit products, 64-bit accumulation.
            // f_ = ω(v) = 2^{D* − depth}: one wide multiply-add when D* ≤ 31, else a shift
            const uint32_t um = U32 * mmu;
            const uint32_t wm = W32 * mnu;
            if (WIDE)
                acc += (unsigned long long)(um < wm ? um : wm) << f_;
            else
                acc += (unsigned long long)(um < wm ? um : wm) * f_;
        };
        for (uint32_t rb = r0; rb < r1; rb += 32) {
            const uint32_t r = rb + lane;
            int id = -1;
            uint32_t y = 0;
            if (r < r1) {
                const uint2 rec = a.qt[r];
                y = rec.y;
                const uint32_t bw = bits[rec.x >> 5], bpos = rec.x & 31u;
                if ((bw >> bpos) & 1u) id = (int)(rank[rec.x >> 5] + __popc(bw & ((1u << bpos) - 1u)));
            }
            // compact the batch's hits into the warp's queue, then visit them two at a time with
            // broadcast loads (every lane reads the same {posting offset, m_μ, D* − depth})
            const unsigned hm = __ballot_sync(0xffffffffu, id >= 0);
            const int nh = __popc(hm);
            // the compacting lane decodes the record once: every lane then reads a ready entry
            if (id >= 0)
                hq[__popc(hm & lt)] = make_uint4((uint32_t)id * QT_QC, y & 0xFFFFu,
                                                 WIDE ? (uint32_t)(a.d_star - (int)(y >> 16))
                                                      : 1u << (a.d_star - (int)(y >> 16)),
                                                 0u);
            if (nh & 1) {
                if (lane == 0) hq[nh] = make_uint4(0u, 0u, 0u, 0u);      // pad: mass 0 contributes 0
            }
            __syncwarp();
            for (int h = 0; h < nh; h += 2) {
                const uint4 e1 = hq[h], e2 = hq[h + 1];
                const uint32_t p1 = post[e1.x + lane];
                const uint32_t p2 = post[e2.x + lane];
                term(p1, e1.y, e1.z);
                term(p2, e2.y, e2.z);
            }
            __syncwarp();
        }
        qt_store(a, sh, nqc, cy, dp, doc, acc, W32, A, th);
    }
}

// Pair scan (dense pair structure): lane l scores queries l of chunk cy and l of chunk cy + 1; each
// hit reads one u16 per lane holding both queries' masses, so a record pass, its membership tests
// and the hit compaction serve 64 queries.
template <bool WIDE>
__device__ __forceinline__ void qt_scan_dense2(const QtArgs& a, const uint32_t* __restrict__ bits,
                                               const uint32_t* __restrict__ rank, const uint16_t* __restrict__ post,
                                               uint4* __restrict__ hq, const ChunkHdr& sa, const ChunkHdr& sb,
                                               int cy) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int na = (int)sa.nq, nb = (int)sb.nq;
    const QtThr tha = qt_thr(a, na, cy, sa.U[lane]), thb = qt_thr(a, nb, cy + 1, sb.U[lane]);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t Ua = sa.U[lane], Ub = sb.U[lane];
    const int64_t d0 = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t d1 = min(a.n_docs, d0 + a.docs_per_cta);
    for (int64_t dp = d0 + warp; dp < d1; dp += QT_WARPS) {
        const int64_t doc = a.docs ? a.docs[dp] : dp;
        if (doc < 0 || doc >= a.n) {
            if (!a.thr) {
                if (lane < na) a.out[(int64_t)(cy * QT_QC + lane) * a.out_ld + dp] = __longlong_as_double(0x7ff8000000000000ll);
                if (lane < nb)
                    a.out[(int64_t)((cy + 1) * QT_QC + lane) * a.out_ld + dp] = __longlong_as_double(0x7ff8000000000000ll);
            }
            if (lane == 0) atomicOr(a.err, FTI_ERR_RANGE);
            continue;
        }
        const uint32_t r0 = a.qt_off[doc], r1 = a.qt_off[doc + 1];
        const uint32_t W32 = a.W[doc];
        const unsigned long long A = a.A[doc];
        unsigned long long acca = 0, accb = 0;
        auto term = [&](uint32_t p, uint32_t mmu, uint32_t f_) {
            // masses < 256 here: U·m_μ and W·m_ν < 2^32, 64-bit accumulation as in the 32-query scan
            const uint32_t wa = W32 * (p & 0xFFu), wb = W32 * (p >> 8);
            const uint32_t ua = Ua * mmu, ub = Ub * mmu;
            if (WIDE) {
                acca += (unsigned long long)(ua < wa ? ua : wa) << f_;
                accb += (unsigned long long)(ub < wb ? ub : wb) << f_;
            } else {
                acca += (unsigned long long)(ua < wa ? ua : wa) * f_;
                accb += (unsigned long long)(ub < wb ? ub : wb) * f_;
            }
        };
        for (uint32_t rb = r0; rb < r1; rb += 32) {
            const uint32_t r = rb + lane;
            int id = -1;
            uint32_t y = 0;
            if (r < r1) {
                const uint2 rec = a.qt[r];
                y = rec.y;
                const uint32_t bw = bits[rec.x >> 5], bpos = rec.x & 31u;
                if ((bw >> bpos) & 1u) id = (int)(rank[rec.x >> 5] + __popc(bw & ((1u << bpos) - 1u)));
            }
            const unsigned hm = __ballot_sync(0xffffffffu, id >= 0);
            const int nh = __popc(hm);
            if (id >= 0)
                hq[__popc(hm & lt)] = make_uint4((uint32_t)id * QT_QC, y & 0xFFFFu,
                                                 WIDE ? (uint32_t)(a.d_star - (int)(y >> 16))
                                                      : 1u << (a.d_star - (int)(y >> 16)),
                                                 0u);
            if (nh & 1) {
                if (lane == 0) hq[nh] = make_uint4(0u, 0u, 0u, 0u);      // pad: mass 0 contributes 0
            }
            __syncwarp();
            for (int h = 0; h < nh; h += 2) {
                const uint4 e1 = hq[h], e2 = hq[h + 1];
                const uint32_t p1 = post[e1.x + lane];
                const uint32_t p2 = post[e2.x + lane];
                term(p1, e1.y, e1.z);
                term(p2, e2.y, e2.z);
            }
            __syncwarp();
        }
        qt_store(a, sa, na, cy, dp, doc, acca, W32, A, tha);
        qt_store(a, sb, nb, cy + 1, dp, doc, accb, W32, A, thb);
    }
}

// the doc scan of one CTA (hash structure); SMEM: the masks/offsets and postings are in shared memory (the common
// case), so every lookup is an LDS rather than a generic load
template <bool SMEM>
__device__ __forceinline__ void qt_scan(const QtArgs& a, const uint32_t* __restrict__ keys,
                                        const uint2* __restrict__ ent, const uint32_t* __restrict__ post,
                                        const uint16_t* __restrict__ idxs, const ChunkHdr& sh, int nqc, int cy) {
    const ChunkGeom& g = a.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const QtThr th = qt_thr(a, nqc, cy, sh.U[threadIdx.x & 31]);
    const uint32_t cmask = (uint32_t)g.cap - 1;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t U32 = sh.U[lane];
    const int q = cy * QT_QC + lane;
    const int64_t d0 = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t d1 = min(a.n_docs, d0 + a.docs_per_cta);
    for (int64_t dp = d0 + warp; dp < d1; dp += QT_WARPS) {
        const int64_t doc = a.docs ? a.docs[dp] : dp;
        if (doc < 0 || doc >= a.n) {
            if (lane < nqc && !a.thr) a.out[(int64_t)q * a.out_ld + dp] = __longlong_as_double(0x7ff8000000000000ll);
            if (lane == 0) atomicOr(a.err, FTI_ERR_RANGE);
            continue;
        }
        const uint32_t r0 = a.qt_off[doc], r1 = a.qt_off[doc + 1];
        const uint32_t W32 = a.W[doc];
        const unsigned long long A = a.A[doc];
        unsigned long long acc = 0;
        for (uint32_t rb = r0; rb < r1; rb += 32) {
            const uint32_t r = rb + lane;
            uint2 rec = make_uint2(FTI_EMPTY, 0);
            int id = -1;
            if (r < r1) {
                rec = a.qt[r];
                int h = probe_slot(keys, cmask, rec.x);
                if (h >= 0) id = idxs[h];
            }
            unsigned hm = __ballot_sync(0xffffffffu, id >= 0);
            // two hits per iteration: independent lookup chains the scheduler can overlap
            auto visit = [&](const uint2 e, uint32_t mmu) {
                if ((e.x >> lane) & 1u) {
                    const uint32_t p = post[e.y + __popc(e.x & lt)];
                    // U·m_μ and W·m_ν are < 2^32 (W, U ≤ 65535): 32-bit products, 64-bit accumulation
                    const uint32_t um = U32 * (mmu & 0xFFFFu);
                    const uint32_t wm = W32 * (p & 0xFFFFu);
                    acc += (unsigned long long)(um < wm ? um : wm) << (a.d_star - (int)((p >> 16) & 63u));
                }
            };
            while (hm) {
                const int l1 = __ffs(hm) - 1;
                hm &= hm - 1;
                const int l2 = hm ? __ffs(hm) - 1 : l1;
                const bool two = hm != 0u;
                hm &= hm - 1;
                const int id1 = __shfl_sync(0xffffffffu, id, l1);
                const uint32_t m1 = __shfl_sync(0xffffffffu, rec.y, l1);
                const int id2 = __shfl_sync(0xffffffffu, id, l2);
                const uint32_t m2 = __shfl_sync(0xffffffffu, rec.y, l2);
                const uint2 e1 = ent[id1];
                const uint2 e2 = two ? ent[id2] : make_uint2(0u, 0u);
                visit(e1, m1);
                visit(e2, m2);
            }
        }
        qt_store(a, sh, nqc, cy, dp, doc, acc, W32, A, th);
    }
}

// the scan of chunk cy by this CTA (dense or hash structure)
__device__ __forceinline__ void qt_chunk(const QtArgs& a, int cy, ChunkHdr& sh, DenseHdr& dh) {
    extern __shared__ uint32_t sm[];
    const ChunkGeom& g = a.g;
    uint32_t* keys = sm;                                  // cap
    uint2* ent_s = (uint2*)(keys + g.cap);                // ucap_s {query mask, posting offset}
    uint32_t* post_s = (uint32_t*)(ent_s + g.ucap_s);     // pcap_s
    uint16_t* idxs = (uint16_t*)(post_s + g.pcap_s);      // cap
    const uint8_t* src = a.chunks + (size_t)cy * g.stride;
    const uint8_t* dsrc = a.dchunks ? a.dchunks + (size_t)cy * a.dg.stride : nullptr;
    __syncthreads();   // the previous chunk's structures are consumed
    if (threadIdx.x == 0) {
        sh = *(const ChunkHdr*)src;
        dh = dsrc ? *(const DenseHdr*)dsrc : DenseHdr{0u, 0u, 0u, 0u};
    }
    __syncthreads();
    if (dh.flag) {
        uint32_t* bits = sm;
        uint32_t* rank = sm + a.dg.mw;
        uint16_t* post = (uint16_t*)(rank + a.dg.mw);
        const uint32_t* gb = (const uint32_t*)(dsrc + sizeof(DenseHdr));
        const int nwords = 2 * a.dg.mw + (int)dh.nU * QT_QC / 2;    // bits | rank | post, contiguous
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) sm[i] = gb[i];
        uint4* hq = (uint4*)(sm + ((2 * a.dg.mw + a.dg.cap * QT_QC / 2 + 3) & ~3));   // per-warp hit queues
        __syncthreads();
        if (a.d_star > 31)
            qt_scan_dense<true>(a, bits, rank, post, hq + (threadIdx.x >> 5) * 32, sh, (int)sh.nq, cy);
        else
            qt_scan_dense<false>(a, bits, rank, post, hq + (threadIdx.x >> 5) * 32, sh, (int)sh.nq, cy);
        return;
    }
    const int nU = (int)sh.nU, nP = min((int)sh.nP, g.pmax), nqc = (int)sh.nq;
    const uint2* ge = (const uint2*)(src + g.off_mask);
    const uint32_t* gp = (const uint32_t*)(src + g.off_post);
    // the hash lives in shared memory; masks/offsets/postings too when they fit, else in L2
    const uint2* ent = nU <= g.ucap_s ? ent_s : ge;
    const uint32_t* post = nP <= g.pcap_s ? post_s : gp;
    {
        const uint4* k4 = (const uint4*)(src + g.off_keys);
        for (int i = threadIdx.x; i < g.cap / 4; i += blockDim.x) ((uint4*)keys)[i] = k4[i];
        const uint4* i4 = (const uint4*)(src + g.off_idx);
        for (int i = threadIdx.x; i < g.cap / 8; i += blockDim.x) ((uint4*)idxs)[i] = i4[i];
        if (nU <= g.ucap_s)
            for (int i = threadIdx.x; i < nU; i += blockDim.x) ent_s[i] = ge[i];
        if (nP <= g.pcap_s)
            for (int i = threadIdx.x; i < nP; i += blockDim.x) post_s[i] = gp[i];
    }
    __syncthreads();
    if (nU <= g.ucap_s && nP <= g.pcap_s)
        qt_scan<true>(a, keys, ent_s, post_s, idxs, sh, nqc, cy);
    else
        qt_scan<false>(a, keys, ent, post, idxs, sh, nqc, cy);
}

// grid.y = chunks (or chunk pairs in pair mode), grid.x = doc ranges
__global__ void __launch_bounds__(QT_WARPS * 32) k_qt(QtArgs a) {
    extern __shared__ uint32_t sm[];
    __shared__ ChunkHdr sh, sh2;
    __shared__ DenseHdr dh;
    const int per = a.pair ? 2 : 1;
    const int cy0 = (int)blockIdx.y * per;
    const int cy1 = min(a.nchunks, cy0 + per);
    if (a.qflag) {   // fallback mode: chunks without a flagged query have nothing to do
        int f = 0;
        if (threadIdx.x < per * QT_QC) {
            const int q = cy0 * QT_QC + threadIdx.x;
            f = q < a.nq && a.qflag[q] != 0u;
        }
        if (!__syncthreads_or(f)) return;
    }
    if (a.pair && cy1 - cy0 == 2) {
        const uint8_t* d2 = a.dchunks2 + (size_t)blockIdx.y * a.dg.stride2;
        if (threadIdx.x == 0) {
            dh = *(const DenseHdr*)d2;
            sh = *(const ChunkHdr*)(a.chunks + (size_t)cy0 * a.g.stride);
            sh2 = *(const ChunkHdr*)(a.chunks + (size_t)(cy0 + 1) * a.g.stride);
        }
        __syncthreads();
        if (dh.flag) {
            uint32_t* bits = sm;
            uint32_t* rank = sm + a.dg.mw;
            uint16_t* post = (uint16_t*)(rank + a.dg.mw);
            const uint32_t* gb = (const uint32_t*)(d2 + sizeof(DenseHdr));
            const int nwords = 2 * a.dg.mw + (int)dh.nU * QT_QC / 2;
            for (int i = threadIdx.x; i < nwords; i += blockDim.x) sm[i] = gb[i];
            uint4* hq = (uint4*)(sm + ((2 * a.dg.mw + a.dg.cap2 * QT_QC / 2 + 3) & ~3));
            __syncthreads();
            if (a.d_star > 31)
                qt_scan_dense2<true>(a, bits, rank, post, hq + (threadIdx.x >> 5) * 32, sh, sh2, cy0);
            else
                qt_scan_dense2<false>(a, bits, rank, post, hq + (threadIdx.x >> 5) * 32, sh, sh2, cy0);
            return;
        }
    }
    for (int cy = cy0; cy < cy1; cy++) qt_chunk(a, cy, sh, dh);
}

}  // namespace

namespace {

// chunk structures of a query batch (shared by every scan of the batch) and the scan's geometry
struct QtPlan {
    ChunkGeom g;
    DenseGeom dg;
    int nchunks;
    size_t smem;
    int ctas_per_sm;
};

cudaError_t qt_prepare(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq, cudaStream_t st,
                       QtPlan& P) {
    P.g = chunk_geom(ds, L, std::min<int>(nq, QT_QC));
    P.nchunks = (nq + QT_QC - 1) / QT_QC;
    if (!chunk_fits(P.g)) return cudaErrorInvalidConfiguration;   // callers split such batches (qt_fit_queries)
    cudaError_t e = ds->s_chunk.reserve(P.g.stride * (size_t)P.nchunks);
    if (e != cudaSuccess) return e;
    size_t smem_c = 4ull * P.g.cap + 8ull * P.g.umax + 2ull * P.g.cap;
    e = cudaFuncSetAttribute(k_qt_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c);
    if (e != cudaSuccess) return e;
    k_qt_chunk<<<P.nchunks, 1024, smem_c, st>>>(d_qblock, L, nq, P.g, ds->s_chunk.as<uint8_t>(), ds->err_dev);
    fti_count_launches(1);
    // dense structure: node-id bitmap + ranks in shared memory (M ≤ ~393k nodes), union ≤ cap
    DenseGeom& dg = P.dg;
    dg = DenseGeom{};
    dg.mw = (int)((ds->ix->M + 31) / 32);
    const size_t dense_budget = 200 * 1024;
    dg.cap = 0;
    if ((size_t)dg.mw * 8 <= 96 * 1024 && !fti_opt(FT_OPT_QT_HASH))   // FT_OPT_QT_HASH: test option, hash path only
        dg.cap = (int)std::min<size_t>(2048, (dense_budget - (size_t)dg.mw * 8) / (QT_QC * 2)) & ~31;
    dg.stride = (sizeof(DenseHdr) + (size_t)dg.mw * 8 + (size_t)dg.cap * QT_QC * 2 + 15) / 16 * 16;
    if (dg.cap > 0) {
        e = ds->s_chunkd.reserve(dg.stride * (size_t)P.nchunks);
        if (e != cudaSuccess) return e;
        const size_t smem_d = (size_t)dg.mw * 8;
        e = cudaFuncSetAttribute(k_qt_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
        if (e != cudaSuccess) return e;
        k_qt_dense<<<P.nchunks, 1024, smem_d, st>>>(d_qblock, L, nq, dg, ds->s_chunkd.as<uint8_t>());
        fti_count_launches(1);
    }
    // chunk pairs (64 queries per record pass) when the dense path is on and there are ≥ 2 chunks
    dg.cap2 = 0;
    dg.stride2 = 0;
    if (dg.cap > 0 && P.nchunks >= 2 && !fti_opt(FT_OPT_QT_PAIR_OFF)) {
        const size_t avail = (size_t)212 * 1024 - (size_t)dg.mw * 8 - (size_t)QT_WARPS * 32 * 16;
        dg.cap2 = (int)std::min<size_t>(2880, avail / (QT_QC * 2)) & ~31;
        dg.stride2 = (sizeof(DenseHdr) + (size_t)dg.mw * 8 + (size_t)dg.cap2 * QT_QC * 2 + 15) / 16 * 16;
        const int npairs = (P.nchunks + 1) / 2;
        e = ds->s_chunkd2.reserve(dg.stride2 * (size_t)npairs);
        if (e != cudaSuccess) return e;
        const size_t smem_d = (size_t)dg.mw * 8;
        e = cudaFuncSetAttribute(k_qt_dense2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
        if (e != cudaSuccess) return e;
        k_qt_dense2<<<npairs, 1024, smem_d, st>>>(d_qblock, L, nq, dg, ds->s_chunkd2.as<uint8_t>());
        fti_count_launches(1);
    }
    const size_t hqb = (size_t)QT_WARPS * 32 * 16;
    P.smem = std::max<size_t>(4ull * P.g.cap + 8ull * P.g.ucap_s + 4ull * P.g.pcap_s + 2ull * P.g.cap,
                              dg.cap > 0 ? (size_t)dg.mw * 8 + (size_t)dg.cap * QT_QC * 2 + 16 + hqb : 0);
    if (dg.cap2 > 0) P.smem = std::max(P.smem, (size_t)dg.mw * 8 + (size_t)dg.cap2 * QT_QC * 2 + 16 + hqb);
    e = cudaFuncSetAttribute(k_qt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem);
    if (e != cudaSuccess) return e;
    P.ctas_per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&P.ctas_per_sm, k_qt, QT_WARPS * 32, P.smem);
    P.ctas_per_sm = std::max(1, P.ctas_per_sm);
    return cudaSuccess;
}

// one scan of n_docs docs (d_docs, or all) with the prepared chunks; `mode` carries the threshold /
// fallback fields (zero: plain values into d_out)
cudaError_t qt_scan(ft_dataset* ds, const QtPlan& P, int32_t nq, const int64_t* d_docs, int64_t n_docs, double* d_out,
                    int64_t out_ld, const QtArgs& mode, int waves, cudaStream_t st) {
    QtArgs a = mode;
    a.qt_off = ds->qt_off; a.qt = ds->qt; a.W = ds->W; a.A = ds->A;
    a.chunks = ds->s_chunk.as<uint8_t>(); a.g = P.g;
    a.dchunks = P.dg.cap > 0 ? ds->s_chunkd.as<uint8_t>() : nullptr; a.dg = P.dg;
    a.pair = P.dg.cap2 > 0 ? 1 : 0;
    a.nchunks = P.nchunks;
    a.dchunks2 = a.pair ? ds->s_chunkd2.as<uint8_t>() : nullptr;
    a.nq = nq; a.docs = d_docs; a.n_docs = n_docs; a.n = ds->n;
    a.out = d_out; a.out_ld = out_ld;
    a.d_star = ds->ix->d_star; a.l_root = ds->ix->l_root;
    a.pow2 = std::abs(a.l_root - a.d_star) <= 960 ? std::ldexp(1.0, a.l_root - a.d_star) : 0.0;
    a.pow2f = std::abs(a.l_root - a.d_star) <= 100 ? std::ldexp(1.0f, a.l_root - a.d_star) : 0.0f;
    a.wide = a.d_star > 31 ? 1 : 0;
    a.err = ds->err_dev;
    const int64_t target = (int64_t)148 * P.ctas_per_sm * waves;
    const int64_t rows_y = P.dg.cap2 > 0 ? (P.nchunks + 1) / 2 : P.nchunks;
    // whole waves only: the grid never exceeds `target` CTAs (rounding up had given the 1/32-sample
    // scan 160 CTAs on 148 SMs — a second wave of 12)
    int64_t bx = std::max<int64_t>(1, std::min<int64_t>((n_docs + 31) / 32, target / rows_y));
    a.docs_per_cta = (n_docs + bx - 1) / bx;
    bx = (n_docs + a.docs_per_cta - 1) / a.docs_per_cta;
    const int gy = a.pair ? (P.nchunks + 1) / 2 : P.nchunks;
    k_qt<<<dim3((unsigned)bx, (unsigned)gy), QT_WARPS * 32, P.smem, st>>>(a);
    fti_count_launches(1);
    return cudaGetLastError();
}

// CTAs per SM slot over a full scan (single chunks: 4 → 2.48 ms, 8 → 2.19, 12 → 2.34 ms per reviews
// batch; chunk pairs: 4 → 2.17, 6 → 2.41, 8 → 2.22, 16 → 2.37 ms, stress 3.76 / 3.79 / 3.84 / 4.00
// ms); FT_OPT_QT_WAVES tunes it
int qt_waves() { return fti_opt(FT_OPT_QT_WAVES) > 0 ? (int)fti_opt(FT_OPT_QT_WAVES) : 4; }

// flags [nq] from a row list {count, rows...}
__global__ void k_rows_to_flags(const int* __restrict__ list, uint32_t* __restrict__ flag, int32_t nq) {
    for (int i = threadIdx.x; i < nq; i += blockDim.x) flag[i] = 0u;
    __syncthreads();
    const int c = list[0];
    for (int i = threadIdx.x; i < c; i += blockDim.x) flag[list[1 + i]] = 1u;
}

}  // namespace

cudaError_t fti_launch_qt(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                          const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, double* d_out, int64_t out_ld,
                          cudaStream_t st) {
    (void)docs_ld;   // the Quadtree stage always scores one doc list shared by the batch
    if (nq <= 0 || n_docs <= 0) return cudaSuccess;
    const int qc = qt_fit_queries(ds, L);
    if (qc <= 0) return cudaErrorInvalidConfiguration;
    if (qc < QT_QC && nq > qc) {   // large supports on a deep tree: sub-batches of qc queries
        for (int32_t q0 = 0; q0 < nq; q0 += qc) {
            cudaError_t es = fti_launch_qt(ds, L, d_qblock + (size_t)q0 * L.stride, std::min<int32_t>(qc, nq - q0), d_docs,
                                           docs_ld, n_docs, d_out + (int64_t)q0 * out_ld, out_ld, st);
            if (es != cudaSuccess) return es;
        }
        return cudaSuccess;
    }
    QtPlan P;
    cudaError_t e = qt_prepare(ds, L, d_qblock, nq, st, P);
    if (e != cudaSuccess) return e;
    return qt_scan(ds, P, nq, d_docs, n_docs, d_out, out_ld, QtArgs{}, qt_waves(), st);
}

// The prefilter (a3 + a4 fused): per query the m smallest (Quadtree value, doc id)
// over all n docs, without writing the nq × n value matrix:
//   1. scan a strided sample of n_s = n / 32 docs; per query the threshold t_q ≥ the sample's
//      (r+1)-th smallest value (rounded up to FP32), r = E + 4√E + 8 with E = m·n_s/n the expected
//      sample rank of the m-th key (so count(value ≤ t_q) ≥ m over all docs except with vanishing
//      probability);
//   2. scan all docs, appending every (value, doc) with value ≤ t_q to the query's list;
//   3. select the m smallest (value, id) of each list (as a set: the Flowtree stage does not need
//      them ordered).  Exact whenever m ≤ |list| ≤ capacity: every doc with a value ≤ the m-th key
//      is listed;
//   4. rows where that fails (list too short or overflowing — rare) are recomputed in full and
//      selected as before (chunks and rows without such a query exit at once).
// Falls back to the unfused pair (values written, then selected) when n < 32·m.
cudaError_t fti_launch_prefilter(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq, int64_t m,
                                 int64_t* d_cand, double* d_cval, int* d_sel_scratch, cudaStream_t st) {
    const int64_t n = ds->n;
    cudaError_t e;
    if (nq <= 0) return cudaSuccess;
    const int qc = qt_fit_queries(ds, L);
    if (qc <= 0) return cudaErrorInvalidConfiguration;
    if (qc < QT_QC && nq > qc) {   // large supports on a deep tree: sub-batches of qc queries
        for (int32_t q0 = 0; q0 < nq; q0 += qc)
            if ((e = fti_launch_prefilter(ds, L, d_qblock + (size_t)q0 * L.stride, std::min<int32_t>(qc, nq - q0), m,
                                          d_cand + (int64_t)q0 * m, d_cval + (int64_t)q0 * m, d_sel_scratch, st)) !=
                cudaSuccess)
                return e;
        return cudaSuccess;
    }
    const int64_t ns = n / 32;
    if (n < 32 * m || fti_opt(FT_OPT_PREFILTER_UNFUSED) || ns < 1) {
        if ((e = ds->s_vals.reserve(sizeof(double) * nq * n)) != cudaSuccess) return e;
        if ((e = fti_launch_qt(ds, L, d_qblock, nq, nullptr, 0, n, ds->s_vals.as<double>(), n, st)) != cudaSuccess)
            return e;
        return fti_launch_select(ds->s_vals.as<double>(), n, nullptr, 0, n, nq, (int32_t)m, d_cand, d_cval, m,
                                 d_sel_scratch, st);
    }
    // the strided sample's doc ids, built once per dataset
    if (ds->pf_ns != ns) {
        std::vector<int64_t> h((size_t)ns);
        for (int64_t i = 0; i < ns; i++) h[(size_t)i] = i * n / ns;
        if ((e = ds->s_pf_samp.reserve(sizeof(int64_t) * ns)) != cudaSuccess) return e;
        if ((e = cudaMemcpy(ds->s_pf_samp.p, h.data(), sizeof(int64_t) * ns, cudaMemcpyHostToDevice)) != cudaSuccess)
            return e;
        ds->pf_ns = ns;
    }
    const double ex = (double)m * (double)ns / (double)n;
    const int64_t r = std::min<int64_t>(ns - 1, (int64_t)std::ceil(ex + 4.0 * std::sqrt(ex) + 8.0));
    const int64_t cap = FTI_PREFILTER_CAP;
    if ((e = ds->s_pf_sval.reserve(sizeof(double) * nq * ns)) != cudaSuccess) return e;
    if ((e = ds->s_pf_tval.reserve(sizeof(double) * nq)) != cudaSuccess) return e;
    if ((e = ds->s_pf_cnt.reserve(sizeof(uint32_t) * nq)) != cudaSuccess) return e;
    if ((e = ds->s_pf_cval.reserve(sizeof(double) * nq * cap)) != cudaSuccess) return e;
    if ((e = ds->s_pf_cid.reserve(sizeof(int64_t) * nq * cap)) != cudaSuccess) return e;
    if ((e = ds->s_pf_bad.reserve(sizeof(int) * ((size_t)nq + 1))) != cudaSuccess) return e;
    if ((e = ds->s_pf_flag.reserve(sizeof(uint32_t) * nq)) != cudaSuccess) return e;
    QtPlan P;
    if ((e = qt_prepare(ds, L, d_qblock, nq, st, P)) != cudaSuccess) return e;
    // 1. the sample and its per-query threshold
    if ((e = qt_scan(ds, P, nq, ds->s_pf_samp.as<int64_t>(), ns, ds->s_pf_sval.as<double>(), ns, QtArgs{},
                     std::max(1, qt_waves() / 4), st)) != cudaSuccess)
        return e;
    if ((e = fti_launch_row_threshold(ds->s_pf_sval.as<double>(), ns, ns, nq, r, ds->s_pf_tval.as<double>(), st)) !=
        cudaSuccess)
        return e;
    // 2. every doc ≤ its query's threshold into the query's list
    if ((e = cudaMemsetAsync(ds->s_pf_cnt.p, 0, sizeof(uint32_t) * nq, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ds->s_pf_bad.p, 0, sizeof(int), st)) != cudaSuccess) return e;
    QtArgs tm{};
    tm.thr = ds->s_pf_tval.as<double>();
    tm.thr_ld = 1;
    tm.ccnt = ds->s_pf_cnt.as<uint32_t>();
    tm.cval = ds->s_pf_cval.as<double>();
    tm.cid = ds->s_pf_cid.as<int64_t>();
    tm.ccap = cap;
    if ((e = qt_scan(ds, P, nq, nullptr, n, nullptr, 0, tm, qt_waves(), st)) != cudaSuccess) return e;
    // 3. the m smallest of each list; rows whose list is short or overflowed are listed in pf_bad
    if ((e = fti_launch_select(ds->s_pf_cval.as<double>(), cap, ds->s_pf_cid.as<int64_t>(), cap, cap, nq, (int32_t)m,
                               d_cand, d_cval, m, d_sel_scratch, st, 0, ds->s_pf_cnt.as<uint32_t>(), nullptr, nullptr,
                               ds->s_pf_bad.as<int>(), /*nosort=*/true)) != cudaSuccess)
        return e;
    // 4. those rows in full (every other CTA exits at once)
    if ((e = ds->s_vals.reserve(sizeof(double) * nq * n)) != cudaSuccess) return e;
    k_rows_to_flags<<<1, 1024, 0, st>>>(ds->s_pf_bad.as<int>(), ds->s_pf_flag.as<uint32_t>(), nq);
    fti_count_launches(1);
    QtArgs fb{};
    fb.qflag = ds->s_pf_flag.as<uint32_t>();
    if ((e = qt_scan(ds, P, nq, nullptr, n, ds->s_vals.as<double>(), n, fb, 1, st)) != cudaSuccess) return e;
    return fti_launch_select(ds->s_vals.as<double>(), n, nullptr, 0, n, nq, (int32_t)m, d_cand, d_cval, m,
                             d_sel_scratch, st, 0, nullptr, ds->s_pf_bad.as<int>() + 1, ds->s_pf_bad.as<int>());
}
