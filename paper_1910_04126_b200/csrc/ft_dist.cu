// ft_dist.cu — a5: distance table D[c][j] = ||x_{v_c} − y_j||_2 between the candidate vocabulary and
// the query support, read by the Flowtree kernel to price its flow (
// Lemma 1's O(d) per matched pair).
//
// The table is a dense contraction, so it runs on the 5th-generation tensor cores (tcgen05):
//   ||x − y||^2 = ||x − c||^2 + ||y − c||^2 − 2 (x − c)·(y − c),   c = the query's centroid
// (centering keeps the Gram-form cancellation small for the near pairs that matter).  The dot
// products are 3xTF32 — every operand split as hi = tf32_rn(v), lo = v − hi, and
// D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi — keeping ~22 significant bits, FP32 accumulation in TMEM.
//
// k_dist_tc is persistent and warp specialised over a device-built list of (query, 128-row tile)
// work items:
//   * 4 producer warps, one candidate row per thread: cp.async (16 B) streams the row's raw fp32
//     K-chunks into a private 4-deep ring, then the thread centres, splits and writes the chunk into
//     the A stage in the canonical K-major core-matrix layout (SWIZZLE_NONE, LBO 128 B, SBO 512 B);
//     thread 0 also bulk-copies (cp.async.bulk, mbarrier complete_tx) the query's pre-split B chunk;
//   * 1 MMA warp: one thread waits the stage's full barrier, issues 2 K-steps × 3 tcgen05.mma
//     (kind::tf32, M=128, N=NP) and commits the stage's empty barrier; after the last chunk it commits
//     the tile's accumulator barrier;
//   * 4 epilogue warps: tcgen05.ld (32x32b) the accumulator (TMEM double buffer), form the distance
//     in FP32, force an id present on both sides to exactly 0, write the row.
// k_dist_prep computes per query the centroid, the pre-split B chunks and ||y − c||^2.
//
// Candidate vocabulary for the prefiltered pipeline: k_mark flags every vocab id of the query's
// m candidates in a per-query map [N], k_compact turns the flags into dense row ids and the row
// list (block-wide scan over N), k_row_base places each query's rows compactly and lists the tiles.
#include <algorithm>

#include "ft_device.cuh"

namespace {

constexpr int TM = 128;                 // rows per work item = UMMA M
constexpr int KC = 16;                  // K elements per chunk (64 B per row)
constexpr int RR = 4;                   // raw cp.async ring depth per producer thread
constexpr int NCB = 256;                // query points per column block = max UMMA N
constexpr int SBO = (KC / 4) * 128;     // bytes between 8-row core-matrix groups
constexpr int NPROD = 256;              // producer threads: 2 per row, 8 of the 16 K elements each
constexpr int MMA_WARP = NPROD / 32;    // warp 8
constexpr int NTHREADS = NPROD + 32 + 128;   // 8 producer + 1 MMA + 4 epilogue warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    // K-major, SWIZZLE_NONE: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)((uint32_t)SBO >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ uint32_t tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// byte offset of element (r, k) of a [rows x KC] K-major tile in core-matrix layout
__device__ __forceinline__ uint32_t cm_off(int r, int k) {
    return (uint32_t)((r >> 3) * SBO + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ void split_store(uint8_t* hi_base, uint8_t* lo_base, int r, int g, float4 v) {
    uint4 h, l;
    h.x = tf32_rn(v.x); l.x = __float_as_uint(v.x - __uint_as_float(h.x));
    h.y = tf32_rn(v.y); l.y = __float_as_uint(v.y - __uint_as_float(h.y));
    h.z = tf32_rn(v.z); l.z = __float_as_uint(v.z - __uint_as_float(h.z));
    h.w = tf32_rn(v.w); l.w = __float_as_uint(v.w - __uint_as_float(h.w));
    const uint32_t o = cm_off(r, 4 * g);
    *(uint4*)(hi_base + o) = h;
    *(uint4*)(lo_base + o) = l;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(RR - 1) : "memory"); }

struct DistArgs {
    const float* X;
    int d;
    int nch;                    // K chunks = ceil(d / KC)
    const uint8_t* qblock;
    QueryLayout L;
    int nq;
    const float* centers;       // [nq][d]
    const uint8_t* bsplit;      // [nq][nch][NPa*128 B]
    const float* ny;            // [nq][NPa]
    const int32_t* rows;        // [nq][rows_cap] or null (row = vocab)
    const int32_t* rowcnt;      // [nq] or null (N)
    int64_t rows_cap;
    const int64_t* row_base;    // [nq] or null (q * rows_cap)
    const int64_t* tile_base;   // [nq + 1] exclusive prefix of tiles per query
    float* table;
    int ld;
    int cb;                     // column block (query points cb*256 ...)
    int NPa;                    // padded N of the MMA (multiple of 16, ≤ 256)
    int R;                      // stage ring depth
};

__device__ __forceinline__ void decode_tile(const DistArgs& a, int64_t w, int& q, int64_t& tile) {
    int lo = 0, hi = a.nq - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.tile_base[mid] <= w) lo = mid; else hi = mid - 1;
    }
    q = lo;
    tile = w - a.tile_base[q];
}

__global__ void __launch_bounds__(NTHREADS, 1) k_dist_tc(DistArgs a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t a_bytes = TM * KC * 4;              // one of hi / lo
    const uint32_t b_bytes = (uint32_t)a.NPa * KC * 4;
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
    uint8_t* stages = sm;
    float* raw = (float*)(sm + (size_t)a.R * stage_bytes);        // [RR][TM][KC]
    float* nxs = raw + RR * TM * KC;                                // [2 buffers][2 halves][TM]
    float* eny = nxs + 4 * TM;                                      // [NCB] ||y − c||^2 (epilogue)
    uint32_t* eyid = (uint32_t*)(eny + NCB);                        // [NCB] query vocab ids (epilogue)
    uint64_t* bars = (uint64_t*)(eyid + NCB);                       // full[R], empty[R], accf[2], acce[2], nxr[2]
    uint64_t* full = bars;
    uint64_t* empty = bars + a.R;
    uint64_t* accf = bars + 2 * a.R;
    uint64_t* acce = accf + 2;
    uint64_t* nxr = acce + 2;
    uint32_t* tmem_slot = (uint32_t*)(nxr + 2);

    const int64_t T = a.tile_base[a.nq];
    const uint32_t ncols = (uint32_t)fti_pow2_at_least(max(32, 2 * a.NPa));
    if (t == 0) {
        for (int s = 0; s < a.R; s++) { mbar_init(&full[s], NPROD + 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; b++) { mbar_init(&accf[b], 1); mbar_init(&acce[b], TM); mbar_init(&nxr[b], NPROD); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp < MMA_WARP) {
        // ------------------------------------------------------------------ producers
        // thread t handles row r = t % 128, K elements [8h, 8h + 8) of every 16-wide chunk, h = t / 128
        const bool vec = (a.d & 3) == 0;
        const int r = t & (TM - 1), h = t >> 7;
        uint32_t it = 0;
        int k = 0;
        for (int64_t w = blockIdx.x; w < T; w += gridDim.x, k++) {
            int q;
            int64_t tile;
            decode_tile(a, w, q, tile);
            const int64_t nrows = a.rowcnt ? (int64_t)a.rowcnt[q] : a.rows_cap;
            const int64_t row = tile * TM + r;
            const int32_t xid = row < nrows ? (a.rows ? a.rows[(int64_t)q * a.rows_cap + row] : (int32_t)row) : -1;
            const float* xr = a.X + (int64_t)(xid >= 0 ? xid : 0) * a.d;
            const float* cq = a.centers + (int64_t)q * a.d;
            const uint8_t* bq = a.bsplit + (size_t)q * a.nch * (2 * b_bytes);
            float* myraw = raw + r * KC + 8 * h;
            auto issue = [&](int cc) {
                if (xid >= 0 && cc < a.nch) {
                    float* dst = myraw + (cc % RR) * TM * KC;
                    const int k0 = cc * KC + 8 * h;
                    if (vec) {
#pragma unroll
                        for (int g = 0; g < 2; g++)
                            if (k0 + 4 * g < a.d) cp_async16(dst + 4 * g, xr + k0 + 4 * g);
                    } else {
                        for (int e = 0; e < 8; e++)
                            if (k0 + e < a.d) cp_async4(dst + e, xr + k0 + e);
                    }
                }
                cp_commit();
            };
            for (int cc = 0; cc < RR - 1; cc++) issue(cc);
            float nx = 0.f;
            const int b = k & 1;
            for (int cc = 0; cc < a.nch; cc++, it++) {
                issue(cc + RR - 1);
                cp_wait_ring();
                const int s = (int)(it % (uint32_t)a.R);
                const uint32_t rnd = it / (uint32_t)a.R;
                if (rnd > 0) mbar_wait(&empty[s], (rnd - 1) & 1u);
                uint8_t* st = stages + (size_t)s * stage_bytes;
                if (t == 0) {
                    mbar_arrive_tx(&full[s], 2 * b_bytes);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(st + 2 * a_bytes)),
                        "l"(bq + (size_t)cc * 2 * b_bytes), "r"(2 * b_bytes), "r"(smem_u32(&full[s]))
                        : "memory");
                }
                const float* src = myraw + (cc % RR) * TM * KC;
                const int k0 = cc * KC + 8 * h;
#pragma unroll
                for (int g = 0; g < 2; g++) {
                    const int kk = k0 + 4 * g;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (xid >= 0) {
                        const float4 r4 = *(const float4*)(src + 4 * g);
                        float4 c4;
                        if (vec && kk < a.d) {
                            c4 = __ldg((const float4*)(cq + kk));
                        } else {
                            c4.x = kk + 0 < a.d ? cq[kk + 0] : 0.f;
                            c4.y = kk + 1 < a.d ? cq[kk + 1] : 0.f;
                            c4.z = kk + 2 < a.d ? cq[kk + 2] : 0.f;
                            c4.w = kk + 3 < a.d ? cq[kk + 3] : 0.f;
                        }
                        v.x = kk + 0 < a.d ? r4.x - c4.x : 0.f;
                        v.y = kk + 1 < a.d ? r4.y - c4.y : 0.f;
                        v.z = kk + 2 < a.d ? r4.z - c4.z : 0.f;
                        v.w = kk + 3 < a.d ? r4.w - c4.w : 0.f;
                    }
                    nx = fmaf(v.x, v.x, nx); nx = fmaf(v.y, v.y, nx); nx = fmaf(v.z, v.z, nx); nx = fmaf(v.w, v.w, nx);
                    split_store(st, st + a_bytes, r, 2 * h + g, v);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&full[s]);
            }
            // hand the partial ||x − c||^2 to the epilogue (after it released this buffer two tiles ago)
            if (k >= 2) mbar_wait(&acce[b], ((k >> 1) - 1) & 1);
            nxs[(b * 2 + h) * TM + r] = nx;
            mbar_arrive(&nxr[b]);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(a.NPa >> 3) << 17) |
                               ((uint32_t)(TM >> 4) << 24);
        uint32_t it = 0;
        int k = 0;
        for (int64_t w = blockIdx.x; w < T; w += gridDim.x, k++) {
            const int b = k & 1;
            if (k >= 2) mbar_wait(&acce[b], ((k >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t dt = tmem + (uint32_t)(b * a.NPa);
            for (int cc = 0; cc < a.nch; cc++, it++) {
                const int s = (int)(it % (uint32_t)a.R);
                mbar_wait(&full[s], (it / (uint32_t)a.R) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(stages + (size_t)s * stage_bytes);
#pragma unroll
                    for (int ks = 0; ks < KC / 8; ks++) {
                        const uint64_t ah = umma_desc(st + 256 * ks), al = umma_desc(st + a_bytes + 256 * ks);
                        const uint64_t bh = umma_desc(st + 2 * a_bytes + 256 * ks);
                        const uint64_t bl = umma_desc(st + 2 * a_bytes + b_bytes + 256 * ks);
                        const uint32_t acc0 = (cc > 0 || ks > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
                            "l"(ah), "l"(bh), "r"(idesc), "r"(acc0));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(dt), "l"(ah),
                                     "l"(bl), "r"(idesc));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(dt), "l"(al),
                                     "l"(bh), "r"(idesc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&empty[s]))
                                 : "memory");
                }
                __syncwarp();
            }
            if (lane == 0)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&accf[b]))
                             : "memory");
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------------ epilogue
        const int quarter = warp & 3;                 // TMEM lanes 32*quarter .. +31
        const int r = quarter * 32 + lane;
        const int et = t - (NPROD + 32);              // 0..127 within the epilogue warps
        int k = 0, cur_q = -1;
        for (int64_t w = blockIdx.x; w < T; w += gridDim.x, k++) {
            const int b = k & 1;
            int q;
            int64_t tile;
            decode_tile(a, w, q, tile);
            const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
            const QHeader* hdr = (const QHeader*)slot;
            const int sq = hdr->err ? 0 : (int)hdr->s;
            const int nb = min(NCB, max(0, sq - a.cb * NCB));
            if (q != cur_q) {   // stage the query's ids and norms once per query (named barrier: epilogue only)
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const uint2* qitems = (const uint2*)(slot + a.L.off_items);
                for (int j = et; j < NCB; j += 128) {
                    eyid[j] = j < nb ? (qitems[a.cb * NCB + j].x & FTI_VOCAB_MASK) : 0xFFFFFFFFu;
                    eny[j] = j < a.NPa ? a.ny[(int64_t)q * a.NPa + j] : 0.f;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                cur_q = q;
            }
            const int64_t nrows = a.rowcnt ? (int64_t)a.rowcnt[q] : a.rows_cap;
            const int64_t row = tile * TM + r;
            const int32_t xid = row < nrows ? (a.rows ? a.rows[(int64_t)q * a.rows_cap + row] : (int32_t)row) : -1;
            float* trow = a.table + ((a.row_base ? a.row_base[q] : (int64_t)q * a.rows_cap) + row) * a.ld + a.cb * NCB;
            mbar_wait(&nxr[b], (k >> 1) & 1);
            const float nx = nxs[(b * 2) * TM + r] + nxs[(b * 2 + 1) * TM + r];
            mbar_wait(&accf[b], (k >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * a.NPa);
            for (int c0 = 0; c0 < a.NPa; c0 += 8) {
                uint32_t v[8];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                    : "r"(tb + (uint32_t)c0));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (xid >= 0 && c0 < nb) {
                    float o[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int j = c0 + i;
                        const float d2 = nx + eny[j] - 2.f * __uint_as_float(v[i]);
                        o[i] = ((uint32_t)xid == eyid[j]) ? 0.f : sqrtf(fmaxf(d2, 0.f));
                    }
                    if (c0 + 8 <= nb && ((a.ld & 3) == 0)) {
                        *(float4*)(trow + c0) = make_float4(o[0], o[1], o[2], o[3]);
                        *(float4*)(trow + c0 + 4) = make_float4(o[4], o[5], o[6], o[7]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; i++)
                            if (c0 + i < nb) trow[c0 + i] = o[i];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&acce[b]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

// per query: centroid c (FP32 mean of the support points), the centred query points of column
// block cb split into TF32 hi/lo in the MMA core-matrix layout per K chunk, and ||y − c||^2
__global__ void __launch_bounds__(256) k_dist_prep(DistArgs a, float* __restrict__ centers,
                                                  uint8_t* __restrict__ bsplit, float* __restrict__ ny) {
    __shared__ uint32_t yid[NCB];
    const int q = blockIdx.x;
    const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    const uint2* qitems = (const uint2*)(slot + a.L.off_items);
    const int s = hdr->err ? 0 : (int)hdr->s;
    float* cq = centers + (int64_t)q * a.d;
    for (int i = threadIdx.x; i < a.d; i += blockDim.x) {
        float acc = 0.f;
        for (int j = 0; j < s; j++) acc += a.X[(int64_t)(qitems[j].x & FTI_VOCAB_MASK) * a.d + i];
        cq[i] = s ? acc / (float)s : 0.f;
    }
    const int nb = min(NCB, max(0, s - a.cb * NCB));
    for (int j = threadIdx.x; j < NCB; j += blockDim.x)
        yid[j] = j < nb ? (qitems[a.cb * NCB + j].x & FTI_VOCAB_MASK) : 0xFFFFFFFFu;
    __syncthreads();
    const uint32_t b_bytes = (uint32_t)a.NPa * KC * 4;
    uint8_t* bq = bsplit + (size_t)q * a.nch * (2 * b_bytes);
    // thread per (chunk, row, 4-group)
    const int groups = a.nch * a.NPa * (KC / 4);
    for (int e = threadIdx.x; e < groups; e += blockDim.x) {
        const int g = e % (KC / 4);
        const int j = (e / (KC / 4)) % a.NPa;
        const int cc = e / ((KC / 4) * a.NPa);
        const int k = cc * KC + 4 * g;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < nb) {
            const float* yr = a.X + (int64_t)yid[j] * a.d;
            v.x = k + 0 < a.d ? yr[k + 0] - cq[k + 0] : 0.f;
            v.y = k + 1 < a.d ? yr[k + 1] - cq[k + 1] : 0.f;
            v.z = k + 2 < a.d ? yr[k + 2] - cq[k + 2] : 0.f;
            v.w = k + 3 < a.d ? yr[k + 3] - cq[k + 3] : 0.f;
        }
        uint8_t* st = bq + (size_t)cc * 2 * b_bytes;
        split_store(st, st + b_bytes, j, g, v);
    }
    for (int j = threadIdx.x; j < a.NPa; j += blockDim.x) {
        float acc = 0.f;
        if (j < nb) {
            const float* yr = a.X + (int64_t)yid[j] * a.d;
            for (int k = 0; k < a.d; k++) {
                const float v = yr[k] - cq[k];
                acc = fmaf(v, v, acc);
            }
        }
        ny[(int64_t)q * a.NPa + j] = acc;
    }
}

// one CTA per query: the candidates' vocabulary as a shared-memory bitmap (shared atomics), then
// per-word ranks (dense row ids in vocab order), the row list and the row count
__global__ void __launch_bounds__(1024) k_vocab(const uint32_t* __restrict__ doc_off, const uint2* __restrict__ items,
                                                const int64_t* __restrict__ cand, int64_t cand_ld, int64_t n_cand,
                                                int64_t nwords, uint2* __restrict__ map, int32_t* __restrict__ rows,
                                                int32_t* __restrict__ rowcnt, int64_t rows_cap) {
    extern __shared__ uint32_t sbits[];
    __shared__ int tmp[32];
    const int q = blockIdx.x;
    for (int64_t i = threadIdx.x; i < nwords; i += blockDim.x) sbits[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t c = warp; c < n_cand; c += nw) {
        const int64_t doc = cand[(int64_t)q * cand_ld + c];
        if (doc < 0) continue;
        const uint32_t i0 = doc_off[doc], i1 = doc_off[doc + 1];
        for (uint32_t i = i0 + lane; i < i1; i += 32) {
            const uint32_t x = items[i].x & FTI_VOCAB_MASK;
            atomicOr(&sbits[x >> 5], 1u << (x & 31));
        }
    }
    __syncthreads();
    uint2* mq = map + (int64_t)q * nwords;
    int32_t* rq = rows + (int64_t)q * rows_cap;
    int run = 0;
    for (int64_t c = 0; c < nwords; c += blockDim.x) {
        const int64_t wi = c + threadIdx.x;
        uint32_t bits = wi < nwords ? sbits[wi] : 0u;
        int tot;
        const int r = run + fti_block_exclusive_sum(__popc(bits), tmp, &tot);
        if (wi < nwords) {
            mq[wi] = make_uint2(bits, (uint32_t)r);
            int rr = r;
            while (bits) {
                const int bpos = __ffs(bits) - 1;
                bits &= bits - 1;
                if (rr < rows_cap) rq[rr] = (int32_t)(wi * 32 + bpos);
                rr++;
            }
        }
        run += tot;
    }
    if (threadIdx.x == 0) rowcnt[q] = run < rows_cap ? run : (int32_t)rows_cap;
}

// compact table placement (exclusive prefix of the row counts) and the work list of 128-row tiles
// (with `units`: adds the stage's algorithmic bytes Σ_q rows_q · (4 d + 4 s_q) for the profiler)
__global__ void k_row_base(const int32_t* __restrict__ rowcnt, int64_t rows_cap, int nq,
                           int64_t* __restrict__ row_base, int64_t* __restrict__ tile_base,
                           const uint8_t* qblock, QueryLayout L, int d, unsigned long long* units) {
    if (threadIdx.x == 0) {
        int64_t acc = 0, tacc = 0;
        unsigned long long bytes = 0;
        for (int q = 0; q < nq; q++) {
            const int64_t r = rowcnt ? (int64_t)rowcnt[q] : rows_cap;
            if (row_base) row_base[q] = acc;
            if (tile_base) tile_base[q] = tacc;
            acc += r;
            tacc += (r + TM - 1) / TM;
            if (units) {
                const QHeader* h = (const QHeader*)(qblock + (size_t)q * L.stride);
                bytes += (unsigned long long)r * (4ull * d + 4ull * (h->err ? 0u : h->s));
            }
        }
        if (tile_base) tile_base[nq] = tacc;
        if (units) atomicAdd(units, bytes);
    }
}

}  // namespace

cudaError_t fti_launch_dist_table(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                                  const int32_t* d_rows, const int32_t* d_rowcnt, int64_t rows_cap,
                                  const int64_t* d_row_base, float* d_table, int32_t ld, cudaStream_t st) {
    if (nq <= 0 || rows_cap <= 0) return cudaSuccess;
    const ft_index* ix = ds->ix;
    DistArgs a{};
    a.X = ix->X;
    a.d = ix->d;
    a.nch = (ix->d + KC - 1) / KC;
    a.qblock = d_qblock;
    a.L = L;
    a.nq = nq;
    a.rows = d_rows;
    a.rowcnt = d_rowcnt;
    a.rows_cap = rows_cap;
    a.row_base = d_row_base;
    a.table = d_table;
    a.ld = ld;
    const int ncb = (L.smax + NCB - 1) / NCB;
    const int np_max = std::min(NCB, L.smax);
    a.NPa = std::max(16, ((np_max + 15) / 16) * 16);
    const size_t b_bytes = (size_t)a.NPa * KC * 4;
    cudaError_t e;
    if ((e = ds->s_centers.reserve((size_t)nq * ix->d * 4)) != cudaSuccess) return e;
    if ((e = ds->s_bsplit.reserve((size_t)nq * a.nch * 2 * b_bytes)) != cudaSuccess) return e;
    if ((e = ds->s_ny.reserve((size_t)nq * a.NPa * 4)) != cudaSuccess) return e;
    if ((e = ds->s_tiles.reserve((size_t)(nq + 1) * 8)) != cudaSuccess) return e;
    a.centers = ds->s_centers.as<float>();
    a.bsplit = ds->s_bsplit.as<uint8_t>();
    a.ny = ds->s_ny.as<float>();
    a.tile_base = ds->s_tiles.as<int64_t>();
    k_row_base<<<1, 32, 0, st>>>(d_rowcnt, rows_cap, nq, nullptr, ds->s_tiles.as<int64_t>(), d_qblock, L, ix->d,
                                 ds->units_ptr(FTI_ST_DIST));
    const size_t stage_bytes = 2 * (size_t)TM * KC * 4 + 2 * b_bytes;
    const size_t fixed = (size_t)RR * TM * KC * 4 + 4 * TM * 4 + 2 * NCB * 4 + 64;
    const int R = (int)std::max<size_t>(2, std::min<size_t>(8, (200 * 1024 - fixed) / stage_bytes));
    a.R = R;
    const size_t smem = (size_t)R * stage_bytes + fixed + (size_t)(2 * R + 6) * 8 + 16;
    if ((e = cudaFuncSetAttribute(k_dist_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    for (int cb = 0; cb < ncb; cb++) {
        a.cb = cb;
        k_dist_prep<<<nq, 256, 0, st>>>(a, ds->s_centers.as<float>(), ds->s_bsplit.as<uint8_t>(), ds->s_ny.as<float>());
        k_dist_tc<<<148, NTHREADS, smem, st>>>(a);
        fti_count_launches(2);
    }
    fti_count_launches(1);
    return cudaGetLastError();
}

cudaError_t fti_launch_vocab_map(const ft_dataset* ds, int32_t nq, const int64_t* d_cand, int64_t cand_ld,
                                 int64_t n_cand, uint2* d_map, int32_t* d_rows, int32_t* d_rowcnt, int64_t rows_cap,
                                 int64_t* d_row_base, cudaStream_t st) {
    if (nq <= 0) return cudaSuccess;
    const int64_t nwords = (ds->ix->N + 31) / 32;
    const size_t smem = (size_t)nwords * 4;
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;   // N > 1.6M: not supported by the bitmap
    cudaError_t e = cudaFuncSetAttribute(k_vocab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_vocab<<<nq, 1024, smem, st>>>(ds->doc_off, ds->items, d_cand, cand_ld, n_cand, nwords, d_map, d_rows, d_rowcnt,
                                    rows_cap);
    k_row_base<<<1, 32, 0, st>>>(d_rowcnt, rows_cap, nq, d_row_base, nullptr, nullptr, QueryLayout{}, 0, nullptr);
    fti_count_launches(2);
    return cudaGetLastError();
}
