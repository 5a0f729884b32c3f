// ft_dist.cu — a5: distance table D[c][j] = ||x_{v_c} − y_j||_2 between the candidate vocabulary and
// the query support, read by the Flowtree kernel to price its flow (
// Lemma 1's O(d) per matched pair).
//
// The table is a dense contraction, so it runs on the 5th-generation tensor cores (tcgen05):
//   ||x − y||^2 = ||x̃||^2 + ||ỹ||^2 − 2 x̃·ỹ,   x̃ = x − μ,  μ = the FP64 mean of all points
// (translating by the mean removes any common offset of the embedding, which would otherwise
// dominate the Gram-form cancellation; ||x̃||^2 is precomputed per point in FP64).  The dot
// products are 3xTF32 — every operand split as hi = tf32_rn(v), lo = v − hi, and
// D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi — keeping ~22 significant bits, FP32 accumulation in TMEM.
// The translated points X̃ are kept once per index, FP32, rows padded to a multiple of 32 with a
// trailing all-zero row (the source of every padding row of a tile).
//
// k_dist_tc is persistent (one CTA per SM) and warp specialised over a device-built list of
// (query, 128-row tile) work items; each query has its own MMA width N = its support rounded up
// to 16 (≤ 96 per column block), so a batch with a long query does not pad the short ones:
//   * 4 copy warps cp.async whole 128-byte row segments of the tile's 32-wide K chunk into a
//     Q-deep raw ring in shared memory (row pitch 144 B), arriving on the slot's mbarrier with
//     cp.async.mbarrier.arrive.noinc; lane 0 of warp 0 bulk-copies (cp.async.bulk, complete_tx)
//     the query's pre-split B chunk [B_hi | B_lo] (canonical K-major core-matrix layout,
//     SWIZZLE_NONE, LBO 128 B, SBO 1024 B);
//   * 4 converter warps, thread = TMEM lane = tile row: read the raw row, write hi = raw and
//     lo = x − trunc_tf32(x) into a TMEM A ring with tcgen05.st.32x32b.x32;
//   * 1 MMA warp: an elected lane waits the slot's full barrier and issues 4 K-steps × 3
//     tcgen05.mma (kind::tf32, M = 128, N = N_q, A from TMEM): A_hi·B_hi, A_hi·B_lo, A_lo·B_hi into
//     one accumulator; it commits the slot's empty barrier, and after the last chunk the tile's
//     accumulator barrier;
//   * 8 epilogue warps (2 per TMEM lane quarter, alternating 16-column blocks): tcgen05.ld the
//     double-buffered accumulator, form the distance in FP32 (branch-free MUFU square root), force an
//     id present on both sides to exactly 0, write the rows coalesced through a per-warp transpose.
// k_tile_plan / k_tiles build the work list, k_dist_prep the per-query pre-split B chunks.
//
// Candidate vocabulary for the prefiltered pipeline: k_vocab marks every vocab id of the query's
// m candidates in a shared-memory bitmap and turns it into dense row ids and the row list;
// the host places each query's rows compactly (ft_api.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ft_device.cuh"

namespace {

constexpr int TM = 128;                 // rows per work item = UMMA M
constexpr int KC = 32;                  // K elements per chunk (128 B per row)
constexpr int NCB = 96;                 // query points per column block (accumulator N ≤ 96 columns)
constexpr int SBO = (KC / 4) * 128;     // B operand: bytes between 8-row core-matrix groups
constexpr int RPITCH = KC * 4 + 16;     // raw ring row pitch (bytes): conflict-free row- and granule-wise access
constexpr int NCOPY = 128;              // copy threads (warps 0-3)
constexpr int NCONV = 128;              // converter threads: one tile row each (warps 4-7)
constexpr int NLOAD = NCOPY + NCONV;
constexpr int MMA_WARP = NLOAD / 32;    // warp 8
constexpr int NEPI = 8;                 // epilogue warps: 2 per TMEM lane quarter, alternating 16-column blocks
constexpr int NTHREADS = NLOAD + 32 + 32 * NEPI;   // + 1 MMA + 8 epilogue warps
constexpr int MAXASLOT = 4;             // TMEM A ring: up to 4 slots of 2 KC columns (hi | lo)
constexpr uint32_t TMEM_COLS = 512;     // [0, 2 accw) double-buffered accumulators, then the A ring
constexpr int TPITCH = 20;              // epilogue transpose buffer pitch (floats): conflict-free float4 rows

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one elected lane of a converged warp; ptxas then knows the tcgen05.mma operands are uniform
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    // K-major, SWIZZLE_NONE: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)((uint32_t)SBO >> 4) << 32) | (1ull << 46);
}

// TF32 round to nearest, ties away from zero (= cvt.rna.tf32.f32 for finite x, which sm_100 would
// expand with an extra inf/nan guard): add half an ulp of the 10-bit mantissa, truncate
__device__ __forceinline__ uint32_t tf32_rn(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }

// byte offset of element (r, k) of a [rows x KC] K-major tile in core-matrix layout
__device__ __forceinline__ uint32_t cm_off(int r, int k) {
    return (uint32_t)((r >> 3) * SBO + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ void split_store(uint8_t* hi_base, uint8_t* lo_base, uint32_t o, float4 v) {
    uint4 h, l;
    h.x = tf32_rn(v.x); l.x = __float_as_uint(v.x - __uint_as_float(h.x));
    h.y = tf32_rn(v.y); l.y = __float_as_uint(v.y - __uint_as_float(h.y));
    h.z = tf32_rn(v.z); l.z = __float_as_uint(v.z - __uint_as_float(h.z));
    h.w = tf32_rn(v.w); l.w = __float_as_uint(v.w - __uint_as_float(h.w));
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
// this thread's TMEM lane, 32 consecutive 32-bit columns from `taddr`
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

// arrive on `bar` once all of this thread's prior cp.async copies have landed (count not incremented)
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct DistArgs {
    const float* Xc;            // [(N+1) * dpad] translated points, zero row N
    const float* xnorm;         // [N+1]
    int64_t N;
    int dpad;
    int nch;                    // K chunks = dpad / KC
    const uint8_t* qblock;
    QueryLayout L;
    int nq;
    const uint8_t* bsplit;      // query q at byte 16·qinfo[q].x: [nch][hi | lo][N_q x KC] core-matrix layout
    float* ny;                  // [nq][NCB] ||ỹ||^2
    uint2* qinfo;               // [nq] {B offset / 16 bytes, N_q (0: no columns in this block)}
    int4* wdesc;                // [T] {q, tile, B offset / 16 bytes, N_q}
    int32_t* wrow;              // [T][TM] vocab id of each row of the tile, −1 past the query's rows
    int64_t* tile_base;         // [nq + 1] exclusive prefix of tiles per query (T = tile_base[nq])
    const int32_t* rows;        // [nq][rows_cap] or null (row = vocab)
    const int32_t* rowcnt;      // [nq] or null (rows_cap)
    int64_t rows_cap;
    const int64_t* row_base;    // [nq] ELEMENT offset of each query's table
    const int32_t* pitch;       // [nq] per-query row pitch (floats)
    float* table;
    int cb;                     // column block (query points cb*256 ...)
    int NPmax;                  // B stage capacity: max N_q of the launch
    int Q;                      // raw ring depth (chunks in flight)
    int accw;                   // accumulator columns per buffer = NPmax
    int naslot;                 // TMEM A ring slots = (512 − 2 accw) / (2 KC)
};

__device__ unsigned long long g_dbg[16];
#define TW(i, stmt)                                          \
    do {                                                     \
        if (DBG) {                                           \
            const long long t0_ = clock64();                 \
            stmt;                                            \
            dbg[i] += (unsigned long long)(clock64() - t0_); \
        } else {                                             \
            stmt;                                            \
        }                                                    \
    } while (0)

template <bool DBG>
__global__ void __launch_bounds__(NTHREADS, 1) k_dist_tc(DistArgs a) {
    unsigned long long dbg[4] = {0, 0, 0, 0};
    const long long tstart = clock64();
    extern __shared__ __align__(1024) uint8_t sm[];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // shared memory: raw ring [Q][TM rows][RPITCH] | B ring [NASLOT][hi | lo][NPmax x KC] |
    // epilogue staging | barriers.  TMEM: accumulators [0, 256), A ring [256, 512) of hi | lo slots.
    const uint32_t raw_bytes = TM * RPITCH;
    const uint32_t b_slot = 2 * (uint32_t)a.NPmax * KC * 4;
    uint8_t* rring = sm;
    uint8_t* bring = sm + (size_t)a.Q * raw_bytes;
    const int NASLOT = a.naslot;
    const uint32_t ACC_COLS = 2 * (uint32_t)a.accw;
    float* eny = (float*)(bring + (size_t)MAXASLOT * b_slot);         // [NCB] ||ỹ||^2 (epilogue)
    uint32_t* eyid = (uint32_t*)(eny + NCB);                        // [NCB] query vocab ids (epilogue)
    float* tstage = (float*)(eyid + NCB);                           // [NEPI warps][32][TPITCH] epilogue transpose
    uint64_t* bars = (uint64_t*)(tstage + NEPI * 32 * TPITCH);
    uint64_t* rawf = bars;                  // [Q] raw chunk landed (copy threads, noinc)
    uint64_t* remp = rawf + a.Q;            // [Q] raw slot read (converter warps)
    uint64_t* full = remp + a.Q;            // [NASLOT] A slot written + B landed
    uint64_t* aemp = full + MAXASLOT;       // [NASLOT] A/B slot released (MMA commit)
    uint64_t* accf = aemp + MAXASLOT;
    uint64_t* acce = accf + 2;
    uint32_t* tmem_slot = (uint32_t*)(acce + 2);

    // each CTA takes a contiguous range of work items (tiles of a query are adjacent, so the query
    // changes rarely within a CTA)
    const int64_t T = a.tile_base[a.nq];
    const int64_t w_begin = T * blockIdx.x / gridDim.x, w_end = T * (blockIdx.x + 1) / gridDim.x;
    if (t == 0) {
        for (int q = 0; q < a.Q; q++) { mbar_init(&rawf[q], NCOPY); mbar_init(&remp[q], NCONV / 32); }
        for (int s = 0; s < NASLOT; s++) { mbar_init(&full[s], NCONV / 32 + 1); mbar_init(&aemp[s], 1); }
        for (int b = 0; b < 2; b++) { mbar_init(&accf[b], 1); mbar_init(&acce[b], 32 * NEPI); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (t < NCOPY) {
        // ------------------------------------------------------------------ copy threads
        // warp cw copies rows 32 cw .. +31 of each K chunk into a raw slot; lane → (row & 7,
        // granule): each cp.async instruction moves 8 rows × 64 contiguous bytes (full sectors) into
        // 8 distinct bank quads; arrive (noinc) on the slot's barrier when they land.
        const int rl = lane & 7, g0 = lane >> 3;
        const int rbase = warp * 32;
        uint32_t off[8];
#pragma unroll
        for (int rg = 0; rg < 4; rg++)
#pragma unroll
            for (int h = 0; h < 2; h++) off[2 * rg + h] = (uint32_t)((rbase + 8 * rg + rl) * RPITCH + 16 * (4 * h + g0));
        int32_t px[4];
#pragma unroll
        for (int rg = 0; rg < 4; rg++) px[rg] = w_begin < w_end ? a.wrow[w_begin * TM + rbase + 8 * rg + rl] : -1;
        int q = 0;
        uint32_t eph = 0;
        bool first = true;
        for (int64_t w = w_begin; w < w_end; w++) {
            const float* src[4];
#pragma unroll
            for (int rg = 0; rg < 4; rg++) {
                src[rg] = a.Xc + (px[rg] >= 0 ? (int64_t)px[rg] : a.N) * a.dpad + 4 * g0;
                if (w + 1 < w_end) px[rg] = a.wrow[(w + 1) * TM + rbase + 8 * rg + rl];
            }
            for (int cc = 0; cc < a.nch; cc++) {
                if (!first) TW(0, mbar_wait(&remp[q], eph));
                uint8_t* st = rring + (size_t)q * raw_bytes;
#pragma unroll
                for (int rg = 0; rg < 4; rg++)
#pragma unroll
                    for (int h = 0; h < 2; h++) cp_async16(st + off[2 * rg + h], src[rg] + cc * KC + 16 * h);
                cp_arrive_noinc(&rawf[q]);
                if (++q == a.Q) {
                    q = 0;
                    if (first) first = false; else eph ^= 1u;
                }
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp < MMA_WARP) {
        // ------------------------------------------------------------------ converters
        // thread = tile row = TMEM lane: read the row's raw chunk (8 conflict-free 16-B loads), store
        // hi = the raw value (the MMA reads its top 19 bits) and lo = x − trunc_tf32(x) into the A
        // slot's two 32-column halves with tcgen05.st; the first thread bulk-copies the chunk's B.
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const bool leader = t == NCOPY;
        const uint32_t tlane = (uint32_t)(quarter * 32) << 16;
        int q = 0, p = 0;
        uint32_t rph = 0, aph = 0;
        bool afirst = true;
        int4 dsc = leader && w_begin < w_end ? a.wdesc[w_begin] : make_int4(0, 0, 0, 0);
        for (int64_t w = w_begin; w < w_end; w++) {
            const int4 cur = dsc;
            if (leader && w + 1 < w_end) dsc = a.wdesc[w + 1];
            const uint32_t bb = (uint32_t)cur.w * KC * 4;
            for (int cc = 0; cc < a.nch; cc++) {
                TW(1, mbar_wait(&rawf[q], rph));
                const uint8_t* rs = rring + (size_t)q * raw_bytes + r * RPITCH;
                uint32_t x[KC];
#pragma unroll
                for (int g = 0; g < KC / 4; g++) {
                    const uint4 v = *(const uint4*)(rs + 16 * g);
                    x[4 * g] = v.x; x[4 * g + 1] = v.y; x[4 * g + 2] = v.z; x[4 * g + 3] = v.w;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&remp[q]);
                if (++q == a.Q) { q = 0; rph ^= 1u; }
                if (!afirst) TW(0, mbar_wait(&aemp[p], aph));
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (leader) {
                    uint8_t* bs = bring + (size_t)p * b_slot;
                    mbar_arrive_tx(&full[p], 2 * bb);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(bs)),
                        "l"(a.bsplit + 16 * (size_t)(uint32_t)cur.z + (size_t)cc * 2 * bb), "r"(2 * bb),
                        "r"(smem_u32(&full[p]))
                        : "memory");
                }
                uint32_t lo[KC];
#pragma unroll
                for (int e = 0; e < KC; e++)
                    lo[e] = __float_as_uint(__uint_as_float(x[e]) - __uint_as_float(x[e] & 0xFFFFE000u));
                const uint32_t ta = tmem + tlane + ACC_COLS + (uint32_t)(p * 2 * KC);
                tmem_st32(ta, x);
                tmem_st32(ta + KC, lo);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[p]);
                if (++p == NASLOT) {
                    p = 0;
                    if (afirst) afirst = false; else aph ^= 1u;
                }
            }
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer
        const uint32_t idesc0 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TM >> 4) << 24);
        int p = 0;
        uint32_t fph = 0;
        int k = 0;
        for (int64_t w = w_begin; w < w_end; w++, k++) {
            const int b = k & 1;
            const int np = a.wdesc[w].w;
            const uint32_t idesc = idesc0 | ((uint32_t)(np >> 3) << 17);
            const uint32_t blo = (uint32_t)np * KC * 4;                        // B_lo follows B_hi (np rows)
            if (k >= 2) TW(0, mbar_wait(&acce[b], ((k >> 1) - 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t dt = tmem + (uint32_t)(b * a.accw);
            for (int cc = 0; cc < a.nch; cc++) {
                TW(1, mbar_wait(&full[p], fph));
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (elect_one()) {
                    const uint32_t ta = tmem + ACC_COLS + (uint32_t)(p * 2 * KC);
                    const uint32_t bs = smem_u32(bring + (size_t)p * b_slot);
#pragma unroll
                    for (int ks = 0; ks < KC / 8; ks++) {
                        // D[:, 0:np) (+)= A_hi·B_hi;  += A_hi·B_lo;  += A_lo·B_hi   (A from TMEM)
                        const uint32_t ah = ta + 8 * ks, al = ta + KC + 8 * ks;
                        const uint64_t bh = umma_desc(bs + 256 * ks), bl = umma_desc(bs + blo + 256 * ks);
                        const uint32_t acc0 = (cc > 0 || ks > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
                            "r"(ah), "l"(bh), "r"(idesc), "r"(acc0));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(dt), "r"(ah),
                                     "l"(bl), "r"(idesc));
                        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(dt), "r"(al),
                                     "l"(bh), "r"(idesc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&aemp[p]))
                                 : "memory");
                }
                __syncwarp();
                if (++p == NASLOT) { p = 0; fph ^= 1u; }
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
        const int ew = warp - MMA_WARP - 1;           // 0..NEPI-1
        const int half = ew >> 2;                     // which alternate 16-column blocks this warp takes
        const int et = t - (NLOAD + 32);              // 0..32*NEPI-1 within the epilogue warps
        float* tbuf = tstage + (size_t)ew * 32 * TPITCH;   // this warp's 32x16 transpose buffer
        int k = 0, cur_q = -1, nb = 0;
        int64_t rb = 0;               // the query's table base (elements)
        int32_t rld = 8;              // its row pitch
        // next tile's descriptor, row id and row norm, loaded one tile ahead
        int4 ndsc = make_int4(0, 0, 0, 0);
        float nnx = 0.f;
        int32_t nxid = -1;
        auto prefetch = [&](int64_t w) {
            if (w < w_end) {
                ndsc = a.wdesc[w];
                nxid = a.wrow[w * TM + r];
                nnx = a.xnorm[nxid >= 0 ? (int64_t)nxid : a.N];
            }
        };
        prefetch(w_begin);
        for (int64_t w = w_begin; w < w_end; w++, k++) {
            const int b = k & 1;
            const int4 dsc = ndsc;
            const int32_t xid = nxid;
            const float nx = nnx;
            prefetch(w + 1);
            const int q = dsc.x, np = dsc.w;
            if (q != cur_q) {   // stage the query's ids and norms once per query (named barrier: epilogue only)
                const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
                const QHeader* hdr = (const QHeader*)slot;
                const int sq = hdr->err ? 0 : (int)hdr->s;
                nb = min(NCB, max(0, sq - a.cb * NCB));
                rld = a.pitch[q];
                rb = a.row_base[q];                 // elements
                asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");
                const uint2* qitems = (const uint2*)(slot + a.L.off_items);
                for (int j = et; j < NCB; j += 32 * NEPI) {
                    eyid[j] = j < nb ? (qitems[a.cb * NCB + j].x & FTI_VOCAB_MASK) : 0xFFFFFFFFu;
                    eny[j] = a.ny[(int64_t)q * NCB + j];
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");
                cur_q = q;
            }
            // rows of this warp: tile row 32*quarter + i; the table rows are contiguous
            float* wrow0 = a.table + rb + ((int64_t)dsc.y * TM + quarter * 32) * rld + a.cb * NCB;
            const unsigned valid = __ballot_sync(0xffffffffu, xid >= 0);     // rows that exist (a prefix)
            TW(0, mbar_wait(&accf[b], (k >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * a.accw);
            for (int c0 = 16 * half; c0 < np; c0 += 32) {
                uint32_t v[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15])
                    : "r"(tb + (uint32_t)c0));
                TW(1, asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"));
                if (c0 >= nb || valid == 0u) continue;
                const long long tc0 = clock64();
                // branch-free: the 16 columns' norms and ids as vectors, MUFU square root (relative
                // error ~2^-22, far inside the 1e-5 Flowtree bar), a select for shared ids
                float o[16];
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 ny4 = *(const float4*)(eny + c0 + i);
                    const uint4 id4 = *(const uint4*)(eyid + c0 + i);
                    const float nyv[4] = {ny4.x, ny4.y, ny4.z, ny4.w};
                    const uint32_t idv[4] = {id4.x, id4.y, id4.z, id4.w};
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const float dot = __uint_as_float(v[i + u]);
                        const float d2 = fmaxf(fmaf(-2.f, dot, nx + nyv[u]), 0.f);
                        float sq;
                        asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(d2));
                        o[i + u] = ((uint32_t)xid == idv[u]) ? 0.f : sq;
                    }
                }
                if (DBG) dbg[2] += (unsigned long long)(clock64() - tc0);
                if (c0 + 16 <= nb && (rld & 3) == 0) {
                    // transpose through shared memory: lane (8 rows x 4 granules per store) writes 16 B of
                    // a row, so each store instruction covers 8 rows x 64 contiguous bytes
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *(float4*)(tbuf + lane * TPITCH + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
                    __syncwarp();
                    const int ra = lane >> 2, gb = lane & 3;
#pragma unroll
                    for (int s8 = 0; s8 < 4; s8++) {
                        const int row = 8 * s8 + ra;
                        if ((valid >> row) & 1u)
                            *(float4*)(wrow0 + (int64_t)row * rld + c0 + 4 * gb) =
                                *(const float4*)(tbuf + row * TPITCH + 4 * gb);
                    }
                    __syncwarp();
                } else if (xid >= 0) {
#pragma unroll
                    for (int i = 0; i < 16; i++)
                        if (c0 + i < nb) wrow0[(int64_t)lane * rld + c0 + i] = o[i];
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(&acce[b]);
        }
    }
    if (DBG) {
        const unsigned long long tt = (unsigned long long)(clock64() - tstart);
        if (t == NCOPY) { atomicAdd(&g_dbg[14], dbg[1]); atomicAdd(&g_dbg[15], dbg[0]); atomicAdd(&g_dbg[11], tt); }
        if (t == 0) { atomicAdd(&g_dbg[13], (unsigned long long)(w_end - w_begin)); atomicAdd(&g_dbg[0], tt); atomicAdd(&g_dbg[1], dbg[0]); atomicAdd(&g_dbg[2], dbg[1]); atomicAdd(&g_dbg[12], 1ull); }
        if (t == NLOAD) { atomicAdd(&g_dbg[3], tt); atomicAdd(&g_dbg[4], dbg[0]); atomicAdd(&g_dbg[5], dbg[1]); }
        if (t == NLOAD + 32) { atomicAdd(&g_dbg[6], tt); atomicAdd(&g_dbg[7], dbg[0]); atomicAdd(&g_dbg[8], dbg[1]); atomicAdd(&g_dbg[9], dbg[2]); }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// Per column block: every query's MMA width N_q (its columns in this block rounded up to 16; 0 when
// it has none), the offset of its pre-split B chunks, and the work list's tile prefix (queries
// without columns get no tiles).  One CTA, block-wide scans over 1024-query slabs.  With `units`:
// adds the stage's algorithmic bytes Σ_q rows_q · (4 d [first block only] + 4 s_q,block), and in
// the next slot its algorithmic flops Σ_q 2 · rows_q · s_q,block · d.
__global__ void __launch_bounds__(1024) k_tile_plan(DistArgs a, int d, unsigned long long* units) {
    __shared__ int tmp_t[32], tmp_b[32];
    int64_t tacc = 0, bacc = 0;
    unsigned long long bytes = 0, flops = 0;
    for (int q0 = 0; q0 < a.nq; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        int np = 0, tiles = 0, nb = 0;
        int64_t r = 0;
        if (q < a.nq) {
            const QHeader* h = (const QHeader*)(a.qblock + (size_t)q * a.L.stride);
            const int sq = h->err ? 0 : (int)h->s;
            nb = min(NCB, max(0, sq - a.cb * NCB));
            np = nb > 0 ? max(16, (nb + 15) & ~15) : 0;
            r = a.rowcnt ? (int64_t)a.rowcnt[q] : a.rows_cap;
            tiles = np ? (int)((r + TM - 1) / TM) : 0;
        }
        const int bsz = a.nch * 2 * np * KC * 4 / 16;   // B bytes / 16
        int tt, bt;
        const int tex = fti_block_exclusive_sum(tiles, tmp_t, &tt);
        const int bex = fti_block_exclusive_sum(bsz, tmp_b, &bt);
        if (q < a.nq) {
            a.tile_base[q] = tacc + tex;
            a.qinfo[q] = make_uint2((uint32_t)(bacc + bex), (uint32_t)np);
            if (np) {
                bytes += (unsigned long long)r * ((a.cb == 0 ? 4ull * d : 0ull) + 4ull * nb);
                flops += 2ull * (unsigned long long)r * (unsigned long long)nb * (unsigned long long)d;
            }
        }
        tacc += tt;
        bacc += bt;
        __syncthreads();
    }
    if (threadIdx.x == 0) a.tile_base[a.nq] = tacc;
    if (units && bytes) atomicAdd(units, bytes);
    if (units && flops) atomicAdd(units + (FT_PROF_DIST_FLOPS - FTI_ST_DIST), flops);
}

// grid (nq, slices): the tiles' descriptors and row ids
__global__ void __launch_bounds__(TM) k_tiles(DistArgs a) {
    const int q = blockIdx.x;
    const uint2 qi = a.qinfo[q];
    if (qi.y == 0) return;
    const int64_t t0 = a.tile_base[q], t1 = a.tile_base[q + 1];
    const int64_t nrows = a.rowcnt ? (int64_t)a.rowcnt[q] : a.rows_cap;
    for (int64_t w = t0 + blockIdx.y; w < t1; w += gridDim.y) {
        const int64_t tile = w - t0;
        const int64_t row = tile * TM + threadIdx.x;
        int32_t xid = -1;
        if (row < nrows) xid = a.rows ? a.rows[(int64_t)q * a.rows_cap + row] : (int32_t)row;
        a.wrow[w * TM + threadIdx.x] = xid;
        if (threadIdx.x == 0) a.wdesc[w] = make_int4(q, (int)tile, (int)qi.x, (int)qi.y);
    }
}

// per query: the translated query points of column block cb split into TF32 hi/lo in the MMA
// core-matrix layout per K chunk, and their norms ||ỹ||^2
__global__ void __launch_bounds__(256) k_dist_prep(DistArgs a) {
    __shared__ uint32_t yid[NCB];
    const int q = blockIdx.x;
    const uint2 qi = a.qinfo[q];
    const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    const uint2* qitems = (const uint2*)(slot + a.L.off_items);
    const int s = hdr->err ? 0 : (int)hdr->s;
    const int nb = min(NCB, max(0, s - a.cb * NCB));
    const int np = (int)qi.y;
    for (int j = threadIdx.x; j < NCB; j += blockDim.x) {
        const uint32_t y = j < nb ? (qitems[a.cb * NCB + j].x & FTI_VOCAB_MASK) : 0xFFFFFFFFu;
        yid[j] = y;
        if (blockIdx.y == 0) a.ny[(int64_t)q * NCB + j] = j < nb ? a.xnorm[y] : 0.f;
    }
    __syncthreads();
    if (!np) return;
    const uint32_t b_bytes = (uint32_t)np * KC * 4;
    uint8_t* bq = (uint8_t*)a.bsplit + 16 * (size_t)qi.x;
    // CTA (query, K-chunk slice); thread per (chunk, row, 4-group)
    const int groups = a.nch * np * (KC / 4);
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < groups; e += gridDim.y * blockDim.x) {
        const int g = e % (KC / 4);
        const int j = (e / (KC / 4)) % np;
        const int cc = e / ((KC / 4) * np);
        const int64_t src = j < nb ? (int64_t)yid[j] : a.N;     // the zero row pads N_q
        const float4 v = *(const float4*)(a.Xc + src * a.dpad + cc * KC + 4 * g);
        uint8_t* st = bq + (size_t)cc * 2 * b_bytes;
        split_store(st, st + b_bytes, cm_off(j, 4 * g), v);
    }
}

// X̃ = X − μ, μ the FP64 mean of the points: one CTA per coordinate
__global__ void __launch_bounds__(256) k_center_mean(const float* __restrict__ X, int64_t N, int d,
                                                     double* __restrict__ mean) {
    __shared__ double red[256];
    const int k = blockIdx.x;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) acc += (double)X[i * d + k];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) mean[k] = red[0] / (double)N;
}

// one warp per row (N + 1 rows, the last all zero): X̃ rounded to FP32, padded, and ||X̃||^2 in FP64
__global__ void __launch_bounds__(256) k_center_rows(const float* __restrict__ X, int64_t N, int d, int dpad,
                                                     const double* __restrict__ mean, float* __restrict__ Xc,
                                                     float* __restrict__ xnorm) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i > N) return;
    double acc = 0.0;
    for (int k = lane; k < dpad; k += 32) {
        float v = 0.f;
        if (i < N && k < d) v = (float)((double)X[i * d + k] - mean[k]);
        Xc[i * dpad + k] = v;
        acc += (double)v * (double)v;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) xnorm[i] = (float)acc;
}

// one CTA per query: the candidates' vocabulary as a shared-memory bitmap (shared atomics), then
// per-word ranks (dense row ids in vocab order), the row list and the row count
__global__ void __launch_bounds__(1024) k_vocab(const uint32_t* __restrict__ doc_off, const uint2* __restrict__ items,
                                                const int64_t* __restrict__ cand, int64_t cand_ld, int64_t n_cand,
                                                int64_t n, int64_t nwords, uint2* __restrict__ map, int32_t* __restrict__ rows,
                                                int32_t* __restrict__ rowcnt, int64_t rows_cap) {
    extern __shared__ uint32_t sbits[];
    __shared__ int tmp[32];
    const int q = blockIdx.x;
    for (int64_t i = threadIdx.x; i < nwords; i += blockDim.x) sbits[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t c = warp; c < n_cand; c += nw) {
        const int64_t doc = cand[(int64_t)q * cand_ld + c];
        // a negative candidate (padding / another shard's doc) has no rows; an index >= n is
        // reported (NaN + FT_ERANGE) by the Flowtree kernels and contributes no rows here
        if (doc < 0 || doc >= n) continue;
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

// the index's translated operand, built once on first use
cudaError_t prepare_centered(ft_index* ix, cudaStream_t st) {
    if (ix->Xc) return cudaSuccess;
    const int dpad = (ix->d + KC - 1) / KC * KC;
    float* Xc = nullptr;
    float* xn = nullptr;
    double* mean = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&Xc, sizeof(float) * (size_t)(ix->N + 1) * dpad)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&xn, sizeof(float) * (size_t)(ix->N + 1))) != cudaSuccess) { cudaFree(Xc); return e; }
    if ((e = cudaMalloc(&mean, sizeof(double) * ix->d)) != cudaSuccess) { cudaFree(Xc); cudaFree(xn); return e; }
    k_center_mean<<<ix->d, 256, 0, st>>>(ix->X, ix->N, ix->d, mean);
    k_center_rows<<<(unsigned)((ix->N + 1 + 7) / 8), 256, 0, st>>>(ix->X, ix->N, ix->d, dpad, mean, Xc, xn);
    fti_count_launches(2);
    e = cudaStreamSynchronize(st);
    cudaFree(mean);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) { cudaFree(Xc); cudaFree(xn); return e; }
    ix->Xc = Xc;
    ix->xnorm = xn;
    ix->dpad = dpad;
    return cudaSuccess;
}

}  // namespace

cudaError_t fti_launch_dist_table(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                                  const int32_t* d_rows, const int32_t* d_rowcnt, int64_t rows_cap,
                                  const int64_t* d_row_base, const int32_t* d_pitch, float* d_table, cudaStream_t st) {
    if (nq <= 0 || rows_cap <= 0) return cudaSuccess;
    ft_index* ix = const_cast<ft_index*>(ds->ix);
    cudaError_t e;
    if ((e = prepare_centered(ix, st)) != cudaSuccess) return e;
    DistArgs a{};
    a.Xc = ix->Xc;
    a.xnorm = ix->xnorm;
    a.N = ix->N;
    a.dpad = ix->dpad;
    a.nch = ix->dpad / KC;
    a.qblock = d_qblock;
    a.L = L;
    a.nq = nq;
    a.rows = d_rows;
    a.rowcnt = d_rowcnt;
    a.rows_cap = rows_cap;
    a.row_base = d_row_base;
    a.pitch = d_pitch;
    a.table = d_table;
    const int ncb = (L.smax + NCB - 1) / NCB;
    const int np_max = std::min(NCB, L.smax);
    a.NPmax = std::max(16, ((np_max + 15) / 16) * 16);
    const int64_t tmax = (int64_t)nq * ((rows_cap + TM - 1) / TM);
    if ((e = ds->s_bsplit.reserve((size_t)nq * a.nch * 2 * a.NPmax * KC * 4)) != cudaSuccess) return e;
    if ((e = ds->s_ny.reserve((size_t)nq * NCB * 4)) != cudaSuccess) return e;
    if ((e = ds->s_tiles.reserve((size_t)(nq + 1) * 8)) != cudaSuccess) return e;
    if ((e = ds->s_qinfo.reserve((size_t)nq * 8)) != cudaSuccess) return e;
    if ((e = ds->s_wdesc.reserve((size_t)tmax * 16)) != cudaSuccess) return e;
    if ((e = ds->s_wrow.reserve((size_t)tmax * TM * 4)) != cudaSuccess) return e;
    a.bsplit = ds->s_bsplit.as<uint8_t>();
    a.ny = ds->s_ny.as<float>();
    a.tile_base = ds->s_tiles.as<int64_t>();
    a.qinfo = ds->s_qinfo.as<uint2>();
    a.wdesc = ds->s_wdesc.as<int4>();
    a.wrow = ds->s_wrow.as<int32_t>();
    // shared memory: Q raw slots, NASLOT B slots, epilogue staging, barriers
    const size_t raw_bytes = (size_t)TM * RPITCH;
    const size_t b_slot = 2 * (size_t)a.NPmax * KC * 4;
    const size_t fixed = 2 * NCB * 4 + NEPI * 32 * TPITCH * 4 + 512;
    a.accw = a.NPmax;
    a.naslot = std::min(MAXASLOT, (int)(TMEM_COLS - 2 * a.accw) / (2 * KC));
    if (a.naslot < 2) return cudaErrorInvalidConfiguration;
    const size_t budget = 224 * 1024 - fixed - (size_t)MAXASLOT * b_slot;
    const int Q = (int)std::min<size_t>(8, budget / raw_bytes);
    if (Q < 2) return cudaErrorInvalidConfiguration;
    a.Q = Q;
    const size_t smem = (size_t)Q * raw_bytes + (size_t)MAXASLOT * b_slot + fixed;
    const bool dbg = (fti_opt(FT_OPT_DEBUG) & FTI_DBG_DIST) != 0;
    auto kern = dbg ? k_dist_tc<true> : k_dist_tc<false>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    const unsigned slices = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (148 * 8 + nq - 1) / nq));
    for (int cb = 0; cb < ncb; cb++) {
        a.cb = cb;
        k_tile_plan<<<1, 1024, 0, st>>>(a, ix->d, ds->units_ptr(FTI_ST_DIST));
        k_tiles<<<dim3((unsigned)nq, slices), TM, 0, st>>>(a);
        k_dist_prep<<<dim3((unsigned)nq, (unsigned)std::min(a.nch, 8)), 256, 0, st>>>(a);
        kern<<<148, NTHREADS, smem, st>>>(a);
        fti_count_launches(4);
        if (dbg) {
            unsigned long long h[16];
            cudaStreamSynchronize(st);
            cudaMemcpyFromSymbol(h, g_dbg, sizeof(h));
            const double n = h[12] ? (double)h[12] * 1e3 : 1.0;
            fprintf(stderr, "dist dbg per CTA (kcyc): copy total %.1f wait_empty %.1f conv total %.1f wait_raw %.1f wait_aslot %.1f | mma total %.1f wait_acce %.1f wait_full %.1f | epi total %.1f wait_accf %.1f tmem_ld %.1f math %.1f | tiles %.1f\n",
                    h[0] / n, h[1] / n, h[11] / n, h[14] / n, h[15] / n, h[3] / n, h[4] / n, h[5] / n, h[6] / n, h[7] / n, h[8] / n, h[9] / n, (double)h[13] / (n / 1e3));
            memset(h, 0, sizeof(h));
            cudaMemcpyToSymbol(g_dbg, h, sizeof(h));
        }
    }
    return cudaGetLastError();
}

cudaError_t fti_launch_vocab_map(const ft_dataset* ds, int32_t nq, const int64_t* d_cand, int64_t cand_ld,
                                 int64_t n_cand, uint2* d_map, int32_t* d_rows, int32_t* d_rowcnt, int64_t rows_cap,
                                 cudaStream_t st) {
    if (nq <= 0) return cudaSuccess;
    const int64_t nwords = (ds->ix->N + 31) / 32;
    const size_t smem = (size_t)nwords * 4;
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;   // N > 1.6M: not supported by the bitmap
    cudaError_t e = cudaFuncSetAttribute(k_vocab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_vocab<<<nq, 1024, smem, st>>>(ds->doc_off, ds->items, d_cand, cand_ld, n_cand, ds->n, nwords, d_map, d_rows,
                                    d_rowcnt, rows_cap);
    fti_count_launches(1);
    return cudaGetLastError();
}
