// ft_dist.cu — a5: distance table D[c][j] = ||x_{v_c} − y_j||_2 between the candidate vocabulary and
// the query support, read by the Flowtree kernels to price the flow (PAPER.md:150,
// "Σ f(x, x')·||x − x'||"; Lemma 1's O(d) per matched pair).
//
// The table is a dense contraction, so it runs on the 5th-generation tensor cores (tcgen05), in
// EXACT integer arithmetic:
//   * every point is translated by the FP64 mean of the ground set and quantised once per index to
//     24-bit fixed point v = rint((x − mean)·2^e), e the largest exponent with max|v| ≤ 2^23 − 2^16,
//     and split into three balanced signed bytes v = a0 + 2^8·a1 + 2^16·a2 (a_i ∈ [−128, 127]);
//   * ||v_x − v_y||² = ||v_x||² + ||v_y||² − 2·v_x·v_y with v_x·v_y = Σ_t 2^{8t} T_t, the five "tiers"
//     T_t = Σ_{p+q=t} A_p·B_q computed by nine tcgen05.mma.kind::i8 products accumulated in s32 TMEM
//     (|T_t| ≤ 3·d·2^14 < 2^31), combined in int64 by the epilogue: d² of the quantised points is
//     exact, so identical coordinates (the same id, or duplicates under distinct ids) give exactly
//     0 and near pairs suffer no Gram-form cancellation;
//   * D = sqrt((float)d²)·2^-e in FP32.  |D − ||x − y||| ≤ ||δ_x − δ_y|| ≤ sqrt(d)·2^-e (each
//     coordinate rounds by ≤ 2^-(e+1)), plus ≈2^-22 relative from the FP32 conversion and the
//     MUFU square root
//     (DESIGN.md §7).
//
// k_dist_i8 is persistent (one CTA per SM) and warp specialised over a device-built list of
// (query, 96-column group, 128-row tile) work items:
//   * 2 copy warps cp.async the tile's 128 gathered rows, 64 coordinates × 3 limbs (192 B) per K
//     stage, into a 4-deep ring in the canonical no-swizzle K-major core-matrix layout, arriving on
//     the stage's mbarrier with cp.async.mbarrier.arrive.noinc;
//   * 1 MMA warp: when the (query, group) changes it bulk-copies the group's pre-arranged B (the
//     query points' limbs, each 48-column block's three limbs stacked along N) into shared memory;
//     per K step an elected lane issues, per block, three tcgen05.mma.kind::i8 (M = 128,
//     N = 3·48, A and B from shared memory): A_p·[B_0 | B_1 | B_2] into TMEM columns starting at
//     p·48, so the product A_p·B_q lands on tier p + q and each A limb is read once per K step (the
//     first K step splits them so every tier is initialised once).  Accumulators: two TMEM slots
//     of 5 tiers × 48 s32 columns, so a one-block item's epilogue overlaps the next item's MMAs;
//   * 8 epilogue warps (2 per TMEM lane quarter, alternating 8-column chunks, the next chunk's
//     loads in flight): tcgen05.ld the five tiers, combine them exactly in int64 (wide
//     multiply-adds), write each row's 8 distances as two 16-byte stores.
// k_tile_plan / k_tiles build the work list, k_dist_prep the per-(query, group) B operand.
//
// Candidate vocabulary for the prefiltered pipeline: k_vocab marks every vocab id of the query's
// m candidates in a shared-memory bitmap and turns it into dense row ids and the row list; the
// host places each query's rows compactly (ft_api.cu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ft_device.cuh"

namespace {

constexpr int TM = 128;                  // rows per work item = UMMA M
constexpr int NL = 3;                    // int8 limbs per coordinate
constexpr int NTIER = 5;                 // tiers t = p + q of the limb products
constexpr int KS = 64;                   // K bytes (= coordinates) per stage and limb
constexpr int ROWB = NL * KS;            // global row bytes per stage: [limb][64]
constexpr int STAGE_LIMB = TM * KS;      // 8 KB
constexpr int STAGE_BYTES = NL * STAGE_LIMB;
constexpr int NSTAGE_MAX = 8;
constexpr int SBO_A = (KS / 16) * 128;   // A stage: bytes between 8-row core-matrix groups
#ifndef FTD_NBLK
#define FTD_NBLK 48
#endif
constexpr int NBLK = FTD_NBLK;           // accumulator columns per block (5 tiers × NBLK per slot)
#ifndef FTD_NGRP
#define FTD_NGRP 96
#endif
constexpr int NGRP = FTD_NGRP;           // query columns per work item
constexpr int NBMAX = NGRP / NBLK;       // blocks per work item
constexpr int NSLOT = 512 / (5 * NBLK);  // TMEM accumulator slots (2 for 48 columns, 3 for 32)
constexpr int SLOT_COLS = 5 * NBLK;      // TMEM columns per accumulator slot
#ifndef FTD_NCOPY
#define FTD_NCOPY 64
#endif
constexpr int NCOPY = FTD_NCOPY;         // copy threads (warps 0 .. NCOPY/32 − 1)
constexpr int MMA_WARP = NCOPY / 32;     // warp 2
#ifndef FTD_NEPI
#define FTD_NEPI 8
#endif
#ifndef FTD_ABL
#define FTD_ABL 0          // ablation (timing experiments only; wrong tables): 1 no copies, 2 no MMAs,
                           // 4 no epilogue work, 8 no table stores
#endif
#ifndef FTD_REV
#define FTD_REV 0          // block-outer order: the item's narrowest (last) block first
#endif
#ifndef FTD_EDB
#define FTD_EDB 1          // epilogue: the next chunk's TMEM loads in flight while one is combined
#endif
constexpr int NEPI = FTD_NEPI;           // epilogue warps (a multiple of 4: NEPI / 4 per TMEM lane quarter)
constexpr int NPART = NEPI / 4;          // epilogue warps per quarter, on interleaved 8-column chunks
constexpr int NTHREADS = NCOPY + 32 + 32 * NEPI;
constexpr uint32_t TMEM_COLS = 512;
constexpr int QMAX_ABS = (1 << 23) - (1 << 16);   // |v| bound: the top balanced limb stays in [−128, 127]

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one elected lane of a converged warp; ptxas then knows the tcgen05.mma operands are uniform
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

// shared-memory matrix descriptor, K-major, SWIZZLE_NONE: start >> 4 [0,14), LBO >> 4 [16,30)
// (K-adjacent core matrices, 128 B apart), SBO >> 4 [32,46) (8-row groups), version 1 [46,48)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46);
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
#ifndef FTD_L2POL
#define FTD_L2POL 0        // 1: X̃q rows evict_last, table stores evict_first in L2
#endif
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
#ifndef FTD_CPCA
#define FTD_CPCA 0         // 1: cp.async.ca (through L1) instead of .cg
#endif
#ifndef FTD_KOUTER
#define FTD_KOUTER 0       // 1: K-outer MMA order with the deepest ring that fits (test option)
#endif
#ifndef FTD_LDGCP
#define FTD_LDGCP 0        // 1: copy warps load 32-byte sectors into registers and st.shared them
#endif
#ifndef FTD_ST256
#define FTD_ST256 1        // one 256-bit store per row chunk of 8 distances (one full sector; 0: two 16-byte stores)
#endif
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    if (FTD_CPCA)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void st_f8(float* p, const float (&o)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                 "f"(o[3]), "f"(o[4]), "f"(o[5]), "f"(o[6]), "f"(o[7])
                 : "memory");
}
__device__ __forceinline__ void cp_async16_pol(uint32_t dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_f1(float* p, float v, uint64_t pol) {
    if (FTD_L2POL)
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
    else
        *p = v;
}
__device__ __forceinline__ void st_f4(float* p, float4 v, uint64_t pol) {
    if (FTD_L2POL)
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
                     "f"(v.z), "f"(v.w), "l"(pol)
                     : "memory");
    else
        *(float4*)p = v;
}
// arrive on `bar` once all of this thread's prior cp.async copies have landed (count not incremented)
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// FP32 value of a non-negative integer < 2^57 (relative error < 2^-23) on the FMA/ALU pipes: three
// 23-bit chunks, each converted exactly by the 2^23 magic-number add.  (I2F.S64 runs on the XU pipe,
// which the epilogue's conversions had saturated — 97% XU, ncu.)
__device__ __forceinline__ float u57_to_f32(unsigned long long u) {
    const uint32_t c0 = (uint32_t)u & 0x7FFFFFu, c1 = (uint32_t)(u >> 23) & 0x7FFFFFu, c2 = (uint32_t)(u >> 46);
    const float f0 = __int_as_float(0x4B000000 | c0) - 8388608.f;
    const float f1 = __int_as_float(0x4B000000 | c1) - 8388608.f;
    const float f2 = __int_as_float(0x4B000000 | c2) - 8388608.f;
    return fmaf(f2, 70368744177664.f, fmaf(f1, 8388608.f, f0));   // f2·2^46 + f1·2^23 + f0
}

// byte offset of (row r, K byte kb) in a K-major no-swizzle core-matrix tile whose 8-row groups are
// `sbo` bytes apart
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int kb, int sbo) {
    return (uint32_t)((r >> 3) * sbo + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15));
}

// query columns of group g (≤ 96) and their MMA width (rounded up to 16)
__device__ __forceinline__ int group_cols(int s, int g) { return min(NGRP, s - NGRP * g); }

struct DistArgs {
    const int8_t* Xq;           // [(N+1)][nks][3][64] quantised limbs, zero row N
    const long long* xnq;       // [N+1] Σ v²
    int64_t N;
    int nks;                    // K stages (64 coordinates each)
    int kpad;                   // 64 · nks
    float scale;                // 2^-e
    const uint8_t* qblock;
    QueryLayout L;
    int nq;
    int8_t* bq;                 // B operands, query q group g at byte 16·(qinfo[q].x) + g·3·96·kpad
    long long* ny;              // [nq][ny_ld] Σ v² of the query points
    int ny_ld;
    uint2* qinfo;               // [nq] {B offset / 16 bytes, s_q (0: invalid query)}
    int4* wdesc;                // [T] {q, tile, g | group columns << 16, B offset / 16 of the group}
    int32_t* wrow;              // [T][TM] vocab id of each row of the tile, −1 past the query's rows
    int64_t* tile_base;         // [nq + 1] exclusive prefix of work items per query (T = tile_base[nq])
    const int32_t* rows;        // [nq][rows_cap] or null (row = vocab)
    const int32_t* rowcnt;      // [nq] or null (rows_cap)
    int64_t rows_cap;
    const int64_t* row_base;    // [nq] ELEMENT offset of each query's table
    const int32_t* pitch;       // [nq] per-query row pitch (floats)
    float* table;
    int kz;                     // K bytes from kz on are zero padding in every row (round_up(d, 16))
    int nstage;                 // A ring depth
    int blk_outer;              // the ring holds a tile's whole K range (nstage == nks)
    // tile-major order (exhaustive tables: every query's rows are all vocab ids): item
    // tile·GQ + gbase[q] + g, so consecutive items share their A tile and its copy is skipped
    int tmajor;
    int32_t* gbase;             // [nq + 1] exclusive prefix of the queries' column groups (GQ = gbase[nq])
};

__device__ unsigned long long g_dbg[16];
// DBG: clock64 totals of each role's waits (FT_OPT_DEBUG bit 1)
#define TW(slot, stmt)                                         \
    do {                                                       \
        if (DBG) {                                             \
            const long long t0_ = clock64();                   \
            stmt;                                              \
            dbgc[slot] += (unsigned long long)(clock64() - t0_); \
        } else {                                               \
            stmt;                                              \
        }                                                      \
    } while (0)

template <bool DBG>
// NTHREADS threads, one CTA per SM; ≤ 3 warps per SM sub-partition leave 168 registers a thread
#if (FTD_NCOPY / 32 + 1 + FTD_NEPI) <= 12
#define FTD_KATTR __maxnreg__(168)
#else
#define FTD_KATTR __launch_bounds__(NTHREADS, 1)
#endif
__global__ void FTD_KATTR k_dist_i8(DistArgs a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int NSTAGE = a.nstage;
    unsigned long long dbgc[4] = {0, 0, 0, 0};
    const long long tstart = DBG ? clock64() : 0;
    // shared memory: A ring [NSTAGE][3 limbs][128 rows × 64 B] | B [3 limbs][≤ 96 rows × kpad] |
    // epilogue ny [96] | barriers
    uint8_t* aring = sm;
    uint8_t* bsm = sm + (size_t)NSTAGE * STAGE_BYTES;
    const uint32_t b_limb_max = (uint32_t)NGRP * a.kpad;
    long long* eny = (long long*)(bsm + (size_t)NL * b_limb_max);
    uint64_t* bars = (uint64_t*)(eny + NGRP);
    uint64_t* full = bars;                   // [NSTAGE] A stage landed (copy threads, noinc)
    uint64_t* empty = full + NSTAGE_MAX;     // [NSTAGE] A stage consumed (MMA commit)
    uint64_t* accf = empty + NSTAGE_MAX;     // [NSLOT] slot accumulated (MMA commit)
    uint64_t* acce = accf + NSLOT;           // [NSLOT] slot drained (epilogue warps)
    uint64_t* bfull = acce + NSLOT;          // B landed (complete_tx)
    uint64_t* bdone = bfull + 1;             // MMAs reading the old B finished (commit)
    uint32_t* tmem_slot = (uint32_t*)(bdone + 1);
    const uint32_t sbo_b = (uint32_t)a.kpad * 8;   // B: (kpad / 16) core matrices × 128 B per 8-row group

    const int64_t T = a.tile_base[a.nq];
    const int64_t w_begin = T * blockIdx.x / gridDim.x, w_end = T * (blockIdx.x + 1) / gridDim.x;
    if (t == 0) {
        for (int s = 0; s < NSTAGE; s++) { mbar_init(&full[s], NCOPY); mbar_init(&empty[s], 1); }
        for (int b = 0; b < NSLOT; b++) { mbar_init(&accf[b], 1); mbar_init(&acce[b], NEPI); }
        mbar_init(bfull, 1);
        mbar_init(bdone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // with the ring slot of K stage c fixed (nstage == nks), the all-zero K granules of the padding
    // (K ≥ round_up(d, 16)) are zeroed once here and never copied
    const bool kfixed = NSTAGE == a.nks;
    if (kfixed && a.kz < a.kpad) {
        const int gz0 = a.kz / 16, gz1 = a.kpad / 16;   // dead 16-byte K granules [gz0, gz1)
        const int per = (gz1 - gz0) * TM * NL;
        for (int e = t; e < per; e += blockDim.x) {
            const int g = gz0 + e % (gz1 - gz0), rest = e / (gz1 - gz0);
            const int r = rest % TM, p = rest / TM;
            const int c = g / (KS / 16), kb = (g % (KS / 16)) * 16;
            *(uint4*)(aring + (size_t)c * STAGE_BYTES + p * STAGE_LIMB + cm_off(r, kb, SBO_A)) = make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (FTD_LDGCP && t < NCOPY) {
        // ------------------------------------------------------------------ copy threads (LDG path)
        // 32-byte register loads (each lane one full sector: 16-byte cp.async requests fetch every
        // sector twice) stored to the ring with st.shared, then a proxy fence and an arrive.  Warp
        // cw fills rows 64 cw .. +63; per stage it issues 12 load slots over 4 pairs of 8-row
        // groups (3 per pair: units 0-3 of each group, then units 4-5 of both), in two halves of 6
        // slots that are double buffered in registers.  Unit k of a row = limb k / 2, 32-byte half
        // k % 2 of the stage's 64 coordinates.
        static_assert(!FTD_LDGCP || NCOPY == 64, "LDG copy path: two copy warps");
        const int cw = warp;
        const uint32_t abase = smem_u32(aring);
        const size_t rstride = (size_t)a.nks * ROWB;
        // slot sl (pair pp = sl / 3, kind = sl % 3) of this lane: its 8-row group selector, unit k
        auto slot_g = [&](int sl) { return sl % 3 == 2 ? (lane >> 4) : sl % 3; };
        auto slot_k = [&](int sl) { return sl % 3 == 2 ? 4 + ((lane >> 3) & 1) : (lane >> 3); };
        auto slot_dof = [&](int sl) {
            const int k = slot_k(sl);
            const int r = 8 * (2 * (4 * cw + sl / 3) + slot_g(sl)) + (lane & 7);
            return (uint32_t)((k >> 1) * STAGE_LIMB) + cm_off(r, 32 * (k & 1), SBO_A);
        };
        auto rowid = [&](int64_t w, int j) {   // row id j of the lane in item w (−1 → zero row)
            const int pp = j >> 1, gsel = j & 1;
            const int32_t x = a.wrow[w * TM + 8 * (2 * (4 * cw + pp) + gsel) + (lane & 7)];
            return x >= 0 ? x : (int32_t)a.N;
        };
        int32_t px[8];
        if (w_begin < w_end)
#pragma unroll
            for (int j = 0; j < 8; j++) px[j] = rowid(w_begin, j);
        uint32_t ra[6][8], rb[6][8];
        auto ld8 = [&](uint32_t (&r)[8], const int8_t* g) {
            if (!(FTD_ABL & 1))
                asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                               "=r"(r[7])
                             : "l"(g));
        };
        auto st8 = [&](uint32_t dst, const uint32_t (&r)[8]) {
            if (!(FTD_ABL & 1)) {
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                             "r"(r[3])
                             : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 128u), "r"(r[4]), "r"(r[5]),
                             "r"(r[6]), "r"(r[7])
                             : "memory");
            }
        };
        // half hf of stage c of the item whose row ids are px
        auto load_half = [&](uint32_t (&r)[6][8], const int32_t (&rows)[8], int c, int hf) {
#pragma unroll
            for (int u = 0; u < 6; u++) {
                const int sl = 6 * hf + u;
                const int32_t x = rows[2 * (sl / 3) + (sl % 3 == 2 ? 0 : sl % 3)];
                const int32_t x1 = rows[2 * (sl / 3) + 1];
                const int32_t xr = (sl % 3 == 2 && (lane >> 4)) ? x1 : x;
                ld8(r[u], a.Xq + (size_t)xr * rstride + (size_t)c * ROWB + 32 * slot_k(sl));
            }
        };
        auto store_half = [&](const uint32_t (&r)[6][8], uint32_t st, int hf) {
#pragma unroll
            for (int u = 0; u < 6; u++) st8(st + slot_dof(6 * hf + u), r[u]);
        };
        int s = 0;
        uint32_t eph = 0;
        bool first = true;
        if (w_begin < w_end) load_half(ra, px, 0, 0);
        for (int64_t w = w_begin; w < w_end; w++) {
            int32_t pn[8];
            const bool more = w + 1 < w_end;
            if (more)
#pragma unroll
                for (int j = 0; j < 8; j++) pn[j] = rowid(w + 1, j);
            for (int c = 0; c < a.nks; c++) {
                load_half(rb, px, c, 1);
                if (!first) TW(0, mbar_wait(&empty[s], eph));
                const uint32_t st = abase + (uint32_t)s * STAGE_BYTES;
                store_half(ra, st, 0);
                if (c + 1 < a.nks) load_half(ra, px, c + 1, 0);
                else if (more) load_half(ra, pn, 0, 0);
                store_half(rb, st, 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&full[s]);
                if (++s == NSTAGE) {
                    s = 0;
                    if (first) first = false; else eph ^= 1u;
                }
            }
            if (more)
#pragma unroll
                for (int j = 0; j < 8; j++) px[j] = pn[j];
        }
    } else if (t < NCOPY) {
        // ------------------------------------------------------------------ copy threads
        // lane → (row & 7, 16-byte granule): one cp.async instruction per limb moves 8 rows × 64
        // contiguous bytes (full sectors); warp cw fills rows 64 cw .. +63 of every stage
        constexpr int NCW = NCOPY / 32, RG = (TM / 8 + NCW - 1) / NCW;   // 8-row groups per copy warp
        const int rl = lane & 7, gq = lane >> 3;
        uint32_t doff[RG];
#pragma unroll
        for (int rg = 0; rg < RG; rg++) doff[rg] = cm_off((warp + NCW * rg) * 8 + rl, 16 * gq, SBO_A);
        const uint32_t abase = smem_u32(aring);
        const size_t rstride = (size_t)a.nks * ROWB;
        auto grp_ok = [&](int rg) { return warp + NCW * rg < TM / 8; };
        int32_t px[RG];
#pragma unroll
        for (int rg = 0; rg < RG; rg++)
            px[rg] = (w_begin < w_end && grp_ok(rg)) ? a.wrow[w_begin * TM + (warp + NCW * rg) * 8 + rl] : -1;
        int s = 0;
        uint32_t eph = 0;
        bool first = true;
        const uint64_t pol = FTD_L2POL ? l2_policy_last() : 0ull;
        int prev_tile = -1;
        for (int64_t w = w_begin; w < w_end; w++) {
            const int8_t* src[RG];
#pragma unroll
            for (int rg = 0; rg < RG; rg++) {
                src[rg] = a.Xq + (px[rg] >= 0 ? (int64_t)px[rg] : a.N) * rstride + 16 * gq;
                if (w + 1 < w_end && grp_ok(rg)) px[rg] = a.wrow[(w + 1) * TM + (warp + NCW * rg) * 8 + rl];
            }
            // tile-major order: the ring still holds this tile (every stage keeps its slot)
            const int tile = a.tmajor ? a.wdesc[w].y : -1;
            const bool reuse = kfixed && a.tmajor && tile == prev_tile;
            prev_tile = tile;
            for (int c = 0; c < a.nks; c++) {
                if (!first) TW(0, mbar_wait(&empty[s], eph));
                const uint32_t st = abase + (uint32_t)s * STAGE_BYTES;
                const bool live = !reuse && (!kfixed || KS * c + 16 * gq < a.kz);   // not an all-zero padding granule
#pragma unroll
                for (int p = 0; p < NL; p++)
#pragma unroll
                    for (int rg = 0; rg < RG; rg++)
                        if (grp_ok(rg) && live && !(FTD_ABL & 1)) {
                            if (FTD_L2POL) cp_async16_pol(st + p * STAGE_LIMB + doff[rg], src[rg] + (size_t)c * ROWB + p * KS, pol);
                            else cp_async16(st + p * STAGE_LIMB + doff[rg], src[rg] + (size_t)c * ROWB + p * KS);
                        }
                cp_arrive_noinc(&full[s]);
                if (++s == NSTAGE) {
                    s = 0;
                    if (first) first = false; else eph ^= 1u;
                }
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer
        // idesc: s32 accumulator [4,6) = 2, signed A [7,10) = 1, signed B [10,13) = 1, K-major A/B,
        // N >> 3 at [17,23), M >> 4 at [24,29)
        const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TM >> 4) << 24);
        const uint32_t abase = smem_u32(aring), bbase = smem_u32(bsm);
        int s = 0;
        uint32_t fph = 0, bph = 0, dph = 0;
        int64_t kb = 0;            // accumulator blocks issued so far (slot = kb & 1)
        int64_t it0 = 0;           // ring stages consumed so far (block-outer order)
        int cur_q = -1, cur_g = -1;
        int4 ndsc = w_begin < w_end ? a.wdesc[w_begin] : make_int4(0, 0, 0, 0);
        for (int64_t w = w_begin; w < w_end; w++) {
            const int4 dsc = ndsc;                     // descriptors are loaded one item ahead
            if (w + 1 < w_end) ndsc = a.wdesc[w + 1];
            const int q = dsc.x, g = dsc.z & 0xFFFF;
            const int cols = dsc.z >> 16;
            const int npad = (cols + 15) & ~15;
            const int nb = (npad + NBLK - 1) / NBLK;
            auto nw = [&](int b) { return min(NBLK, npad - NBLK * b); };   // block b's width
            if (q != cur_q || g != cur_g) {
                // reload B once the MMAs reading the previous one have completed
                if (cur_q >= 0) {
                    if (elect_one()) umma_commit(bdone);
                    __syncwarp();
                    TW(2, mbar_wait(bdone, dph));
                    dph ^= 1u;
                }
                const uint32_t bytes = (uint32_t)NL * npad * a.kpad;
                if (lane == 0) {
                    mbar_arrive_tx(bfull, bytes);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            bbase),
                        "l"(a.bq + 16 * (size_t)(uint32_t)dsc.w), "r"(bytes), "r"(smem_u32(bfull))
                        : "memory");
                }
                __syncwarp();
                TW(2, mbar_wait(bfull, bph));
                bph ^= 1u;
                cur_q = q;
                cur_g = g;
            }
            // block b's B region holds its three limbs stacked along N: rows q·nw[b] + j
            // block b's B region follows the earlier blocks' 3·NBLK rows
            auto breg = [&](int b) { return bbase + (uint32_t)(3 * NBLK * b / 8) * sbo_b; };
            // one block's MMAs over K stages [c0, c1): A_p · [B_0 | B_1 | B_2] (N = 3·nb) into columns
            // p·nb .. — the product A_p·B_q lands on tier p + q's columns (p + q)·nb, so the nine limb
            // products take three MMAs and every A limb is read once per K step per block
            auto issue = [&](int b, uint32_t dcol, int c, uint32_t st) {
                const uint32_t n = (uint32_t)nw(b);
#pragma unroll
                for (int ks = 0; ks < KS / 32; ks++) {
                    const uint32_t kbyte = (uint32_t)(c * KS + ks * 32);
                    const uint32_t bk = breg(b) + (kbyte >> 4) * 128;
                    auto mma = [&](int pl, int q0, int nq, uint32_t acc) {
                        const uint64_t ad = umma_desc(st + pl * STAGE_LIMB + ks * 256, SBO_A);
                        const uint64_t bd = umma_desc(bk + (uint32_t)(q0 * n / 8) * sbo_b, sbo_b);
                        const uint32_t idesc = idesc0 | ((uint32_t)(nq * n >> 3) << 17);
                        if (!(FTD_ABL & 2)) asm volatile(
                            "{\n\t.reg .pred pr;\n\tsetp.ne.b32 pr, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pr;\n\t}" ::"r"(
                                dcol + (uint32_t)(pl + q0) * n),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    };
                    if (c == 0 && ks == 0) {
                        // first K step: initialise each tier exactly once
                        mma(0, 0, 3, 0u);              // tiers 0, 1, 2
                        mma(1, 0, 2, 1u);              // tiers 1, 2
                        mma(1, 2, 1, 0u);              // tier 3
                        mma(2, 0, 1, 1u);              // tier 2
                        mma(2, 1, 1, 1u);              // tier 3
                        mma(2, 2, 1, 0u);              // tier 4
                    } else {
                        mma(0, 0, 3, 1u);
                        mma(1, 0, 3, 1u);
                        mma(2, 0, 3, 1u);
                    }
                }
            };
            auto acquire = [&](int64_t k) {           // the slot of the k-th block, once drained
                const int sl = (int)(k % NSLOT);
                if (k >= NSLOT) TW(1, mbar_wait(&acce[sl], (uint32_t)((k / NSLOT - 1) & 1)));
                asm volatile("tcgen05.fence::after_thread_sync;");
                return tmem + (uint32_t)sl * SLOT_COLS;
            };
            if (a.blk_outer) {
                // the ring holds the tile's whole K range (stage = K step): block-outer order, so
                // block 0's accumulator is committed (and drained by the epilogue) while block 1
                // computes; a stage is released after the last block has read it
                // (the ring may be deeper than a tile: stage c of the item is ring slot
                // (it0 + c) mod NSTAGE, so the next item's first stages load while this one computes)
                for (int i = 0; i < nb; i++) {
                    const int b = FTD_REV ? nb - 1 - i : i;    // block i of the item's sequence
                    const uint32_t dcol = acquire(kb + i);
                    int sc = (int)(it0 % NSTAGE);
                    uint32_t ph = (uint32_t)((it0 / NSTAGE) & 1);
                    for (int c = 0; c < a.nks; c++) {
                        if (i == 0) {
                            TW(0, mbar_wait(&full[sc], ph));
                            asm volatile("tcgen05.fence::after_thread_sync;");
                        }
                        if (elect_one()) {
                            issue(b, dcol, c, abase + (uint32_t)sc * STAGE_BYTES);
                            if (i == nb - 1) umma_commit(&empty[sc]);
                        }
                        __syncwarp();
                        if (++sc == NSTAGE) { sc = 0; ph ^= 1u; }
                    }
                    if (elect_one()) umma_commit(&accf[(int)((kb + i) % NSLOT)]);
                    __syncwarp();
                }
                it0 += a.nks;
            } else {
                uint32_t dcol[NBMAX];
                for (int b = 0; b < nb; b++) dcol[b] = acquire(kb + b);
                for (int c = 0; c < a.nks; c++) {
                    TW(0, mbar_wait(&full[s], fph));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (elect_one()) {
                        for (int b = 0; b < nb; b++) issue(b, dcol[b], c, abase + (uint32_t)s * STAGE_BYTES);
                        umma_commit(&empty[s]);
                    }
                    __syncwarp();
                    if (++s == NSTAGE) { s = 0; fph ^= 1u; }
                }
                for (int b = 0; b < nb; b++) {
                    if (elect_one()) umma_commit(&accf[(int)((kb + b) % NSLOT)]);
                    __syncwarp();
                }
            }
            kb += nb;
        }
    } else {
        // ------------------------------------------------------------------ epilogue
        const int quarter = warp & 3;                 // TMEM lanes 32·quarter .. +31 (hardware rule)
        const int part = (warp - MMA_WARP - 1) >> 2;  // which interleaved 8-column chunks this warp takes
        const int et = t - (NCOPY + 32);              // 0 .. 32·NEPI − 1
        const int r = quarter * 32 + lane;            // tile row = TMEM lane
        int64_t kb = 0;
        int cur_q = -1, cur_g = -1;
        const uint64_t wpol = FTD_L2POL ? l2_policy_first() : 0ull;
        // per item: descriptor and row id loaded two items ahead, then (depending on them) the row
        // norm and the table placement one item ahead, so no load's latency is exposed
        int4 adsc = make_int4(0, 0, 0, 0), ndsc = make_int4(0, 0, 0, 0);
        int32_t axid = -1, nxid = -1, npitch = 8;
        long long nnx = 0;
        int64_t nrb = 0;
        auto stage_a = [&](int64_t w) {
            if (w < w_end) {
                adsc = a.wdesc[w];
                axid = a.wrow[w * TM + r];
            }
        };
        auto stage_b = [&](int64_t w) {
            if (w < w_end) {
                ndsc = adsc;
                nxid = axid;
                nnx = nxid >= 0 ? a.xnq[nxid] : 0ll;
                npitch = a.pitch[ndsc.x];
                nrb = a.row_base[ndsc.x];
            }
        };
        stage_a(w_begin);
        stage_b(w_begin);
        stage_a(w_begin + 1);
        for (int64_t w = w_begin; w < w_end; w++) {
            const int4 dsc = ndsc;
            const int32_t xid = nxid;
            const long long nx = nnx;
            const int pitch = npitch;
            const int64_t rbase = nrb;
            stage_b(w + 1);
            stage_a(w + 2);
            const int q = dsc.x, tile = dsc.y, g = dsc.z & 0xFFFF;
            const int cols = dsc.z >> 16;
            const int npad = (cols + 15) & ~15;
            const int nb = (npad + NBLK - 1) / NBLK;
            if (q != cur_q || g != cur_g) {   // the group's ||ỹ||² (named barrier: epilogue warps only)
                asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");
                for (int j = et; j < NGRP; j += 32 * NEPI)
                    eny[j] = j < cols ? a.ny[(int64_t)q * a.ny_ld + NGRP * g + j] : 0ll;
                asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");
                cur_q = q;
                cur_g = g;
            }
            float* trow = a.table + rbase + ((int64_t)tile * TM + r) * pitch + NGRP * g;
            for (int i = 0; i < nb; i++, kb++) {
                const int b = (FTD_REV && a.blk_outer) ? nb - 1 - i : i;
                const int sl = (int)(kb % NSLOT);
                const int nwb = min(NBLK, npad - NBLK * b);   // tier t at columns t·nwb ..
                TW(0, mbar_wait(&accf[sl], (uint32_t)((kb / NSLOT) & 1)));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)sl * SLOT_COLS;
                // chunks of 8 columns, alternating between the quarter's two warps; the next chunk's
                // five tier loads are in flight while this chunk is combined (two register sets)
                const bool rowok = xid >= 0;
                auto combine = [&](const int32_t (&v)[NTIER][8], const long long (&ny)[8], int c0) {
                    const int j0 = NBLK * b + c0;            // column within the group
                    float o[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        // exact: d² = ||v_x||² + ||v_y||² − 2 Σ_t 2^{8t} T_t in int64 (wide
                        // multiply-adds; the 2^33 T4 term only touches the high word), then FP32
                        long long d2 = nx + ny[u];
                        asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(d2) : "r"(v[3][u]), "r"(-(1 << 25)));
                        asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(d2) : "r"(v[2][u]), "r"(-(1 << 17)));
                        asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(d2) : "r"(v[1][u]), "r"(-512));
                        asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(d2) : "r"(v[0][u]), "r"(-2));
                        d2 += (long long)((unsigned long long)(uint32_t)(-2 * v[4][u]) << 32);
                        float sq;
                        asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(u57_to_f32((unsigned long long)d2)));
                        o[u] = sq * a.scale;
                    }
                    if (!rowok || NGRP * g + j0 >= pitch || (FTD_ABL & 8)) return;
                    FTI_ASSERT(NGRP * g + j0 + 8 <= pitch && (!a.rowcnt || (int64_t)tile * TM + r < a.rowcnt[q]));
                    if (FTD_ST256) {
                        st_f8(trow + j0, o);
                    } else {
                        st_f4(trow + j0, make_float4(o[0], o[1], o[2], o[3]), wpol);
                        st_f4(trow + j0 + 4, make_float4(o[4], o[5], o[6], o[7]), wpol);
                    }
                };
                auto load = [&](int32_t (&v)[NTIER][8], int c0) {
#pragma unroll
                    for (int tt = 0; tt < NTIER; tt++) tmem_ld8(tb + (uint32_t)(tt * nwb + c0), v[tt]);
                };
                // ||ỹ||² of a chunk's 8 columns: read one chunk ahead (with its tier loads), so the
                // shared-memory latency — long while the tensor core streams operands — is hidden
                auto loadny = [&](long long (&ny)[8], int c0) {
#pragma unroll
                    for (int u = 0; u < 8; u++) ny[u] = eny[NBLK * b + c0 + u];
                };
                constexpr int STEP = 8 * NPART;
                int32_t va[NTIER][8];
                long long ya[8];
                int c0 = 8 * part;
                if (FTD_ABL & 4) c0 = nwb;
                if (FTD_EDB) {
                    int32_t vb[NTIER][8];
                    long long yb[8];
                    if (c0 < nwb) {
                        load(va, c0);
                        loadny(ya, c0);
                    }
                    while (c0 < nwb) {
                        TW(1, asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"));
                        if (c0 + STEP < nwb) {
                            load(vb, c0 + STEP);
                            loadny(yb, c0 + STEP);
                        }
                        TW(2, combine(va, ya, c0));
                        if (c0 + STEP >= nwb) break;
                        TW(1, asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"));
                        if (c0 + 2 * STEP < nwb) {
                            load(va, c0 + 2 * STEP);
                            loadny(ya, c0 + 2 * STEP);
                        }
                        TW(2, combine(vb, yb, c0 + STEP));
                        c0 += 2 * STEP;
                    }
                } else {
                    // more epilogue warps instead: the other warps of the SM sub-partition hide the
                    // TMEM load latency
                    for (; c0 < nwb; c0 += STEP) {
                        load(va, c0);
                        loadny(ya, c0);
                        TW(1, asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"));
                        TW(2, combine(va, ya, c0));
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(&acce[sl]);
            }
        }
    }
    if (DBG) {
        const unsigned long long tt = (unsigned long long)(clock64() - tstart);
        if (t == 0) { atomicAdd(&g_dbg[0], tt); atomicAdd(&g_dbg[1], dbgc[0]); atomicAdd(&g_dbg[12], 1ull);
                      atomicAdd(&g_dbg[13], (unsigned long long)(w_end - w_begin)); }
        if (t == NCOPY) { atomicAdd(&g_dbg[3], tt); atomicAdd(&g_dbg[4], dbgc[0]); atomicAdd(&g_dbg[5], dbgc[1]);
                          atomicAdd(&g_dbg[6], dbgc[2]); }
        if (t == NCOPY + 32) { atomicAdd(&g_dbg[7], tt); atomicAdd(&g_dbg[8], dbgc[0]); atomicAdd(&g_dbg[9], dbgc[1]);
                               atomicAdd(&g_dbg[10], dbgc[2]); }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == MMA_WARP)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// Work list: per query its 96-column groups G_q = ⌈s_q / 96⌉ and 128-row tiles; items ordered
// (query, group, tile); B operand offsets (16-byte units) of each query's groups.  One CTA,
// block-wide scans over 1024-query slabs.  With `units`: adds the stage's algorithmic bytes
// Σ_q rows_q · (d + 4 s_q) (the quantised rows read once, the table written once) and, in the
// next slot, the algorithmic flops Σ_q 2 · rows_q · s_q · d (one multiply-add per coordinate of
// every entry).
__global__ void __launch_bounds__(1024) k_tile_plan(DistArgs a, int d, unsigned long long* units) {
    __shared__ int tmp_t[32], tmp_b[32], tmp_g[32];
    int64_t tacc = 0, bacc = 0, gacc = 0;
    unsigned long long bytes = 0, flops = 0;
    for (int q0 = 0; q0 < a.nq; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        int items = 0, bsz = 0, s = 0;
        int64_t r = 0;
        if (q < a.nq) {
            const QHeader* h = (const QHeader*)(a.qblock + (size_t)q * a.L.stride);
            s = h->err ? 0 : (int)h->s;
            r = a.rowcnt ? (int64_t)a.rowcnt[q] : a.rows_cap;
            const int G = (s + NGRP - 1) / NGRP;
            items = s > 0 ? G * (int)((r + TM - 1) / TM) : 0;
            // B bytes / 16: full groups of 96 rows, the last rounded up to 16 rows
            const int last = s - NGRP * (G - 1);
            bsz = s > 0 ? (NL * a.kpad / 16) * (NGRP * (G - 1) + ((last + 15) & ~15)) : 0;
        }
        int tt, bt, gt;
        const int tex = fti_block_exclusive_sum(items, tmp_t, &tt);
        const int bex = fti_block_exclusive_sum(bsz, tmp_b, &bt);
        const int ng = s > 0 ? (s + NGRP - 1) / NGRP : 0;
        const int gex = fti_block_exclusive_sum(ng, tmp_g, &gt);
        if (q < a.nq) {
            if (a.gbase) a.gbase[q] = (int32_t)(gacc + gex);
            a.tile_base[q] = tacc + tex;
            a.qinfo[q] = make_uint2((uint32_t)(bacc + bex), (uint32_t)s);
            if (s > 0) {
                bytes += (unsigned long long)r * ((unsigned long long)d + 4ull * s);
                flops += 2ull * (unsigned long long)r * (unsigned long long)s * (unsigned long long)d;
            }
        }
        tacc += tt;
        bacc += bt;
        gacc += gt;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.tile_base[a.nq] = tacc;
        if (a.gbase) a.gbase[a.nq] = (int32_t)gacc;
    }
    if (units && bytes) atomicAdd(units, bytes);
    if (units && flops) atomicAdd(units + (FT_PROF_DIST_FLOPS - FTI_ST_DIST), flops);
}

// grid (nq, slices): the items' descriptors and row ids
__global__ void __launch_bounds__(TM) k_tiles(DistArgs a) {
    const int q = blockIdx.x;
    const uint2 qi = a.qinfo[q];
    if (qi.y == 0) return;
    const int64_t t0 = a.tile_base[q], t1 = a.tile_base[q + 1];
    const int64_t nrows = a.rowcnt ? (int64_t)a.rowcnt[q] : a.rows_cap;
    const int64_t tiles = (nrows + TM - 1) / TM;
    const int64_t GQ = a.tmajor ? (int64_t)a.gbase[a.nq] : 0;
    for (int64_t wl = t0 + blockIdx.y; wl < t1; wl += gridDim.y) {
        const int64_t g = (wl - t0) / tiles, tile = (wl - t0) - g * tiles;
        const int64_t w = a.tmajor ? tile * GQ + a.gbase[q] + g : wl;
        const int64_t row = tile * TM + threadIdx.x;
        int32_t xid = -1;
        if (row < nrows) xid = a.rows ? a.rows[(int64_t)q * a.rows_cap + row] : (int32_t)row;
        a.wrow[w * TM + threadIdx.x] = xid;
        if (threadIdx.x == 0)
            a.wdesc[w] = make_int4(q, (int)tile, (int)g | (group_cols((int)qi.y, (int)g) << 16),
                                   (int)(qi.x + (uint32_t)g * (NL * a.kpad / 16) * NGRP));
    }
}

// per (query, group): the query points' limbs in the B layout [limb][npad rows][kpad] (core
// matrices, 8-row groups kpad·8 bytes apart; rows past the support are zero) and their ||v||²
__global__ void __launch_bounds__(256) k_dist_prep(DistArgs a) {
    __shared__ int32_t yid[NGRP];
    const int q = blockIdx.x, g = blockIdx.y;
    const uint2 qi = a.qinfo[q];
    const int s = (int)qi.y;
    if (g * NGRP >= s) return;
    const uint8_t* slot = a.qblock + (size_t)q * a.L.stride;
    const uint2* qitems = (const uint2*)(slot + a.L.off_items);
    const int cols = group_cols(s, g), npad = (cols + 15) & ~15;
    for (int j = threadIdx.x; j < NGRP; j += blockDim.x) {
        const int32_t y = j < cols ? (int32_t)(qitems[NGRP * g + j].x & FTI_VOCAB_MASK) : -1;
        yid[j] = y;
        if (j < cols) a.ny[(int64_t)q * a.ny_ld + NGRP * g + j] = a.xnq[y];
    }
    __syncthreads();
    int8_t* bg = a.bq + 16 * (size_t)qi.x + (size_t)g * NL * a.kpad * NGRP;
    const size_t rstride = (size_t)a.nks * ROWB;
    const int sbo_b = a.kpad * 8, gran = a.kpad / 16;
    // block b (columns NBLK·b ..) stacks its limbs along N: region rows q·nb + j (nb = the block's
    // width), region b at row 3·NBLK·b
    const int total = NL * npad * gran;                    // thread per (region row, 16-byte K granule)
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int kg = e % gran, rr = e / gran;            // rr: row over the packed regions
        int b = 0, rb = rr;
        while (rb >= 3 * min(NBLK, npad - NBLK * b)) { rb -= 3 * min(NBLK, npad - NBLK * b); b++; }
        const int nbw = min(NBLK, npad - NBLK * b);
        const int p = rb / nbw, j = NBLK * b + rb % nbw;  // limb, query column within the group
        const int64_t src = j < cols ? (int64_t)yid[j] : a.N;     // the zero row pads the group
        const int c = kg / (KS / 16), kb = (kg % (KS / 16)) * 16;
        const uint4 v = *(const uint4*)(a.Xq + src * rstride + (size_t)c * ROWB + p * KS + kb);
        *(uint4*)(bg + (size_t)(3 * NBLK * b) * a.kpad + cm_off(rb, 16 * kg, sbo_b)) = v;
    }
}

// μ = the FP64 mean of the points: one CTA per coordinate
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

// max |x − μ| over all coordinates (a non-negative double's bits order like the double)
__global__ void __launch_bounds__(256) k_absmax(const float* __restrict__ X, int64_t n_el, int d,
                                                const double* __restrict__ mean, unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_el; i += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs((double)X[i] - mean[i % d]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// one warp per row (N + 1 rows, the last all zero): v = rint((x − μ)·2^e) → balanced limbs in the
// [nks][3][64] row layout, ||v||² exact in int64
__global__ void __launch_bounds__(256) k_quantize(const float* __restrict__ X, int64_t N, int d, int nks,
                                                  const double* __restrict__ mean, double scale_up,
                                                  int8_t* __restrict__ Xq, long long* __restrict__ xnq) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i > N) return;
    long long acc = 0;
    int8_t* row = Xq + i * (int64_t)nks * ROWB;
    for (int k = lane; k < nks * KS; k += 32) {
        long long v = 0;
        if (i < N && k < d) v = __double2ll_rn(((double)X[i * d + k] - mean[k]) * scale_up);
        acc += v * v;
        const int a0 = (int)(((v + 128) & 255) - 128);
        const long long v1 = (v - a0) >> 8;
        const int a1 = (int)(((v1 + 128) & 255) - 128);
        const int a2 = (int)((v1 - a1) >> 8);
        int8_t* dst = row + (k / KS) * ROWB + (k % KS);
        dst[0] = (int8_t)a0;
        dst[KS] = (int8_t)a1;
        dst[2 * KS] = (int8_t)a2;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) xnq[i] = acc;
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
    // a warp takes KV docs at a time: lane j < KV loads doc j's id and offsets, then every lane
    // loads its records of all KV docs (their loads in flight together — one doc at a time had
    // made cand -> doc_off -> items one dependent chain per doc)
    constexpr int KV = 4;
    // most items repeat an id that is already set (Zipf head ids: ~50k items, ~14k distinct per
    // reviews query): a plain read first keeps those off the shared-memory atomic unit
    auto set_bit = [&](uint32_t x) {
        const uint32_t b = 1u << (x & 31);
        if (!(((volatile uint32_t*)sbits)[x >> 5] & b)) atomicOr(&sbits[x >> 5], b);
    };
    for (int64_t c0 = (int64_t)warp * KV; c0 < n_cand; c0 += (int64_t)nw * KV) {
        uint32_t mi0 = 0, mi1 = 0;
        if (lane < KV && c0 + lane < n_cand) {
            const int64_t doc = cand[(int64_t)q * cand_ld + c0 + lane];
            // a negative candidate (padding / another shard's doc) has no rows; an index >= n is
            // reported (NaN + FT_ERANGE) by the Flowtree kernels and contributes no rows here
            if (doc >= 0 && doc < n) { mi0 = doc_off[doc]; mi1 = doc_off[doc + 1]; }
        }
        uint32_t i0[KV], i1[KV], xs[KV][3];
#pragma unroll
        for (int j = 0; j < KV; j++) {
            i0[j] = __shfl_sync(0xffffffffu, mi0, j);
            i1[j] = __shfl_sync(0xffffffffu, mi1, j);
#pragma unroll
            for (int t = 0; t < 3; t++) {
                const uint32_t i = i0[j] + lane + 32u * t;
                xs[j][t] = i < i1[j] ? __ldg(&items[i].x) : FTI_EMPTY;
            }
        }
#pragma unroll
        for (int j = 0; j < KV; j++) {
#pragma unroll
            for (int t = 0; t < 3; t++)
                if (xs[j][t] != FTI_EMPTY) set_bit(xs[j][t] & FTI_VOCAB_MASK);
            for (uint32_t i = i0[j] + lane + 96u; i < i1[j]; i += 32) {   // supports beyond 96 items
                set_bit(__ldg(&items[i].x) & FTI_VOCAB_MASK);
            }
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

// the index's quantised operand, built once on first use
cudaError_t prepare_quantized(ft_index* ix, cudaStream_t st) {
    if (ix->Xq) return cudaSuccess;
    const int nks = (ix->d + KS - 1) / KS;
    int8_t* Xq = nullptr;
    long long* xn = nullptr;
    double* mean = nullptr;
    unsigned long long* mx = nullptr;
    cudaError_t e;
    auto cleanup = [&]() { cudaFree(Xq); cudaFree(xn); cudaFree(mean); cudaFree(mx); };
    if ((e = cudaMalloc(&Xq, (size_t)(ix->N + 1) * nks * ROWB)) != cudaSuccess) { cleanup(); return e; }
    if ((e = cudaMalloc(&xn, sizeof(long long) * (size_t)(ix->N + 1))) != cudaSuccess) { cleanup(); return e; }
    if ((e = cudaMalloc(&mean, sizeof(double) * ix->d)) != cudaSuccess) { cleanup(); return e; }
    if ((e = cudaMalloc(&mx, sizeof(unsigned long long))) != cudaSuccess) { cleanup(); return e; }
    cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st);
    k_center_mean<<<ix->d, 256, 0, st>>>(ix->X, ix->N, ix->d, mean);
    k_absmax<<<1184, 256, 0, st>>>(ix->X, ix->N * ix->d, ix->d, mean, mx);
    unsigned long long mbits = 0;
    cudaMemcpyAsync(&mbits, mx, sizeof(mbits), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { cleanup(); return e; }
    double M;
    memcpy(&M, &mbits, sizeof(M));
    // the largest e with M·2^e ≤ 2^23 − 2^16 (so every balanced top limb is a signed byte)
    int qe = 0;
    if (M > 0.0 && std::isfinite(M)) {
        qe = (int)std::floor(std::log2((double)QMAX_ABS / M));
        while (std::ldexp(M, qe) > (double)QMAX_ABS) qe--;
        while (std::ldexp(M, qe + 1) <= (double)QMAX_ABS) qe++;
    }
    k_quantize<<<(unsigned)((ix->N + 1 + 7) / 8), 256, 0, st>>>(ix->X, ix->N, ix->d, nks, mean, std::ldexp(1.0, qe),
                                                                 Xq, xn);
    fti_count_launches(3);
    e = cudaStreamSynchronize(st);
    cudaFree(mean);
    cudaFree(mx);
    mean = nullptr;
    mx = nullptr;
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) { cleanup(); return e; }
    ix->Xq = Xq;
    ix->xnq = xn;
    ix->nks = nks;
    ix->qexp = qe;
    return cudaSuccess;
}

}  // namespace

// shared memory the distance-table kernel needs for a ring of `nstage` A stages at d (B resident)
static size_t dist_smem(int nstage, int kpad) {
    return (size_t)nstage * STAGE_BYTES + (size_t)NL * NGRP * kpad + NGRP * 8 + (2 * NSTAGE_MAX + 8) * 8 + 64;
}

bool fti_dist_supported(const ft_index* ix) {
    const int kpad = (ix->d + KS - 1) / KS * KS;
    return dist_smem(2, kpad) <= 227 * 1024;
}

cudaError_t fti_launch_dist_table(ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                                  const int32_t* d_rows, const int32_t* d_rowcnt, int64_t rows_cap,
                                  const int64_t* d_row_base, const int32_t* d_pitch, float* d_table, cudaStream_t st) {
    if (nq <= 0 || rows_cap <= 0) return cudaSuccess;
    ft_index* ix = const_cast<ft_index*>(ds->ix);
    if (!fti_dist_supported(ix)) return cudaErrorNotSupported;
    cudaError_t e;
    if ((e = prepare_quantized(ix, st)) != cudaSuccess) return e;
    DistArgs a{};
    a.Xq = ix->Xq;
    a.xnq = ix->xnq;
    a.N = ix->N;
    a.nks = ix->nks;
    a.kpad = ix->nks * KS;
    a.kz = std::min(a.kpad, (ix->d + 15) & ~15);
    a.scale = (float)std::ldexp(1.0, -ix->qexp);
    a.qblock = d_qblock;
    a.L = L;
    a.nq = nq;
    a.rows = d_rows;
    a.rowcnt = d_rowcnt;
    a.rows_cap = rows_cap;
    a.row_base = d_row_base;
    a.pitch = d_pitch;
    a.table = d_table;
    const int G = (L.smax + NGRP - 1) / NGRP;
    a.ny_ld = G * NGRP;
    const int64_t tmax = (int64_t)nq * G * ((rows_cap + TM - 1) / TM);
    if ((e = ds->s_gbase.reserve((size_t)(nq + 1) * 4)) != cudaSuccess) return e;
    if ((e = ds->s_bsplit.reserve((size_t)nq * G * NL * NGRP * a.kpad)) != cudaSuccess) return e;
    if ((e = ds->s_ny.reserve((size_t)nq * a.ny_ld * 8)) != cudaSuccess) return e;
    if ((e = ds->s_tiles.reserve((size_t)(nq + 1) * 8)) != cudaSuccess) return e;
    if ((e = ds->s_qinfo.reserve((size_t)nq * 8)) != cudaSuccess) return e;
    if ((e = ds->s_wdesc.reserve((size_t)tmax * 16)) != cudaSuccess) return e;
    if ((e = ds->s_wrow.reserve((size_t)tmax * TM * 4)) != cudaSuccess) return e;
    a.bq = ds->s_bsplit.as<int8_t>();
    a.ny = ds->s_ny.as<long long>();
    a.tile_base = ds->s_tiles.as<int64_t>();
    a.qinfo = ds->s_qinfo.as<uint2>();
    a.wdesc = ds->s_wdesc.as<int4>();
    a.wrow = ds->s_wrow.as<int32_t>();
    // the whole K range of a tile resident (block-outer MMA order) when it fits, else a ring of
    // 2..4 stages (K-outer order)
    int nstage = NSTAGE_MAX;
    while (nstage > 2 && dist_smem(nstage, a.kpad) > 227 * 1024) nstage--;
    a.blk_outer = (!FTD_KOUTER && nstage >= a.nks) ? 1 : 0;
    if (!a.blk_outer && !FTD_KOUTER) nstage = std::min(nstage, 4);
    a.nstage = nstage;
    a.gbase = ds->s_gbase.as<int32_t>();
    a.tmajor = (d_rows == nullptr && d_rowcnt == nullptr && a.blk_outer && nstage == a.nks &&
                !fti_opt(FT_OPT_DIST_QMAJOR)) ? 1 : 0;
    const size_t smem = dist_smem(nstage, a.kpad);
    const bool dbg = (fti_opt(FT_OPT_DEBUG) & FTI_DBG_DIST) != 0;
    auto kern = dbg ? k_dist_i8<true> : k_dist_i8<false>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    const unsigned slices = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (148 * 8 + nq - 1) / nq));
    k_tile_plan<<<1, 1024, 0, st>>>(a, ix->d, ds->units_ptr(FTI_ST_DIST));
    k_tiles<<<dim3((unsigned)nq, slices), TM, 0, st>>>(a);
    k_dist_prep<<<dim3((unsigned)nq, (unsigned)G), 256, 0, st>>>(a);
    kern<<<148, NTHREADS, smem, st>>>(a);
    fti_count_launches(4);
    if (dbg) {
        unsigned long long h[16];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_dbg, sizeof(h));
        const double n = h[12] ? (double)h[12] * 1e3 : 1.0;
        fprintf(stderr, "dist_i8 dbg per CTA (kcyc): copy total %.1f wait_empty %.1f | mma total %.1f wait_full %.1f "
                        "wait_acce %.1f wait_B %.1f | epi total %.1f wait_accf %.1f tmem_wait %.1f combine %.1f | "
                        "items/CTA %.1f nstage %d\n",
                h[0] / n, h[1] / n, h[3] / n, h[4] / n, h[5] / n, h[6] / n, h[7] / n, h[8] / n, h[9] / n, h[10] / n,
                (double)h[13] / (n / 1e3), a.nstage);
        memset(h, 0, sizeof(h));
        cudaMemcpyToSymbol(g_dbg, h, sizeof(h));
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
