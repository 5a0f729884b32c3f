// ft_select.cu — a4 / a7: exact top-k selection by (value asc, doc id asc) (
// ties by doc id, reading R14).
//
// One CTA per row.  Keys are 96-bit composites (order-preserving image of the FP64 value, doc id).
// The k-th smallest key is found by MSD radix select with 8-bit digits (shared histograms), with an
// early exit as soon as the k-th key's bucket is taken whole; every key whose processed digits
// are ≤ the selected prefix is then gathered (exactly k of them) and bitonic-sorted in shared
// memory.  Exact for any amount of ties — the Quadtree keys at d = 300 take only a few hundred
// distinct values over 10^5 docs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ft_device.cuh"

namespace {

__device__ __forceinline__ unsigned long long okey(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)b);
}

__device__ __forceinline__ unsigned digit_of(unsigned long long hi, uint32_t lo, int t) {
    return t < 8 ? (unsigned)((hi >> (56 - 8 * t)) & 255ull) : (unsigned)((lo >> (24 - 8 * (t - 8))) & 255u);
}


// Sample-threshold selection (the common case): sort a strided sample of the keys, take a key a
// safe margin above the sample's k/L quantile as threshold t, gather every key ≤ t (exact count,
// warp-aggregated positions) and bitonic-sort the gathered (key, id) pairs; the first k are the
// answer.  Exact whenever k ≤ count(≤ t) ≤ capacity; otherwise the row is flagged for the radix
// kernel.  Two passes over the row instead of up to twelve.

// Block-wide rank selection over keys in shared memory (512 threads): the r-th smallest (0-based)
// of n composite keys (h, l) — or of h alone when l is null (ties then share the answer's h) — by
// MSD radix with 8-bit digits, starting at the first byte where the smallest and largest keys
// differ.  Per pass: a 256-bin histogram of the keys still matching the selected prefix
// (warp-aggregated with __match_any_sync, so a hot bin takes one atomic per warp), warp 0 finds
// the bin holding rank r.  Every thread returns the selected (h, l).
struct SelScratch {
    unsigned hist[256];
    unsigned long long ph, mn, mx;
    uint32_t pl;
    int need, byte0;
};

__device__ void block_rank_select(const unsigned long long* h, const uint32_t* l, int n, int r, SelScratch& sc,
                                  unsigned long long& out_h, uint32_t& out_l) {
    const int tid = threadIdx.x, lane = tid & 31, nt = blockDim.x;
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int i = tid; i < n; i += nt) { mn = min(mn, h[i]); mx = max(mx, h[i]); }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (tid == 0) { sc.mn = ~0ull; sc.mx = 0ull; sc.need = r; sc.pl = 0; }
    __syncthreads();
    if (lane == 0) { atomicMin(&sc.mn, mn); atomicMax(&sc.mx, mx); }
    __syncthreads();
    const int common = sc.mn == sc.mx ? 64 : __clzll((long long)(sc.mn ^ sc.mx));
    const int b0 = common / 8;                           // bytes of h shared by every key
    unsigned long long ph = b0 ? (sc.mn & (~0ull << (64 - 8 * b0))) : 0ull;
    uint32_t pl = 0;
    const int nd = l ? 12 : 8;
    for (int t = b0; t < nd; t++) {
        for (int b = tid; b < 256; b += nt) sc.hist[b] = 0;
        __syncthreads();
        const unsigned long long mh = t == 0 ? 0ull : (t <= 8 ? ~0ull << (64 - 8 * t) : ~0ull);
        const uint32_t ml = t <= 8 ? 0u : ~0u << (32 - 8 * (t - 8));
        for (int i0 = 0; i0 < n; i0 += nt) {
            const int i = i0 + tid;
            bool in = false;
            unsigned dg = 0;
            if (i < n) {
                const unsigned long long hh = h[i];
                const uint32_t ll = l ? l[i] : 0u;
                in = (hh & mh) == ph && (ll & ml) == pl;
                dg = t < 8 ? (unsigned)((hh >> (56 - 8 * t)) & 255ull) : (unsigned)((ll >> (24 - 8 * (t - 8))) & 255u);
            }
            const unsigned act = __ballot_sync(0xffffffffu, in);
            if (in) {
                const unsigned grp = __match_any_sync(act, dg);
                if (lane == __ffs(grp) - 1) atomicAdd(&sc.hist[dg], (unsigned)__popc(grp));
            }
        }
        __syncthreads();
        if (tid < 32) {
            const unsigned need = (unsigned)sc.need;     // read before the shuffles order the write
            unsigned c[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) { c[j] = sc.hist[8 * lane + j]; sum += c[j]; }
            unsigned incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            unsigned cum = incl - sum;
            const bool mine = cum <= need && need < incl;
            if (mine) {
                int j = 0;
                while (cum + c[j] <= need) { cum += c[j]; j++; }
                const unsigned dgt = 8 * lane + j;
                sc.need = (int)(need - cum);
                if (t < 8) sc.ph = ph | ((unsigned long long)dgt << (56 - 8 * t));
                else sc.pl = pl | (dgt << (24 - 8 * (t - 8)));
            }
        }
        __syncthreads();
        if (t < 8) ph = sc.ph; else pl = sc.pl;
    }
    out_h = ph;
    out_l = pl;
    __syncthreads();
}

constexpr int SEL_CAP = 8192;
constexpr int SEL_SAMPLE = 8192;          // = SEL_CAP: the sample fills the key buffer; ±1/√(rank) count noise

__device__ void sort_pairs(unsigned long long* h, uint32_t* l, int P) {
    for (int kb = 2; kb <= P; kb <<= 1) {
        for (int j = kb >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long ah = h[i], bh2 = h[ixj];
                    const uint32_t al = l[i], bl2 = l[ixj];
                    const bool gt = (ah > bh2) || (ah == bh2 && al > bl2);
                    const bool up = (i & kb) == 0;
                    if (gt == up) { h[i] = bh2; h[ixj] = ah; l[i] = bl2; l[ixj] = al; }
                }
            }
            __syncthreads();
        }
    }
}

__device__ unsigned long long g_seldbg[8];

template <bool DBG, int GU>
__global__ void __launch_bounds__(512, 2) k_select_fast(const double* __restrict__ vals, int64_t vals_ld,
                                                     const int64_t* __restrict__ ids, int64_t ids_ld, int64_t L,
                                                     int k, int64_t* __restrict__ out_ids,
                                                     double* __restrict__ out_val, int64_t out_ld,
                                                     int* __restrict__ redo, int* __restrict__ nredo, int64_t id_base,
                                                     const uint32_t* __restrict__ row_len, const int* __restrict__ rows_list,
                                                     const int* __restrict__ nrows_list, int* __restrict__ bad,
                                                     int nosort) {
    extern __shared__ unsigned long long sbuf[];
    unsigned long long* bh = sbuf;                      // SEL_CAP
    uint32_t* bl = (uint32_t*)(sbuf + SEL_CAP);         // SEL_CAP
    __shared__ SelScratch sc;
    __shared__ int s_cnt, s_lt;
    __shared__ int s_wsum[16];
    if (rows_list && (int)blockIdx.x >= *nrows_list) return;
    const int row = rows_list ? rows_list[blockIdx.x] : (int)blockIdx.x;
    const double* v = vals + (int64_t)row * vals_ld;
    const int64_t* id = ids ? ids + (int64_t)row * ids_ld : nullptr;
    if (row_len) {
        // a candidate list: rows shorter than k or longer than the list capacity are handed back
        const int64_t len = (int64_t)row_len[row];
        if (bad && (len > L || len < (int64_t)k)) {
            if (threadIdx.x == 0) bad[1 + atomicAdd(bad, 1)] = row;
            return;
        }
        L = min(L, len);
    }
    const int kk = (int)min((int64_t)k, L);
    const int lane = threadIdx.x & 31;
    long long t0 = DBG ? clock64() : 0, t1 = 0, t2 = 0, t3 = 0;
    if (threadIdx.x == 0) { s_cnt = 0; s_lt = 0; }
    unsigned long long thr = ~0ull;
    if (L > SEL_CAP) {
        // strided sample of S keys; threshold = the sample key at the k/L quantile + margin.  The
        // full 8192-key sample only when the quantile rank of a half sample would be small (the
        // count noise is ±1/√rank)
        const int S = (int64_t)kk * (SEL_SAMPLE / 2) < 32 * L ? SEL_SAMPLE : SEL_SAMPLE / 2;
        {
            constexpr int SU = SEL_SAMPLE / 512;        // all of a thread's sample loads in flight at once
            double sv[SU];
#pragma unroll
            for (int u = 0; u < SU; u++) {
                const int j = u * 512 + threadIdx.x;
                sv[u] = j < S ? v[(int64_t)j * L / S] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < SU; u++) {
                const int j = u * 512 + threadIdx.x;
                if (j < S) bh[j] = okey(sv[u]);
            }
        }
        __syncthreads();
        const double ex = (double)kk * S / (double)L;
        const int ti = min(S - 1, (int)(ex + 4.0 * sqrt(ex) + 8.0));
        uint32_t dummy;
        block_rank_select(bh, nullptr, S, ti, sc, thr, dummy);
    }
    if (DBG) t1 = clock64();
    // gather every key ≤ thr (all of them when L ≤ SEL_CAP); GU loads in flight per thread, then
    // warp-aggregated positions
    for (int64_t i0 = 0; i0 < L; i0 += (int64_t)blockDim.x * GU) {
        double vv[GU];
#pragma unroll
        for (int u = 0; u < GU; u++) {
            const int64_t i = i0 + (int64_t)u * blockDim.x + threadIdx.x;
            vv[u] = i < L ? v[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GU; u++) {
            const int64_t i = i0 + (int64_t)u * blockDim.x + threadIdx.x;
            const unsigned long long hi = okey(vv[u]);
            const bool sel = i < L && hi <= thr;
            const unsigned bal = __ballot_sync(0xffffffffu, sel);
            if (bal == 0u) continue;
            const unsigned blt = __ballot_sync(0xffffffffu, sel && hi < thr);
            int base = 0;
            if (lane == 0) {
                base = atomicAdd(&s_cnt, __popc(bal));
                if (blt) atomicAdd(&s_lt, __popc(blt));
            }
            base = __shfl_sync(0xffffffffu, base, 0);
            if (sel) {
                const int pos = base + __popc(bal & ((1u << lane) - 1u));
                if (pos < SEL_CAP) { bh[pos] = hi; bl[pos] = id ? (uint32_t)id[i] : (uint32_t)(id_base + i); }
            }
        }
    }
    __syncthreads();
    if (DBG) t2 = clock64();
    int cnt = s_cnt;
    const int c_lt = s_lt;
    int nk = cnt;
    const bool below_only = cnt > SEL_CAP && c_lt >= kk && c_lt <= SEL_CAP;   // the keys < t suffice
    const bool tie_fill = cnt > SEL_CAP && !id && c_lt < kk;                   // plus the first ties
    if (tie_fill || below_only) {
        // too many keys tie with the threshold for the buffer (the Quadtree values of a large
        // collection take few distinct values): gather the keys strictly below it, then either
        // they already hold the answer (rank-select below), or the answer is all of them plus the
        // first kk − c_lt tied keys in row order (implicit ids = positions: row order is id order)
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int64_t i0 = 0; i0 < L; i0 += (int64_t)blockDim.x * GU) {
            double vv[GU];
#pragma unroll
            for (int u = 0; u < GU; u++) {
                const int64_t i = i0 + (int64_t)u * blockDim.x + threadIdx.x;
                vv[u] = i < L ? v[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < GU; u++) {
                const int64_t i = i0 + (int64_t)u * blockDim.x + threadIdx.x;
                const unsigned long long hi = okey(vv[u]);
                const bool sel = i < L && hi < thr;
                const unsigned bal = __ballot_sync(0xffffffffu, sel);
                if (bal == 0u) continue;
                int base = 0;
                if (lane == 0) base = atomicAdd(&s_cnt, __popc(bal));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (sel) {
                    const int pos = base + __popc(bal & ((1u << lane) - 1u));
                    bh[pos] = hi;
                    bl[pos] = id ? (uint32_t)id[i] : (uint32_t)(id_base + i);
                }
            }
        }
        __syncthreads();
        cnt = c_lt;
        nk = c_lt;
    }
    if (tie_fill) {
        const int R = kk - c_lt;
        // the tied keys in row order: each thread a contiguous run of GU, block prefix of counts
        const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        int found = 0;
        for (int64_t i0 = 0; i0 < L && found < R; i0 += (int64_t)blockDim.x * GU) {
            const int64_t ib = i0 + (int64_t)threadIdx.x * GU;
            unsigned eqm = 0;
#pragma unroll
            for (int u = 0; u < GU; u++)
                if (ib + u < L && okey(v[ib + u]) == thr) eqm |= 1u << u;
            const int mine = __popc(eqm);
            int incl = mine;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            __syncthreads();                         // s_wsum reuse
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            int woff = 0, tot = 0;
            for (int w = 0; w < nw; w++) {
                const int x = s_wsum[w];
                if (w < warp) woff += x;
                tot += x;
            }
            int pos = found + woff + incl - mine;
            for (int u = 0; u < GU && eqm; u++) {
                if ((eqm >> u) & 1u) {
                    if (pos < R) { bh[c_lt + pos] = thr; bl[c_lt + pos] = (uint32_t)(id_base + ib + u); }
                    pos++;
                }
            }
            found += tot;                            // uniform: every thread summed the same totals
        }
        __syncthreads();
        cnt = kk;
        nk = kk;
    } else if (!below_only && (cnt < kk || cnt > SEL_CAP)) {   // threshold too low / ties with ids: radix
        if (threadIdx.x == 0) redo[atomicAdd(nredo, 1)] = row;
        return;
    }
    // small sets sort faster than they rank-select — unless only the set is wanted (nosort)
    if ((cnt > 2048 || nosort) && cnt > kk && kk > 0) {
        // the kk-th smallest gathered (key, id) — composites are distinct — then keep the kk keys
        // at or below it (positions by warp-aggregated atomics: the sort below fixes the order)
        unsigned long long th;
        uint32_t tl;
        block_rank_select(bh, bl, cnt, kk - 1, sc, th, tl);
        constexpr int PER = SEL_CAP / 512;
        unsigned long long kh[PER];
        uint32_t kl[PER];
#pragma unroll
        for (int j = 0; j < PER; j++) {
            const int i = j * blockDim.x + threadIdx.x;
            kh[j] = i < cnt ? bh[i] : ~0ull;
            kl[j] = i < cnt ? bl[i] : 0xFFFFFFFFu;
        }
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; j++) {
            const int i = j * blockDim.x + threadIdx.x;
            const bool keep = i < cnt && (kh[j] < th || (kh[j] == th && kl[j] <= tl));
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (bal == 0u) continue;
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_cnt, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (keep) {
                const int pos = base + __popc(bal & ((1u << lane) - 1u));
                bh[pos] = kh[j];
                bl[pos] = kl[j];
            }
        }
        __syncthreads();
        nk = kk;
    }
    if (!nosort) {
        const int P = fti_pow2_at_least(max(nk, 2));
        for (int i = nk + threadIdx.x; i < P; i += blockDim.x) { bh[i] = ~0ull; bl[i] = 0xFFFFFFFFu; }
        __syncthreads();
        sort_pairs(bh, bl, P);
    }
    if (DBG) t3 = clock64();
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        int64_t oid = -1;
        double ov = __longlong_as_double(0x7ff0000000000000ll);
        if (t < kk) {
            ov = okey_inv(bh[t]);
            oid = bl[t] == 0xFFFFFFFFu ? -1 : (int64_t)bl[t];
        }
        out_ids[(int64_t)row * out_ld + t] = oid;
        out_val[(int64_t)row * out_ld + t] = ov;
    }
    if (DBG && threadIdx.x == 0) {
        atomicAdd(&g_seldbg[0], (unsigned long long)(t1 - t0));
        atomicAdd(&g_seldbg[1], (unsigned long long)(t2 - t1));
        atomicAdd(&g_seldbg[2], (unsigned long long)(t3 - t2));
        atomicAdd(&g_seldbg[3], (unsigned long long)(clock64() - t3));
        atomicAdd(&g_seldbg[4], 1ull);
        atomicAdd(&g_seldbg[5], (unsigned long long)cnt);
    }
}

// MSD radix selection (rows the sample-threshold pass could not finish; `rows_list` null: all rows)
__global__ void __launch_bounds__(512) k_select(const double* __restrict__ vals, int64_t vals_ld,
                                                const int64_t* __restrict__ ids, int64_t ids_ld, int64_t L, int k,
                                                int64_t* __restrict__ out_ids, double* __restrict__ out_val,
                                                int64_t out_ld, int P, const int* __restrict__ rows_list,
                                                const int* __restrict__ nrows_list, int64_t id_base,
                                                const uint32_t* __restrict__ row_len) {
    if (rows_list && (int)blockIdx.x >= *nrows_list) return;
    extern __shared__ unsigned long long sbuf[];
    unsigned long long* bh = sbuf;               // P
    uint32_t* bl = (uint32_t*)(sbuf + P);        // P
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_ph, s_mh;
    __shared__ uint32_t s_pl, s_ml;
    __shared__ int s_need, s_done, s_cnt;
    const int row = rows_list ? rows_list[blockIdx.x] : blockIdx.x;
    const double* v = vals + (int64_t)row * vals_ld;
    const int64_t* id = ids ? ids + (int64_t)row * ids_ld : nullptr;
    if (row_len) L = std::min<int64_t>(L, (int64_t)row_len[row]);
    const int kk = (int)std::min<int64_t>(k, L);
    if (threadIdx.x == 0) { s_ph = 0; s_mh = 0; s_pl = 0; s_ml = 0; s_need = kk; s_done = 0; s_cnt = 0; }
    __syncthreads();
    if (kk > 0 && kk < L) {
        for (int t = 0; t < 12; t++) {
            for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            const unsigned long long ph = s_ph, mh = s_mh;
            const uint32_t pl = s_pl, ml = s_ml;
            for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
                unsigned long long hi = okey(v[i]);
                uint32_t lo = id ? (uint32_t)id[i] : (uint32_t)(id_base + i);
                if ((hi & mh) == ph && (lo & ml) == pl) atomicAdd(&hist[digit_of(hi, lo, t)], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int need = s_need;
                unsigned cum = 0;
                int b = 0;
                for (; b < 256; b++) {
                    if (cum + hist[b] >= (unsigned)need) break;
                    cum += hist[b];
                }
                need -= (int)cum;
                if (t < 8) {
                    s_ph = ph | ((unsigned long long)b << (56 - 8 * t));
                    s_mh = mh | (255ull << (56 - 8 * t));
                } else {
                    s_pl = pl | ((uint32_t)b << (24 - 8 * (t - 8)));
                    s_ml = ml | (255u << (24 - 8 * (t - 8)));
                }
                s_need = need;
                s_done = (hist[b] == (unsigned)need);
            }
            __syncthreads();
            if (s_done) break;
        }
    }
    const unsigned long long ph = s_ph, mh = s_mh;
    const uint32_t pl = s_pl, ml = s_ml;
    const bool all = (kk >= L);
    for (int64_t i = threadIdx.x; i < L && kk > 0; i += blockDim.x) {
        unsigned long long hi = okey(v[i]);
        uint32_t lo = id ? (uint32_t)id[i] : (uint32_t)(id_base + i);
        unsigned long long h2 = hi & mh;
        uint32_t l2 = lo & ml;
        bool sel = all || h2 < ph || (h2 == ph && l2 <= pl);
        if (sel) {
            int pos = atomicAdd(&s_cnt, 1);
            if (pos < P) { bh[pos] = hi; bl[pos] = lo; }
        }
    }
    __syncthreads();
    const int cnt = min(s_cnt, P);
    for (int i = cnt + threadIdx.x; i < P; i += blockDim.x) { bh[i] = ~0ull; bl[i] = 0xFFFFFFFFu; }
    __syncthreads();
    // bitonic sort by (hi, lo)
    for (int kb = 2; kb <= P; kb <<= 1) {
        for (int j = kb >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    unsigned long long ah = bh[i], bh2 = bh[ixj];
                    uint32_t al = bl[i], bl2 = bl[ixj];
                    bool gt = (ah > bh2) || (ah == bh2 && al > bl2);
                    bool up = (i & kb) == 0;
                    if (gt == up) { bh[i] = bh2; bh[ixj] = ah; bl[i] = bl2; bl[ixj] = al; }
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        int64_t oid = -1;
        double ov = __longlong_as_double(0x7ff0000000000000ll);
        if (t < kk && t < cnt) {
            ov = okey_inv(bh[t]);
            oid = (int64_t)bl[t];
            if (bl[t] == 0xFFFFFFFFu) oid = -1;
        }
        out_ids[(int64_t)row * out_ld + t] = oid;
        out_val[(int64_t)row * out_ld + t] = ov;
    }
}

// Per row, a value t ≥ the r-th smallest (0-based) of the row's L values and within FP32 rounding of
// it: the values rounded up to FP32 (order-preserving u32 keys, NaN largest), the r-th key by MSD
// radix select with 11/11/10-bit digits (three passes over the row through L2).  The prefilter's
// sample threshold (only count(value ≤ t) ≥ m matters there, so the FP32 round-up is harmless).
__global__ void __launch_bounds__(256) k_row_threshold(const double* __restrict__ vals, int64_t ld, int64_t L, int64_t r,
                                                       double* __restrict__ thr) {
    __shared__ unsigned hist[2048];
    __shared__ uint32_t s_pre, s_need;
    __shared__ int s_tmp[32];
    const int row = blockIdx.x;
    const double* v = vals + (int64_t)row * ld;
    auto key_of = [](double x) -> uint32_t {
        if (x != x) return 0xFFFFFFFFu;
        const uint32_t b = __float_as_uint(__double2float_ru(x));
        return (b >> 31) ? ~b : (b | 0x80000000u);
    };
    if (threadIdx.x == 0) { s_pre = 0u; s_need = (uint32_t)r; }
    const int shift[3] = {21, 10, 0}, width[3] = {11, 11, 10};
    uint32_t pmask = 0u;
    for (int p = 0; p < 3; p++) {
        for (int b = threadIdx.x; b < 2048; b += blockDim.x) hist[b] = 0u;
        __syncthreads();
        const uint32_t pre = s_pre;
        const uint32_t dm = (1u << width[p]) - 1u;
        for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
            const uint32_t k = key_of(v[i]);
            if ((k & pmask) == pre) atomicAdd(&hist[(k >> shift[p]) & dm], 1u);
        }
        __syncthreads();
        {
            // the digit holding the need-th key: each thread sums a run of bins, a block scan places
            // the runs, and the one thread whose run holds it walks its bins (a single thread
            // walking all 2048 bins had made this kernel latency-bound: 0.19 ms per 1,000 rows)
            const int nb = 1 << width[p], per = (nb + (int)blockDim.x - 1) / (int)blockDim.x;
            const int b0 = (int)threadIdx.x * per;
            uint32_t run = 0u;
            for (int j = 0; j < per && b0 + j < nb; j++) run += hist[b0 + j];
            const uint32_t need = s_need;
            const uint32_t before = (uint32_t)fti_block_exclusive_sum((int)run, s_tmp, nullptr);
            if (run > 0u && before <= need && need < before + run) {
                uint32_t cum = before;
                int b = b0;
                while (cum + hist[b] <= need) { cum += hist[b]; b++; }
                s_need = need - cum;
                s_pre = pre | ((uint32_t)b << shift[p]);
            }
        }
        pmask |= dm << shift[p];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint32_t k = s_pre;
        const uint32_t b = (k >> 31) ? (k & 0x7FFFFFFFu) : ~k;
        thr[row] = k == 0xFFFFFFFFu ? __longlong_as_double(0x7ff0000000000000ll) : (double)__uint_as_float(b);
    }
}

}  // namespace

cudaError_t fti_launch_row_threshold(const double* d_vals, int64_t ld, int64_t L, int32_t rows, int64_t r,
                                     double* d_thr, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    k_row_threshold<<<rows, 256, 0, st>>>(d_vals, ld, L, r, d_thr);
    fti_count_launches(1);
    return cudaGetLastError();
}

cudaError_t fti_launch_select(const double* d_vals, int64_t vals_ld, const int64_t* d_ids, int64_t ids_ld, int64_t L,
                              int32_t rows, int32_t k, int64_t* d_out_ids, double* d_out_val, int64_t out_ld,
                              int* d_scratch, cudaStream_t st, int64_t id_base, const uint32_t* d_row_len,
                              const int* d_rows_list, const int* d_nrows_list, int* d_bad, bool nosort) {
    if (rows <= 0) return cudaSuccess;
    int kk = (int)std::min<int64_t>(k, L);
    int P = fti_pow2_at_least(std::max(kk, 2));
    size_t smem = (size_t)P * 12 + 16;
    cudaError_t e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (fti_opt(FT_OPT_SELECT_RADIX)) {   // test option: the radix kernel for every row
        k_select<<<rows, 512, smem, st>>>(d_vals, vals_ld, d_ids, ids_ld, L, k, d_out_ids, d_out_val, out_ld, P,
                                          d_rows_list, d_nrows_list, id_base, d_row_len);
        fti_count_launches(1);
        return cudaGetLastError();
    }
    // pass 1: sample threshold + gather + sort; rows it cannot finish are listed in d_scratch[1..]
    int* nredo = d_scratch;
    int* redo = d_scratch + 1;
    e = cudaMemsetAsync(nredo, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    const size_t smem_f = (size_t)SEL_CAP * 12;
    const bool dbg = (fti_opt(FT_OPT_DEBUG) & FTI_DBG_SELECT) != 0;
    auto kf = L > SEL_CAP ? (dbg ? k_select_fast<true, 16> : k_select_fast<false, 16>)
                          : (dbg ? k_select_fast<true, 2> : k_select_fast<false, 2>);
    e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
    if (e != cudaSuccess) return e;
    // two 98 KB CTAs per SM need the maximum shared-memory carveout
    e = cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    kf<<<rows, 512, smem_f, st>>>(d_vals, vals_ld, d_ids, ids_ld, L, k, d_out_ids, d_out_val, out_ld, redo, nredo,
                                  id_base, d_row_len, d_rows_list, d_nrows_list, d_bad, nosort ? 1 : 0);
    if (dbg) {
        unsigned long long h[8];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_seldbg, sizeof(h));
        const double c = h[4] ? (double)h[4] : 1.0;
        fprintf(stderr, "select dbg per CTA (kcyc): sample %.1f gather %.1f sort %.1f out %.1f | cnt %.0f rows %.0f\n",
                h[0] / c / 1e3, h[1] / c / 1e3, h[2] / c / 1e3, h[3] / c / 1e3, h[5] / c, c);
        memset(h, 0, sizeof(h));
        cudaMemcpyToSymbol(g_seldbg, h, sizeof(h));
    }
    // pass 2: MSD radix selection of the listed rows (CTAs past the list exit at once)
    k_select<<<rows, 512, smem, st>>>(d_vals, vals_ld, d_ids, ids_ld, L, k, d_out_ids, d_out_val, out_ld, P, redo,
                                      nredo, id_base, d_row_len);
    fti_count_launches(2);
    return cudaGetLastError();
}
