// ft_dist.cu — a5: distance table D[c][j] = ||x_{v_c} − y_j||_2 between the candidate vocabulary and
// the query support, read by the Flowtree kernel to price its flow (
// Lemma 1's O(d) per matched pair).
//
// The table is a dense contraction, so it runs on the 5th-generation tensor cores (tcgen05):
//   ||x − y||^2 = ||x − c||^2 + ||y − c||^2 − 2 (x − c)·(y − c),   c = the query's centroid
// (centering keeps the Gram-form cancellation small for the near pairs that matter).  The dot
// products are 3xTF32 — every operand split as hi = tf32_rn(v), lo = v − hi, and
// D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi — which keeps ~22 significant bits, FP32 accumulation in
// TMEM.  One CTA = 128 candidate rows (UMMA M = 128) × the query's points (UMMA N ≤ 256) for one
// query; K = d in 32-wide chunks staged in shared memory in the canonical K-major core-matrix
// layout (SWIZZLE_NONE, LBO = 128 B, SBO = 1 KB); one elected thread issues the MMAs and commits
// to an mbarrier; the epilogue reads TMEM with tcgen05.ld (32x32b), forms the distance in FP32,
// forces an id shared by both sides to exactly 0, and writes the row.
//
// Candidate vocabulary for the prefiltered pipeline: k_mark flags every vocab id of the query's
// m candidates in a per-query map [N], k_compact turns the flags into dense row ids and the row
// list (block-wide scan over N).
#include <algorithm>

#include "ft_device.cuh"

namespace {

constexpr int TM = 128;     // rows per CTA = UMMA M
constexpr int KC = 16;      // K elements staged per chunk (64 B per row)
constexpr int NMAX = 256;   // query points per pass = max UMMA N
constexpr int SBO = (KC / 4) * 128;   // bytes between 8-row core-matrix groups

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    // K-major, SWIZZLE_NONE: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)((uint32_t)SBO >> 4) << 32) |
           (1ull << 46);
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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(phase)
            : "memory");
    }
}

__global__ void __launch_bounds__(TM) k_dist_tc(const float* __restrict__ X, int d, const uint8_t* qblock,
                                                QueryLayout L, const float* __restrict__ centers,
                                                const int32_t* __restrict__ rows, const int32_t* __restrict__ rowcnt,
                                                int64_t rows_cap, float* __restrict__ table, int ld) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t yid[NMAX];
    __shared__ float ny[NMAX];
    const int q = blockIdx.y;
    const uint8_t* slot = qblock + (size_t)q * L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    const uint2* qitems = (const uint2*)(slot + L.off_items);
    const int64_t nrows = rowcnt ? (int64_t)rowcnt[q] : rows_cap;
    const int64_t r0 = (int64_t)blockIdx.x * TM;
    if (r0 >= nrows || hdr->err != 0) return;
    const int sq = (int)hdr->s;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const float* cq = centers + (int64_t)q * d;
    const int64_t my_row = r0 + t;
    const int32_t xid = my_row < nrows ? (rows ? rows[(int64_t)q * rows_cap + my_row] : (int32_t)my_row) : -1;
    float* tq = table + (int64_t)q * rows_cap * ld;

    uint8_t* a_hi = sm;
    uint8_t* a_lo = a_hi + TM * KC * 4;
    uint8_t* b_hi = a_lo + TM * KC * 4;
    uint8_t* b_lo = b_hi + NMAX * KC * 4;

    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int np_max = min(NMAX, ((sq + 15) / 16) * 16);
    const uint32_t ncols = (uint32_t)fti_pow2_at_least(max(32, np_max));
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    uint32_t phase = 0;

    for (int cb = 0; cb < sq; cb += NMAX) {
        const int nb = min(NMAX, sq - cb);
        const int NP = ((nb + 15) / 16) * 16;
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
        for (int j = t; j < NMAX; j += TM) {
            yid[j] = (j < nb) ? (qitems[cb + j].x & FTI_VOCAB_MASK) : 0xFFFFFFFFu;
        }
        __syncthreads();
        float nx = 0.f, nyr[2] = {0.f, 0.f};
        const bool vec = (d & 3) == 0;
        const float* xr = X + (int64_t)(xid >= 0 ? xid : 0) * d;
        const float* yr0 = X + (int64_t)(t < nb ? yid[t] : 0) * d;
        const float* yr1 = X + (int64_t)(t + TM < nb ? yid[t + TM] : 0) * d;
        for (int k0 = 0; k0 < d; k0 += KC) {
            // stage A (this thread's row) and B (query points t, t+128), centered and split;
            // all loads of the chunk are issued before any use
            float4 c4[KC / 4], xv[KC / 4], y0[KC / 4], y1[KC / 4];
#pragma unroll
            for (int g = 0; g < KC / 4; g++) {
                const int k = k0 + 4 * g;
                if (vec) {
                    const bool in = k < d;
                    c4[g] = in ? *(const float4*)(cq + k) : make_float4(0.f, 0.f, 0.f, 0.f);
                    xv[g] = (in && xid >= 0) ? __ldg((const float4*)(xr + k)) : c4[g];
                    y0[g] = (in && t < nb) ? __ldg((const float4*)(yr0 + k)) : c4[g];
                    y1[g] = (in && t + TM < nb) ? __ldg((const float4*)(yr1 + k)) : c4[g];
                } else {
                    float c[4], a[4], b0[4], b1[4];
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const bool in = k + e < d;
                        c[e] = in ? cq[k + e] : 0.f;
                        a[e] = (in && xid >= 0) ? xr[k + e] : c[e];
                        b0[e] = (in && t < nb) ? yr0[k + e] : c[e];
                        b1[e] = (in && t + TM < nb) ? yr1[k + e] : c[e];
                    }
                    c4[g] = make_float4(c[0], c[1], c[2], c[3]);
                    xv[g] = make_float4(a[0], a[1], a[2], a[3]);
                    y0[g] = make_float4(b0[0], b0[1], b0[2], b0[3]);
                    y1[g] = make_float4(b1[0], b1[1], b1[2], b1[3]);
                }
            }
#pragma unroll
            for (int g = 0; g < KC / 4; g++) {
                float4 v = make_float4(xv[g].x - c4[g].x, xv[g].y - c4[g].y, xv[g].z - c4[g].z, xv[g].w - c4[g].w);
                nx = fmaf(v.x, v.x, nx); nx = fmaf(v.y, v.y, nx); nx = fmaf(v.z, v.z, nx); nx = fmaf(v.w, v.w, nx);
                split_store(a_hi, a_lo, t, g, v);
                if (t < NP) {
                    float4 w = make_float4(y0[g].x - c4[g].x, y0[g].y - c4[g].y, y0[g].z - c4[g].z, y0[g].w - c4[g].w);
                    nyr[0] = fmaf(w.x, w.x, nyr[0]); nyr[0] = fmaf(w.y, w.y, nyr[0]);
                    nyr[0] = fmaf(w.z, w.z, nyr[0]); nyr[0] = fmaf(w.w, w.w, nyr[0]);
                    split_store(b_hi, b_lo, t, g, w);
                }
                if (t + TM < NP) {
                    float4 w = make_float4(y1[g].x - c4[g].x, y1[g].y - c4[g].y, y1[g].z - c4[g].z, y1[g].w - c4[g].w);
                    nyr[1] = fmaf(w.x, w.x, nyr[1]); nyr[1] = fmaf(w.y, w.y, nyr[1]);
                    nyr[1] = fmaf(w.z, w.z, nyr[1]); nyr[1] = fmaf(w.w, w.w, nyr[1]);
                    split_store(b_hi, b_lo, t + TM, g, w);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (t == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int s = 0; s < KC / 8; s++) {
                    const uint64_t ah = umma_desc(smem_u32(a_hi) + 256 * s), al = umma_desc(smem_u32(a_lo) + 256 * s);
                    const uint64_t bh = umma_desc(smem_u32(b_hi) + 256 * s), bl = umma_desc(smem_u32(b_lo) + 256 * s);
                    const uint32_t acc0 = (k0 > 0 || s > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                        "l"(ah), "l"(bh), "r"(idesc), "r"(acc0));
                    asm volatile(
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(ah), "l"(bl),
                        "r"(idesc));
                    asm volatile(
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(al), "l"(bh),
                        "r"(idesc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&mbar))
                             : "memory");
            }
            mbar_wait(&mbar, phase);
            phase ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;");
        }
        for (int h = 0; h < 2; h++) {
            const int j = t + h * TM;
            if (j < NMAX) ny[j] = nyr[h];
        }
        __syncthreads();
        // epilogue: TMEM lane = row (warp w owns lanes 32w..32w+31)
        for (int c0 = 0; c0 < NP; c0 += 8) {
            uint32_t v[8];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (xid >= 0) {
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const int j = c0 + i;
                    if (j < nb) {
                        const float dot = __uint_as_float(v[i]);
                        const float d2 = nx + ny[j] - 2.f * dot;
                        const float dist = ((uint32_t)xid == yid[j]) ? 0.f : sqrtf(fmaxf(d2, 0.f));
                        tq[my_row * ld + cb + j] = dist;
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

// per-query centroid of the support points (FP32), the centering point of the Gram form
__global__ void k_query_center(const float* __restrict__ X, int d, const uint8_t* qblock, QueryLayout L,
                               float* __restrict__ centers) {
    const int q = blockIdx.x;
    const uint8_t* slot = qblock + (size_t)q * L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    const uint2* qitems = (const uint2*)(slot + L.off_items);
    const int s = hdr->err ? 0 : (int)hdr->s;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float acc = 0.f;
        for (int j = 0; j < s; j++) acc += X[(int64_t)(qitems[j].x & FTI_VOCAB_MASK) * d + i];
        centers[(int64_t)q * d + i] = s ? acc / (float)s : 0.f;
    }
}

// warp per candidate doc: flag its vocab ids in the query's map
__global__ void k_mark(const uint32_t* __restrict__ doc_off, const uint2* __restrict__ items,
                       const int64_t* __restrict__ cand, int64_t cand_ld, int64_t n_cand, int64_t N,
                       int32_t* __restrict__ map) {
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31;
    int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= n_cand) return;
    int64_t doc = cand[(int64_t)q * cand_ld + c];
    if (doc < 0) return;
    uint32_t i0 = doc_off[doc], i1 = doc_off[doc + 1];
    int32_t* mq = map + (int64_t)q * N;
    for (uint32_t i = i0 + lane; i < i1; i += 32) mq[items[i].x & FTI_VOCAB_MASK] = 1;
}

// one CTA per query: dense row ids in vocab order
__global__ void __launch_bounds__(1024) k_compact(int64_t N, int32_t* __restrict__ map, int32_t* __restrict__ rows,
                                                  int32_t* __restrict__ rowcnt, int64_t rows_cap) {
    __shared__ int tmp[32];
    const int q = blockIdx.x;
    int32_t* mq = map + (int64_t)q * N;
    int32_t* rq = rows + (int64_t)q * rows_cap;
    int run = 0;
    for (int64_t c = 0; c < N; c += blockDim.x) {
        int64_t v = c + threadIdx.x;
        int f = (v < N) ? (mq[v] != 0) : 0;
        int tot;
        int r = run + fti_block_exclusive_sum(f, tmp, &tot);
        if (f) {
            mq[v] = r;
            if (r < rows_cap) rq[r] = (int32_t)v;
        }
        run += tot;
    }
    if (threadIdx.x == 0) rowcnt[q] = run < rows_cap ? run : (int32_t)rows_cap;
}

}  // namespace

cudaError_t fti_launch_dist_table(const ft_index* ix, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                                  const int32_t* d_rows, const int32_t* d_rowcnt, int64_t rows_cap, float* d_table,
                                  int32_t ld, float* d_centers, cudaStream_t st) {
    if (nq <= 0 || rows_cap <= 0) return cudaSuccess;
    k_query_center<<<nq, 128, 0, st>>>(ix->X, ix->d, d_qblock, L, d_centers);
    const size_t smem = (size_t)2 * TM * KC * 4 + (size_t)2 * NMAX * KC * 4;
    cudaError_t e = cudaFuncSetAttribute(k_dist_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((rows_cap + TM - 1) / TM), (unsigned)nq);
    k_dist_tc<<<grid, TM, smem, st>>>(ix->X, ix->d, d_qblock, L, d_centers, d_rows, d_rowcnt, rows_cap, d_table, ld);
    fti_count_launches(2);
    return cudaGetLastError();
}

cudaError_t fti_launch_vocab_map(const ft_dataset* ds, int32_t nq, const int64_t* d_cand, int64_t cand_ld,
                                 int64_t n_cand, int32_t* d_map, int32_t* d_rows, int32_t* d_rowcnt, int64_t rows_cap,
                                 cudaStream_t st) {
    if (nq <= 0) return cudaSuccess;
    const int64_t N = ds->ix->N;
    cudaError_t e = cudaMemsetAsync(d_map, 0, sizeof(int32_t) * N * nq, st);
    if (e != cudaSuccess) return e;
    if (n_cand > 0) {
        dim3 g((unsigned)((n_cand * 32 + 255) / 256), (unsigned)nq);
        k_mark<<<g, 256, 0, st>>>(ds->doc_off, ds->items, d_cand, cand_ld, n_cand, N, d_map);
    }
    k_compact<<<nq, 1024, 0, st>>>(N, d_map, d_rows, d_rowcnt, rows_cap);
    fti_count_launches(n_cand > 0 ? 2 : 1);
    return cudaGetLastError();
}
