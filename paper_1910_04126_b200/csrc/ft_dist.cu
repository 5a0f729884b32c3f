// ft_dist.cu — a5: distance table D[c][j] = ||x_{v_c} − y_j||_2 between the candidate vocabulary
// and the query support, read by the Flowtree kernel to price its flow
// (Lemma 1's O(d) per matched pair).
//
// FP32 direct differences Σ_t (x_t − y_t)^2 (no Gram-form cancellation; an id on both sides gives
// exactly 0), tiled 64 rows × 64 query points per CTA with 32-dim slabs staged in shared memory,
// each thread owning a 4×4 register tile.
//
// Candidate vocabulary for the prefiltered pipeline: k_mark flags every vocab id of the query's
// m candidates in a per-query map [N], k_compact turns the flags into dense row ids and the row
// list (block-wide scan over N).
#include <algorithm>

#include "ft_device.cuh"

namespace {

constexpr int TR = 64, TC = 64, TK = 32;

__global__ void __launch_bounds__(256) k_dist_table(const float* __restrict__ X, int d, const uint8_t* qblock,
                                                    QueryLayout L, const int32_t* __restrict__ rows,
                                                    const int32_t* __restrict__ rowcnt, int64_t rows_cap,
                                                    float* __restrict__ table, int ld) {
    __shared__ float xs[TR][TK + 1];
    __shared__ float ys[TC][TK + 1];
    __shared__ uint32_t yid[TC];
    __shared__ int32_t xid[TR];
    const int q = blockIdx.y;
    const uint8_t* slot = qblock + (size_t)q * L.stride;
    const QHeader* hdr = (const QHeader*)slot;
    const uint2* qitems = (const uint2*)(slot + L.off_items);
    const int64_t nrows = rowcnt ? (int64_t)rowcnt[q] : rows_cap;
    const int64_t r0 = (int64_t)blockIdx.x * TR;
    if (r0 >= nrows || hdr->err != 0) return;
    const int sq = (int)hdr->s;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float* tq = table + (int64_t)q * rows_cap * ld;
    for (int i = threadIdx.x; i < TR; i += blockDim.x) {
        int64_t r = r0 + i;
        xid[i] = r < nrows ? (rows ? rows[(int64_t)q * rows_cap + r] : (int32_t)r) : -1;
    }
    for (int c0 = 0; c0 < sq; c0 += TC) {
        __syncthreads();
        for (int i = threadIdx.x; i < TC; i += blockDim.x)
            yid[i] = (c0 + i < sq) ? (qitems[c0 + i].x & FTI_VOCAB_MASK) : 0xFFFFFFFFu;
        float acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int v = 0; v < 4; v++) acc[u][v] = 0.f;
        for (int k0 = 0; k0 < d; k0 += TK) {
            __syncthreads();
            for (int i = threadIdx.x; i < TR * TK; i += blockDim.x) {
                int r = i / TK, t = i - r * TK;
                int32_t x = xid[r];
                xs[r][t] = (x >= 0 && k0 + t < d) ? X[(int64_t)x * d + k0 + t] : 0.f;
            }
            for (int i = threadIdx.x; i < TC * TK; i += blockDim.x) {
                int cidx = i / TK, t = i - cidx * TK;
                uint32_t y = yid[cidx];
                ys[cidx][t] = (y != 0xFFFFFFFFu && k0 + t < d) ? X[(int64_t)y * d + k0 + t] : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int t = 0; t < TK; t++) {
                float xv[4], yv[4];
#pragma unroll
                for (int u = 0; u < 4; u++) xv[u] = xs[ty + 16 * u][t];
#pragma unroll
                for (int v = 0; v < 4; v++) yv[v] = ys[tx + 16 * v][t];
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int v = 0; v < 4; v++) {
                        float df = xv[u] - yv[v];
                        acc[u][v] = fmaf(df, df, acc[u][v]);
                    }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            int64_t r = r0 + ty + 16 * u;
            if (r >= nrows) continue;
#pragma unroll
            for (int v = 0; v < 4; v++) {
                int cidx = c0 + tx + 16 * v;
                if (cidx < sq) tq[r * ld + cidx] = sqrtf(acc[u][v]);
            }
        }
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
                                  int32_t ld, cudaStream_t st) {
    if (nq <= 0 || rows_cap <= 0) return cudaSuccess;
    dim3 grid((unsigned)((rows_cap + TR - 1) / TR), (unsigned)nq);
    k_dist_table<<<grid, 256, 0, st>>>(ix->X, ix->d, d_qblock, L, d_rows, d_rowcnt, rows_cap, d_table, ld);
    fti_count_launches(1);
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
