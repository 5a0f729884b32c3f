// ft_build.cu — a0: GPU quadtree builder (§2 "Generic Quadtree").
//
// Pipeline (DESIGN.md §7 KB1):
//   k_minmax_*   per-axis min / max in FP64 → Φ = max range (reading R1)
//   k_phi_sigma  σ_i = Φ · U[0,1) from SplitMix64(seed, i) (reading R3); ℓ_root
//   per depth k = 1..D (reading R5):
//     k_bits      child bit-vector of every active point: bit_i = (q_i >> (D−k)) & 1 with the FP64
//                 cell rule q_i = min(⌊(t_i + (Φ − σ_i)) / (2Φ) · 2^D⌋, 2^D − 1) (readings R4, R7)
//     radix sort  LSD by bit-vector words then parent id (CUB radix sort, stable)
//     k_segment   new node = change of (parent, bit-vector); BFS id = level base + rank (R7)
//     k_assign    path table, node depth, node point counts
//     compaction  points in cells with ≥ 2 points continue (singleton leaves)
//   k_vflags     per ground point: leaf holds ≥ 2 points? any non-root ancestor with ≥ 2 points?
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "ft_internal.cuh"

namespace {

// SplitMix64 output i for state `seed` (reading R3) — this library's own implementation.
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_minmax_partial(const float* __restrict__ X, int64_t N, int d, int64_t rows_per_blk,
                                 double* __restrict__ pmn, double* __restrict__ pmx) {
    int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
    int64_t r1 = min(N, r0 + rows_per_blk);
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        double mn = INFINITY, mx = -INFINITY;
        for (int64_t r = r0; r < r1; r++) {
            double v = (double)X[r * d + i];
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
        }
        pmn[(int64_t)blockIdx.x * d + i] = mn;
        pmx[(int64_t)blockIdx.x * d + i] = mx;
    }
}

__global__ void k_minmax_final(const double* __restrict__ pmn, const double* __restrict__ pmx, int nblk, int d,
                               double* __restrict__ mn, double* __restrict__ range) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d) return;
    double a = INFINITY, b = -INFINITY;
    for (int t = 0; t < nblk; t++) {
        double u = pmn[(int64_t)t * d + i], v = pmx[(int64_t)t * d + i];
        a = u < a ? u : a;
        b = v > b ? v : b;
    }
    mn[i] = a;
    range[i] = __dsub_rn(b, a);
}

// one block: Φ = max_i range_i; σ; a_i = Φ − σ_i; ℓ_root = ⌈log2 Φ⌉ + 1 via frexp.
__global__ void k_phi_sigma(const double* __restrict__ range, int d, const double* __restrict__ sigma_in,
                            uint64_t seed, double* __restrict__ scal, double* __restrict__ sigma,
                            double* __restrict__ a) {
    __shared__ double red[1024];
    double m = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) m = range[i] > m ? range[i] : m;
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = red[threadIdx.x + s] > red[threadIdx.x] ? red[threadIdx.x + s] : red[threadIdx.x];
        __syncthreads();
    }
    double phi = red[0];
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        double s;
        if (sigma_in) {
            s = sigma_in[i];
        } else {
            uint64_t z = splitmix64_at(seed, (uint64_t)i);
            double r = (double)(z >> 11) * 0x1.0p-53;
            s = __dmul_rn(phi, r);
        }
        sigma[i] = s;
        a[i] = __dsub_rn(phi, s);
    }
    if (threadIdx.x == 0) {
        scal[0] = phi;
        int e = 0;
        double fr = phi > 0.0 ? frexp(phi, &e) : 0.0;   // phi = fr * 2^e, fr in [0.5, 1)
        int cl = (fr == 0.5) ? (e - 1) : e;
        scal[1] = phi > 0.0 ? (double)(cl + 1) : 0.0;
    }
}

// FP64 cell coordinate at the cap depth D (reading R4: half-open cells, top face clamped).
__device__ __forceinline__ long long cell_q(float x, double mn, double a, double two_phi, int D) {
    double t = __dsub_rn((double)x, mn);
    double num = __dadd_rn(t, a);
    double u = __ddiv_rn(num, two_phi);
    double s = scalbn(u, D);
    long long q = (long long)floor(s);
    long long top = (1ll << D) - 1;
    return q > top ? top : q;
}

// one warp per (active point, 32-dim chunk): ballot of the depth-k bits, dim 0 first.
// words are [nw][cap] u64, bits of dims 64w..64w+63 with dim 64w at bit 63.
__global__ void k_bits(const float* __restrict__ X, int d, const double* __restrict__ mn,
                       const double* __restrict__ a, const double* __restrict__ scal, int D, int k,
                       const uint32_t* __restrict__ act, int64_t n_act, int nchunk,
                       uint32_t* __restrict__ words32, int64_t cap) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double two_phi = __dmul_rn(2.0, scal[0]);
    for (int64_t t = warp; t < n_act * nchunk; t += nwarps) {
        int64_t ai = t / nchunk;
        int c = (int)(t - ai * nchunk);
        int i = c * 32 + lane;
        uint32_t p = act[ai];
        unsigned bit = 0;
        if (i < d) {
            long long q = cell_q(X[(int64_t)p * d + i], mn[i], a[i], two_phi, D);
            bit = (unsigned)((q >> (D - k)) & 1ll);
        }
        unsigned b = __brev(__ballot_sync(0xffffffffu, bit));
        if (lane == 0) {
            int w = c >> 1;
            // high half (dims 64w..64w+31) at the upper 32 bits of the little-endian u64
            words32[((int64_t)w * cap + ai) * 2 + ((c & 1) ? 0 : 1)] = b;
        }
    }
}

__global__ void k_iota(uint32_t* v, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

__global__ void k_gather_word(const uint64_t* __restrict__ words, const uint32_t* __restrict__ perm, int64_t n,
                              uint64_t* __restrict__ keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = words[perm[i]];
}

__global__ void k_gather_parent(const uint32_t* __restrict__ parent, const uint32_t* __restrict__ perm, int64_t n,
                                uint64_t* __restrict__ keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = parent[perm[i]];
}

__global__ void k_segment(const uint64_t* __restrict__ words, int nw, int64_t cap, const uint32_t* __restrict__ parent,
                          const uint32_t* __restrict__ perm, int64_t n, uint32_t* __restrict__ flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t f = 1;
    if (i > 0) {
        uint32_t p = perm[i], o = perm[i - 1];
        f = parent[p] != parent[o];
        for (int w = 0; w < nw && !f; w++) f = words[(int64_t)w * cap + p] != words[(int64_t)w * cap + o];
    }
    flag[i] = f;
}

__global__ void k_assign(const uint32_t* __restrict__ act, const uint32_t* __restrict__ perm,
                         const uint32_t* __restrict__ rank_incl, int64_t n, int64_t base, int k, int cols,
                         int32_t* __restrict__ path, uint8_t* __restrict__ node_depth,
                         int32_t* __restrict__ node_count, uint8_t* __restrict__ leaf_depth,
                         uint32_t* __restrict__ node_of) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t a = perm[i];
    uint32_t p = act[a];
    int64_t id = base + (int64_t)rank_incl[i] - 1;
    path[(int64_t)p * cols + k] = (int32_t)id;
    node_depth[id] = (uint8_t)k;
    atomicAdd(&node_count[id], 1);
    leaf_depth[p] = (uint8_t)k;
    node_of[i] = (uint32_t)id;
}

__global__ void k_continue_flags(const uint32_t* __restrict__ node_of, const int32_t* __restrict__ node_count,
                                 int64_t n, uint32_t* __restrict__ flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = node_count[node_of[i]] >= 2;
}

__global__ void k_gather_pts(const uint32_t* __restrict__ act, const uint32_t* __restrict__ perm, int64_t n,
                             uint32_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = act[perm[i]];
}

__global__ void k_repack_paths(const int32_t* __restrict__ src, int src_cols, int64_t N, int dst_cols,
                               int32_t* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * dst_cols) return;
    int64_t x = i / dst_cols;
    int c = (int)(i - x * dst_cols);
    dst[i] = src[x * src_cols + c];
}

__global__ void k_vflags(const int32_t* __restrict__ path, int cols, const uint8_t* __restrict__ leaf_depth,
                         const int32_t* __restrict__ node_count, int64_t N, uint32_t* __restrict__ vflags) {
    int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= N) return;
    int ld = leaf_depth[x];
    uint32_t f = 0;
    if (node_count[path[x * cols + ld]] >= 2) f |= FTI_FLAG_MULTI_LEAF;
    for (int k = 1; k <= ld; k++)
        if (node_count[path[x * cols + k]] >= 2) f |= FTI_FLAG_DEEP;
    vflags[x] = f;
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

template <class T>
cudaError_t grow_copy(T*& p, int64_t& cap, int64_t need, cudaStream_t st) {
    if (need <= cap) return cudaSuccess;
    int64_t nc = std::max<int64_t>(need, cap * 2);
    T* q = nullptr;
    cudaError_t e = cudaMalloc(&q, sizeof(T) * nc);
    if (e != cudaSuccess) return e;
    if (p) {
        e = cudaMemcpyAsync(q, p, sizeof(T) * cap, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        cudaStreamSynchronize(st);
        cudaFree(p);
    }
    p = q;
    cap = nc;
    return cudaSuccess;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
static ft_status build_impl(const float* X, int64_t N, int32_t d, const double* sigma_in, uint64_t seed,
                            int32_t max_depth, ft_index** out) {
    if (!out) return fti_fail(FT_EINVAL, "ft_build_quadtree: out is NULL");
    *out = nullptr;
    if (!X) return fti_fail(FT_EINVAL, "ft_build_quadtree: X is NULL");
    if (N < 1 || d < 1) return fti_fail(FT_EINVAL, "ft_build_quadtree: need N >= 1 and d >= 1");
    if (N >= (int64_t)FTI_VOCAB_MASK) return fti_fail(FT_ERANGE, "ft_build_quadtree: N must be < 2^30");
    int D = max_depth <= 0 ? 32 : max_depth;
    if (D > 52) return fti_fail(FT_EINVAL, "ft_build_quadtree: max_depth must be <= 52");

    cudaStream_t st;
    FTI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    ft_index* ix = new ft_index();
    ix->N = N; ix->d = d; ix->D = D;
    FTI_CUDA(cudaGetDevice(&ix->device));

    // device buffers
    FTI_CUDA(cudaMalloc(&ix->X, sizeof(float) * N * d));
    FTI_CUDA(cudaMemcpyAsync(ix->X, X, sizeof(float) * N * d, cudaMemcpyHostToDevice, st));
    int64_t rows_per = 256;
    int nb = (int)std::min<int64_t>((N + rows_per - 1) / rows_per, 4096);
    rows_per = (N + nb - 1) / nb;
    double *pmn, *pmx, *mn, *range, *scal, *sig, *a, *sig_in = nullptr;
    FTI_CUDA(cudaMalloc(&pmn, sizeof(double) * nb * d));
    FTI_CUDA(cudaMalloc(&pmx, sizeof(double) * nb * d));
    FTI_CUDA(cudaMalloc(&mn, sizeof(double) * d));
    FTI_CUDA(cudaMalloc(&range, sizeof(double) * d));
    FTI_CUDA(cudaMalloc(&scal, sizeof(double) * 2));
    FTI_CUDA(cudaMalloc(&sig, sizeof(double) * d));
    FTI_CUDA(cudaMalloc(&a, sizeof(double) * d));
    if (sigma_in) {
        FTI_CUDA(cudaMalloc(&sig_in, sizeof(double) * d));
        FTI_CUDA(cudaMemcpyAsync(sig_in, sigma_in, sizeof(double) * d, cudaMemcpyHostToDevice, st));
    }
    k_minmax_partial<<<nb, 256, 0, st>>>(ix->X, N, d, rows_per, pmn, pmx);
    k_minmax_final<<<nblk(d), 256, 0, st>>>(pmn, pmx, nb, d, mn, range);
    k_phi_sigma<<<1, 1024, 0, st>>>(range, d, sig_in, seed, scal, sig, a);
    double hs[2];
    FTI_CUDA(cudaMemcpyAsync(hs, scal, sizeof(hs), cudaMemcpyDeviceToHost, st));
    ix->sigma.resize(d);
    ix->mn.resize(d);
    FTI_CUDA(cudaMemcpyAsync(ix->sigma.data(), sig, sizeof(double) * d, cudaMemcpyDeviceToHost, st));
    FTI_CUDA(cudaMemcpyAsync(ix->mn.data(), mn, sizeof(double) * d, cudaMemcpyDeviceToHost, st));
    FTI_CUDA(cudaStreamSynchronize(st));
    FTI_CUDA(cudaGetLastError());
    ix->phi = hs[0];
    ix->l_root = (int32_t)hs[1];

    // per-point arrays
    int cols = D + 1;
    int32_t* path_full;
    FTI_CUDA(cudaMalloc(&path_full, sizeof(int32_t) * N * cols));
    FTI_CUDA(cudaMemsetAsync(path_full, 0xFF, sizeof(int32_t) * N * cols, st));
    FTI_CUDA(cudaMalloc(&ix->leaf_depth, N));
    FTI_CUDA(cudaMemsetAsync(ix->leaf_depth, 0, N, st));
    // column 0 = root for every point
    {
        // path[x][0] = 0 (the root) for every point, via a strided memset
        FTI_CUDA(cudaMemset2DAsync(path_full, sizeof(int32_t) * cols, 0, sizeof(int32_t), N, st));
    }
    int64_t node_cap = std::max<int64_t>(2 * N + 1, 1024);
    FTI_CUDA(cudaMalloc(&ix->node_depth, node_cap));
    FTI_CUDA(cudaMalloc(&ix->node_count, sizeof(int32_t) * node_cap));
    FTI_CUDA(cudaMemsetAsync(ix->node_depth, 0, node_cap, st));
    FTI_CUDA(cudaMemsetAsync(ix->node_count, 0, sizeof(int32_t) * node_cap, st));
    {
        int32_t nN = (int32_t)N;
        FTI_CUDA(cudaMemcpyAsync(ix->node_count, &nN, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        FTI_CUDA(cudaStreamSynchronize(st));
    }
    int64_t base = 1;   // node 0 = root
    int d_star = 0;
    ix->level_base.assign(1, 0);

    bool root_internal = (N >= 2 && ix->phi > 0.0 && D >= 1);
    if (root_internal) {
        int nw = (d + 63) / 64, nchunk = (d + 31) / 32;
        int64_t cap = N;
        uint32_t *act, *act_next, *parent, *parent_next, *perm, *perm2, *flag, *rank, *node_of, *cnt_sel;
        uint64_t *words, *keys, *keys2;
        FTI_CUDA(cudaMalloc(&act, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&act_next, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&parent, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&parent_next, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&perm, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&perm2, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&flag, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&rank, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&node_of, sizeof(uint32_t) * cap));
        FTI_CUDA(cudaMalloc(&cnt_sel, sizeof(uint32_t) * 2));
        FTI_CUDA(cudaMalloc(&words, sizeof(uint64_t) * cap * nw));
        FTI_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * cap));
        FTI_CUDA(cudaMalloc(&keys2, sizeof(uint64_t) * cap));
        k_iota<<<nblk(N), 256, 0, st>>>(act, N);
        FTI_CUDA(cudaMemsetAsync(parent, 0, sizeof(uint32_t) * N, st));
        // CUB temp storage (sized for the largest pass)
        size_t tmp_sort = 0, tmp_scan = 0, tmp_sel = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, keys, keys2, perm, perm2, (int)N, 0, 64, st);
        cub::DeviceScan::InclusiveSum(nullptr, tmp_scan, flag, rank, (int)N, st);
        cub::DeviceSelect::Flagged(nullptr, tmp_sel, act, flag, act_next, cnt_sel, (int)N, st);
        size_t tmp_bytes = std::max(tmp_sort, std::max(tmp_scan, tmp_sel));
        void* tmp;
        FTI_CUDA(cudaMalloc(&tmp, tmp_bytes));

        int64_t n_act = N;
        for (int k = 1; k <= D && n_act > 0; k++) {
            ix->level_base.push_back(base);
            FTI_CUDA(cudaMemsetAsync(words, 0, sizeof(uint64_t) * cap * nw, st));
            k_bits<<<std::min<int64_t>(((n_act * nchunk) * 32 + 255) / 256, 148 * 64), 256, 0, st>>>(
                ix->X, d, mn, a, scal, D, k, act, n_act, nchunk, (uint32_t*)words, cap);
            k_iota<<<nblk(n_act), 256, 0, st>>>(perm, n_act);
            // LSD: least significant word first, parent id last
            for (int w = nw - 1; w >= -1; w--) {
                if (w >= 0) k_gather_word<<<nblk(n_act), 256, 0, st>>>(words + (int64_t)w * cap, perm, n_act, keys);
                else k_gather_parent<<<nblk(n_act), 256, 0, st>>>(parent, perm, n_act, keys);
                size_t tb = tmp_bytes;
                FTI_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, perm, perm2, (int)n_act, 0, 64, st));
                std::swap(perm, perm2);
            }
            k_segment<<<nblk(n_act), 256, 0, st>>>(words, nw, cap, parent, perm, n_act, flag);
            size_t tb = tmp_bytes;
            FTI_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, flag, rank, (int)n_act, st));
            uint32_t n_new = 0;
            FTI_CUDA(cudaMemcpyAsync(&n_new, rank + n_act - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            FTI_CUDA(cudaStreamSynchronize(st));
            int64_t old_cap = node_cap;
            if (base + n_new > node_cap) {
                int64_t oc = node_cap;
                FTI_CUDA(grow_copy(ix->node_depth, oc, base + n_new, st));
                oc = node_cap;
                FTI_CUDA(grow_copy(ix->node_count, oc, base + n_new, st));
                node_cap = oc;
                FTI_CUDA(cudaMemsetAsync(ix->node_depth + old_cap, 0, node_cap - old_cap, st));
                FTI_CUDA(cudaMemsetAsync(ix->node_count + old_cap, 0, sizeof(int32_t) * (node_cap - old_cap), st));
            }
            k_assign<<<nblk(n_act), 256, 0, st>>>(act, perm, rank, n_act, base, k, cols, path_full,
                                                    ix->node_depth, ix->node_count, ix->leaf_depth, node_of);
            base += n_new;
            d_star = k;
            if (k == D) break;
            // points in cells with >= 2 points continue, in sorted order; their parent is that cell
            k_continue_flags<<<nblk(n_act), 256, 0, st>>>(node_of, ix->node_count, n_act, flag);
            k_gather_pts<<<nblk(n_act), 256, 0, st>>>(act, perm, n_act, act_next);
            tb = tmp_bytes;
            FTI_CUDA(cub::DeviceSelect::Flagged(tmp, tb, act_next, flag, act, cnt_sel, (int)n_act, st));
            tb = tmp_bytes;
            FTI_CUDA(cub::DeviceSelect::Flagged(tmp, tb, node_of, flag, parent, cnt_sel + 1, (int)n_act, st));
            uint32_t nn = 0;
            FTI_CUDA(cudaMemcpyAsync(&nn, cnt_sel, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            FTI_CUDA(cudaStreamSynchronize(st));
            n_act = nn;
        }
        cudaFree(act); cudaFree(act_next); cudaFree(parent); cudaFree(parent_next); cudaFree(perm);
        cudaFree(perm2); cudaFree(flag); cudaFree(rank); cudaFree(node_of); cudaFree(cnt_sel);
        cudaFree(words); cudaFree(keys); cudaFree(keys2); cudaFree(tmp);
    }
    ix->level_base.push_back(base);
    ix->M = base;
    ix->d_star = d_star;
    // repack the path table to D*+1 columns
    FTI_CUDA(cudaMalloc(&ix->path, sizeof(int32_t) * N * (d_star + 1)));
    k_repack_paths<<<nblk(N * (d_star + 1)), 256, 0, st>>>(path_full, cols, N, d_star + 1, ix->path);
    FTI_CUDA(cudaMalloc(&ix->vflags, sizeof(uint32_t) * N));
    k_vflags<<<nblk(N), 256, 0, st>>>(ix->path, d_star + 1, ix->leaf_depth, ix->node_count, N, ix->vflags);
    FTI_CUDA(cudaStreamSynchronize(st));
    FTI_CUDA(cudaGetLastError());
    cudaFree(path_full); cudaFree(pmn); cudaFree(pmx); cudaFree(mn); cudaFree(range); cudaFree(scal);
    cudaFree(sig); cudaFree(a);
    if (sig_in) cudaFree(sig_in);
    cudaStreamDestroy(st);
    *out = ix;
    return FT_OK;
}

extern "C" ft_status ft_build_quadtree(const float* X, int64_t N, int32_t d, uint64_t seed, int32_t max_depth,
                                       ft_index** out) {
    return build_impl(X, N, d, nullptr, seed, max_depth, out);
}

extern "C" ft_status ft_build_quadtree_shift(const float* X, int64_t N, int32_t d, const double* sigma,
                                             int32_t max_depth, ft_index** out) {
    if (!sigma) return fti_fail(FT_EINVAL, "ft_build_quadtree_shift: sigma is NULL");
    return build_impl(X, N, d, sigma, 0, max_depth, out);
}

extern "C" ft_status ft_index_info(const ft_index* ix, double* phi, int32_t* l_root, int32_t* d_star,
                                   int64_t* n_nodes) {
    if (!ix) return fti_fail(FT_ESTATE, "ft_index_info: NULL index");
    if (phi) *phi = ix->phi;
    if (l_root) *l_root = ix->l_root;
    if (d_star) *d_star = ix->d_star;
    if (n_nodes) *n_nodes = ix->M;
    return FT_OK;
}

extern "C" ft_status ft_index_paths(const ft_index* ix, int32_t* out) {
    if (!ix || !out) return fti_fail(FT_ESTATE, "ft_index_paths: NULL argument");
    FTI_CUDA(cudaMemcpy(out, ix->path, sizeof(int32_t) * ix->N * (ix->d_star + 1), cudaMemcpyDeviceToHost));
    return FT_OK;
}

extern "C" ft_status ft_index_sigma(const ft_index* ix, double* sigma) {
    if (!ix || !sigma) return fti_fail(FT_ESTATE, "ft_index_sigma: NULL argument");
    for (int i = 0; i < ix->d; i++) sigma[i] = ix->sigma[i];
    return FT_OK;
}

extern "C" ft_status ft_index_nodes(const ft_index* ix, int32_t* depth, int32_t* count) {
    if (!ix) return fti_fail(FT_ESTATE, "ft_index_nodes: NULL index");
    if (depth) {
        std::vector<uint8_t> t(ix->M);
        FTI_CUDA(cudaMemcpy(t.data(), ix->node_depth, ix->M, cudaMemcpyDeviceToHost));
        for (int64_t v = 0; v < ix->M; v++) depth[v] = t[v];
    }
    if (count) FTI_CUDA(cudaMemcpy(count, ix->node_count, sizeof(int32_t) * ix->M, cudaMemcpyDeviceToHost));
    return FT_OK;
}

extern "C" void ft_index_free(ft_index* ix) {
    if (!ix) return;
    cudaFree(ix->X); cudaFree(ix->path); cudaFree(ix->leaf_depth); cudaFree(ix->node_depth);
    cudaFree(ix->node_count); cudaFree(ix->vflags); cudaFree(ix->Xq); cudaFree(ix->xnq);
    delete ix;
}
