// ft_qt.cu — a3: Quadtree estimate kernel (§2 "Wasserstein-1 on Quadtree").
//
// For a (query ν, doc μ) pair with cross-scaled masses (reading R13):
//   num = Σ_{v≠root} ω(v) |U m_μ(v) − W m_ν(v)|
//       = U·A + W·B − 2 Σ_{v ∈ nodes(μ) ∩ nodes(ν)} ω(v) min(U m_μ(v), W m_ν(v))
//   QT  = (num · 2^{ℓ_root − D*}) / (W·U)
// so the kernel streams the doc's node-sorted record (the sparse ℓ1 embedding)
// once, probes each record against the query node hashes staged in shared memory, and only the
// common nodes contribute.  The numerator is an exact u64; the value takes two correctly
// rounded FP64 operations, so it is bit-identical to the oracle.
//
// Mapping: a CTA stages QC queries' node hashes in shared memory and streams a contiguous doc
// range; one warp per doc, lane-strided 8-byte records (coalesced); per-warp shared u64
// accumulators per query (hits are rare at d = 300, so atomics do not contend).
#include <algorithm>

#include "ft_device.cuh"

namespace {

struct QtArgs {
    const uint32_t* qt_off;
    const uint2* qt;
    const uint32_t* W;
    const unsigned long long* A;
    const uint8_t* qblock;
    QueryLayout L;
    int32_t nq;
    const int64_t* docs;
    int64_t n_docs;
    int64_t n;
    int64_t docs_per_cta;
    double* out;
    int64_t out_ld;
    int d_star, l_root;
    int QC;
    int hcap;           // hash entries staged per query (max over the batch, = L.nh_cap)
    uint32_t* err;
};

constexpr int QT_WARPS = 8;

__global__ void __launch_bounds__(QT_WARPS * 32) k_qt(QtArgs a) {
    extern __shared__ unsigned long long sm[];
    // layout: acc[QT_WARPS][QC] u64 | hash[QC][hcap] uint2 | depth[QC][hcap] u8
    unsigned long long* acc = sm;
    uint2* hs = (uint2*)(acc + QT_WARPS * a.QC);
    uint8_t* hd = (uint8_t*)(hs + (size_t)a.QC * a.hcap);
    __shared__ uint32_t s_mask[32], s_U[32], s_ok[32];
    __shared__ unsigned long long s_B[32];

    const int q0 = blockIdx.y * a.QC;
    const int nqc = min(a.QC, a.nq - q0);
    for (int t = threadIdx.x; t < nqc; t += blockDim.x) {
        const QHeader* h = (const QHeader*)(a.qblock + (size_t)(q0 + t) * a.L.stride);
        s_mask[t] = h->nh_mask;
        s_U[t] = h->U;
        s_B[t] = h->B;
        s_ok[t] = (h->err == 0 && h->s > 0);
    }
    __syncthreads();
    for (int t = 0; t < nqc; t++) {
        const uint8_t* slot = a.qblock + (size_t)(q0 + t) * a.L.stride;
        const uint2* src = (const uint2*)(slot + a.L.off_nh);
        const uint8_t* srcd = slot + a.L.off_nd;
        int n = (int)s_mask[t] + 1;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            hs[(size_t)t * a.hcap + i] = src[i];
            hd[(size_t)t * a.hcap + i] = srcd[i];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* wacc = acc + warp * a.QC;
    const int64_t d0 = (int64_t)blockIdx.x * a.docs_per_cta;
    const int64_t d1 = min(a.n_docs, d0 + a.docs_per_cta);
    for (int64_t dp = d0 + warp; dp < d1; dp += QT_WARPS) {
        const int64_t doc = a.docs ? a.docs[dp] : dp;
        if (doc < 0 || doc >= a.n) {
            if (lane < nqc) a.out[(int64_t)(q0 + lane) * a.out_ld + dp] = __longlong_as_double(0x7ff8000000000000ll);
            if (lane == 0) atomicOr(a.err, FTI_ERR_RANGE);
            continue;
        }
        const uint32_t r0 = a.qt_off[doc], r1 = a.qt_off[doc + 1];
        const uint32_t W = a.W[doc];
        for (int t = lane; t < nqc; t += 32) wacc[t] = 0ull;
        __syncwarp();
        for (uint32_t r = r0 + lane; r < r1; r += 32) {
            const uint2 rec = a.qt[r];
            const uint32_t hh = fti_hash(rec.x);
            for (int t = 0; t < nqc; t++) {
                const uint32_t mask = s_mask[t];
                const uint2* tab = hs + (size_t)t * a.hcap;
                uint32_t h = hh & mask;
                while (true) {
                    const uint2 e = tab[h];
                    if (e.x == rec.x) {
                        const unsigned long long um = (unsigned long long)s_U[t] * rec.y;
                        const unsigned long long wm = (unsigned long long)W * e.y;
                        const unsigned long long mn = um < wm ? um : wm;
                        atomicAdd(&wacc[t], mn << (a.d_star - hd[(size_t)t * a.hcap + h]));
                        break;
                    }
                    if (e.x == FTI_EMPTY) break;
                    h = (h + 1) & mask;
                }
            }
        }
        __syncwarp();
        if (lane < nqc) {
            double val;
            const unsigned long long U = s_U[lane];
            const unsigned long long A = a.A[doc];
            const unsigned long long B = s_B[lane];
            const unsigned long long S2 = wacc[lane] << 1;
            bool bad = !s_ok[lane];
            bad |= __umul64hi(U, A) != 0ull || __umul64hi((unsigned long long)W, B) != 0ull;
            const unsigned long long ua = U * A, wb = (unsigned long long)W * B;
            const unsigned long long tot = ua + wb;
            bad |= tot < ua;
            const unsigned long long num = tot - S2;
            if (!bad && num >= (1ull << 53)) {
                bad = true;
                atomicOr(a.err, FTI_ERR_OVERFLOW);
            }
            if (bad) {
                val = __longlong_as_double(0x7ff8000000000000ll);
            } else {
                const double scaled = scalbn((double)num, a.l_root - a.d_star);
                val = __ddiv_rn(scaled, (double)(U * (unsigned long long)W));
            }
            a.out[(int64_t)(q0 + lane) * a.out_ld + dp] = val;
        }
        __syncwarp();
    }
}

}  // namespace

cudaError_t fti_launch_qt(const ft_dataset* ds, const QueryLayout& L, const uint8_t* d_qblock, int32_t nq,
                          const int64_t* d_docs, int64_t docs_ld, int64_t n_docs, double* d_out, int64_t out_ld,
                          cudaStream_t st) {
    (void)docs_ld;   // the Quadtree stage always scores one doc list shared by the batch
    if (nq <= 0 || n_docs <= 0) return cudaSuccess;
    QtArgs a{};
    a.qt_off = ds->qt_off; a.qt = ds->qt; a.W = ds->W; a.A = ds->A;
    a.qblock = d_qblock; a.L = L; a.nq = nq; a.docs = d_docs; a.n_docs = n_docs; a.n = ds->n;
    a.out = d_out; a.out_ld = out_ld;
    a.d_star = ds->ix->d_star; a.l_root = ds->ix->l_root;
    a.hcap = L.nh_cap;
    a.err = ds->err_dev;
    const size_t per_q = (size_t)a.hcap * 9 + QT_WARPS * 8;
    int QC = (int)std::min<size_t>(16, std::max<size_t>(1, (96 * 1024) / per_q));
    QC = std::min(QC, nq);
    a.QC = QC;
    const int qchunks = (nq + QC - 1) / QC;
    int64_t bx = std::max<int64_t>(1, std::min<int64_t>((n_docs + 63) / 64, (148 * 6 + qchunks - 1) / qchunks));
    a.docs_per_cta = (n_docs + bx - 1) / bx;
    bx = (n_docs + a.docs_per_cta - 1) / a.docs_per_cta;
    size_t smem = (size_t)QT_WARPS * QC * 8 + (size_t)QC * a.hcap * 8 + (size_t)QC * a.hcap + 16;
    cudaError_t e = cudaFuncSetAttribute(k_qt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_qt<<<dim3((unsigned)bx, (unsigned)qchunks), QT_WARPS * 32, smem, st>>>(a);
    fti_count_launches(1);
    return cudaGetLastError();
}
