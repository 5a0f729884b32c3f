// Micro-benchmark: gathering random 960-byte rows (the distance table's A operand: 320 coordinates ×
// 3 int8 limbs) from a 96 MB array into shared memory, one persistent CTA per SM, by different copy
// mechanisms.  Reports the useful bytes per second.  Build and run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gb tools/gather_bench.cu && /tmp/gb
#include <cstdint>
#include <cstdio>
#include <vector>
#include <random>

constexpr int ROW = 960, NROWS = 100000, TM = 128;
constexpr int RING = 120 * 1024;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(done) : "r"(sa(b)), "r"(ph) : "memory");
}

// mode 0: cp.async 16 B per lane (8 rows × 64 B per warp instruction), all warps, wait_group per tile
// mode 1: ld.global.v8 (32 B per lane) into registers, st.shared, DEPTH tiles... (per warp: 16 loads in flight)
// mode 2: cp.async.bulk of CH bytes per request (one request per lane), mbarrier complete_tx
template <int MODE, int CH>
__global__ void __launch_bounds__(256, 1) k_gather(const int8_t* __restrict__ X, const int32_t* __restrict__ rows,
                                                   int tiles_per_cta, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[2];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    if (t == 0) { mb_init(&bar[0], 1); mb_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    uint32_t acc = 0;
    for (int it = 0; it < tiles_per_cta; it++) {
        const int32_t* tr = rows + ((size_t)blockIdx.x * tiles_per_cta + it) * TM;
        if (MODE == 0) {
            // 128 rows × 960 B = 7680 16-byte granules; thread handles granules t, t + 256, ...
            for (int g = t; g < TM * ROW / 16; g += blockDim.x) {
                const int r = g / (ROW / 16), c = g % (ROW / 16);
                const int8_t* src = X + (size_t)tr[r] * ROW + 16 * c;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(sm + (size_t)g * 16)), "l"(src) : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
        } else if (MODE == 1) {
            // 32-byte units: 128 rows × 30 = 3840; each thread 15 units, all loads in flight
            constexpr int U = TM * ROW / 32 / 256;
            uint32_t v[U][8];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int g = u * 256 + t;
                const int r = g / (ROW / 32), c = g % (ROW / 32);
                asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]), "=r"(v[u][5]),
                               "=r"(v[u][6]), "=r"(v[u][7])
                             : "l"(X + (size_t)tr[r] * ROW + 32 * c));
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int g = u * 256 + t;
                uint4* d = (uint4*)(sm + (size_t)g * 32);
                d[0] = make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
                d[1] = make_uint4(v[u][4], v[u][5], v[u][6], v[u][7]);
            }
            __syncthreads();
        } else if (MODE == 3) {
            // LDG with CH units of 32 B per thread in flight (threads beyond the tile's units idle)
            constexpr int U = CH;
            const int units = TM * ROW / 32;
            for (int g0 = 0; g0 < units; g0 += U * blockDim.x) {
                uint32_t v[U][8];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int g = g0 + u * blockDim.x + t;
                    if (g < units) {
                        const int r = g / (ROW / 32), c = g % (ROW / 32);
                        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                     : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]),
                                       "=r"(v[u][5]), "=r"(v[u][6]), "=r"(v[u][7])
                                     : "l"(X + (size_t)tr[r] * ROW + 32 * c));
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int g = g0 + u * blockDim.x + t;
                    if (g < units) {
                        uint4* d = (uint4*)(sm + (size_t)g * 32);
                        d[0] = make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
                        d[1] = make_uint4(v[u][4], v[u][5], v[u][6], v[u][7]);
                    }
                }
            }
            __syncthreads();
        } else if (MODE == 4) {
            // cp.async rolling: tile it issued, then wait for tile it − 1 (two tiles in flight, 60 KB
            // halves of the ring per tile: rows of 480 B)
            const int half = it & 1;
            for (int g = t; g < TM * ROW / 32; g += blockDim.x) {
                const int r = g / (ROW / 32), c = g % (ROW / 32);
                const int8_t* src = X + (size_t)tr[r] * ROW + 16 * c;   // first half of each row only
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(sm + half * (RING / 2) + (size_t)g * 16)), "l"(src) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
        } else {
            // bulk copies of CH bytes: 128 × 960 / CH requests spread over the threads
            constexpr int NREQ = TM * ROW / CH;
            const uint32_t ph = it & 1;
            if (t == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[0])), "r"(TM * ROW)
                             : "memory");
            __syncthreads();
            for (int q = t; q < NREQ; q += blockDim.x) {
                const int r = q / (ROW / CH), c = q % (ROW / CH);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa(sm + (size_t)q * CH)),
                    "l"(X + (size_t)tr[r] * ROW + CH * c), "r"(CH), "r"(sa(&bar[0]))
                    : "memory");
            }
            mb_wait(&bar[0], ph);
            __syncthreads();
        }
        acc += sm[(it * 97 + t) % RING];
        __syncthreads();
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
    (void)warp; (void)nw; (void)lane;
}

template <int MODE, int CH>
void run(const char* name, const int8_t* X, const int32_t* rows, int tiles, unsigned long long* sink) {
    auto k = k_gather<MODE, CH>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, RING);
    k<<<148, 256, RING>>>(X, rows, tiles, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 3; r++) k<<<148, 256, RING>>>(X, rows, tiles, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 3.0 * 148 * tiles * TM * (double)ROW / (MODE == 4 ? 2 : 1);
    printf("%-28s %8.3f ms  %7.2f TB/s useful  err=%s\n", name, ms / 3, bytes / (ms / 1e3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int tiles = 600;
    int8_t* X;
    int32_t* rows;
    unsigned long long* sink;
    cudaMalloc(&X, (size_t)NROWS * ROW);
    cudaMemset(X, 1, (size_t)NROWS * ROW);
    std::vector<int32_t> h((size_t)148 * tiles * TM);
    std::mt19937 g(1);
    for (auto& x : h) x = (int32_t)(g() % NROWS);
    cudaMalloc(&rows, h.size() * 4);
    cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&sink, 8);
    run<0, 16>("cp.async 16B", X, rows, tiles, sink);
    run<1, 32>("ld.v8 32B + st.shared", X, rows, tiles, sink);
    run<2, 64>("bulk 64B", X, rows, tiles, sink);
    run<2, 192>("bulk 192B", X, rows, tiles, sink);
    run<2, 960>("bulk 960B", X, rows, tiles, sink);
    run<2, 32>("bulk 32B", X, rows, tiles, sink);
    run<3, 2>("ldg 2 units/thread (16 KB)", X, rows, tiles, sink);
    run<3, 4>("ldg 4 units/thread (32 KB)", X, rows, tiles, sink);
    run<3, 8>("ldg 8 units/thread (64 KB)", X, rows, tiles, sink);
    run<3, 15>("ldg 15 units/thread (120 KB)", X, rows, tiles, sink);
    run<4, 16>("cp.async rolling 2x60KB (half rows)", X, rows, tiles, sink);
    return 0;
}
