// tune_zech.cu -- standalone B200 experiment for the Zech dot (not part of the product): is a TMA 1-D
// bulk-copy operand ring in shared memory (beside the 128 KB antilog table) faster than the product's
// register-pipelined LDG stream, whose loads are limited by the 64-register cap of 1024-thread CTAs?
// Same policy math (Zech<SMALL,ALL>::vec from device.cuh), C4 shape: GF(32749), g = 2, 2^26 u16 codes
// per operand, 10% zeros.  Build: make tune   Run: scripts/tune_zech
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device.cuh"

using namespace gfp::dev;
using Z = Zech<true, true>;

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void stage(uint16_t *dst, const uint16_t *src, int entries) {
    const uint4 *s = reinterpret_cast<const uint4 *>(src);
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    for (int i = threadIdx.x; i < entries / 8; i += blockDim.x) d[i] = __ldg(s + i);
}

__device__ __forceinline__ void cta_sum(uint64_t v, unsigned long long *out) {
    __shared__ uint64_t red[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)v);
    }
}

// (1) the product's scheme: register ping-pong pipeline of U 16-byte loads per operand
template <int NT, int U>
__global__ void __launch_bounds__(NT) k_ldg(const uint4 *av, const uint4 *bv, int64_t nvec, KParams K,
                                            const uint16_t *tabg, unsigned long long *out) {
    extern __shared__ __align__(16) uint16_t tab[];
    Z::Acc acc;
    Z::init(acc);
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    uint4 ca[U], cb[U], na[U], nb[U];
    bool have = i0 + (U - 1) * NT < nvec;
    if (have)
        for (int u = 0; u < U; ++u) ca[u] = ld_stream(av + i0 + u * NT), cb[u] = ld_stream(bv + i0 + u * NT);
    stage(tab, tabg, 65536);
    __syncthreads();
    auto one = [&](uint4 (&cx)[U], uint4 (&cy)[U], uint4 (&xa)[U], uint4 (&xb)[U]) {
        const int64_t nx = i0 + step;
        const bool more = nx + (U - 1) * NT < nvec;
        if (more)
#pragma unroll
            for (int u = 0; u < U; ++u) xa[u] = ld_stream(av + nx + u * NT), xb[u] = ld_stream(bv + nx + u * NT);
#pragma unroll
        for (int u = 0; u < U; ++u) Z::vec(acc, cx[u], cy[u], K, tab);
        i0 = nx;
        have = more;
    };
    while (have) {
        one(ca, cb, na, nb);
        if (!have) break;
        one(na, nb, ca, cb);
    }
    for (int u = 0; u < U; ++u)
        if (i0 + u * NT < nvec) Z::vec(acc, ld_stream(av + i0 + u * NT), ld_stream(bv + i0 + u * NT), K, tab);
    cta_sum(Z::finish(acc, K), out);
}

// (2) TMA ring: thread 0 streams CH-byte chunks of both operands into STAGES shared-memory slots with
// cp.async.bulk (mbarrier transaction counts); every thread consumes its vectors of a chunk from shared
// memory; a CTA barrier per chunk frees the slot for the next bulk copy.
template <int NT, int STAGES, int CH>
__global__ void __launch_bounds__(NT) k_tma(const uint4 *av, const uint4 *bv, int64_t nvec, KParams K,
                                            const uint16_t *tabg, unsigned long long *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint16_t *tab = reinterpret_cast<uint16_t *>(sm);
    uint4 *bufA = reinterpret_cast<uint4 *>(sm + 131072);
    uint4 *bufB = reinterpret_cast<uint4 *>(sm + 131072 + STAGES * CH);
    __shared__ __align__(8) uint64_t full[STAGES];
    constexpr int VPC = CH / 16;
    const int64_t nchunks = nvec / VPC;
    auto issue = [&](int64_t c, int s) {
        const uint32_t mb = smem_addr(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(2 * CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_addr(bufA + s * VPC)), "l"(av + c * VPC), "r"(CH), "r"(mb) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_addr(bufB + s * VPC)), "l"(bv + c * VPC), "r"(CH), "r"(mb) : "memory");
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int s = 0; s < STAGES; ++s)
            if (blockIdx.x + (int64_t)s * gridDim.x < nchunks) issue(blockIdx.x + (int64_t)s * gridDim.x, s);
    }
    stage(tab, tabg, 65536);
    __syncthreads();
    Z::Acc acc;
    Z::init(acc);
    int it = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % STAGES;
        const uint32_t parity = (it / STAGES) & 1, mb = smem_addr(&full[s]);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(mb), "r"(parity) : "memory");
#pragma unroll
        for (int v = threadIdx.x; v < VPC; v += NT) Z::vec(acc, bufA[s * VPC + v], bufB[s * VPC + v], K, tab);
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t nc = c + (int64_t)STAGES * gridDim.x;
            if (nc < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;");
                issue(nc, s);
            }
        }
    }
    for (int64_t v = nchunks * VPC + (int64_t)blockIdx.x * NT + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * NT)
        Z::vec(acc, av[v], bv[v], K, tab);
    cta_sum(Z::finish(acc, K), out);
}

template <class F>
double time_it(F launch, int reps, unsigned long long *d_out, unsigned long long *res) {
    CK(cudaMemset(d_out, 0, 8));
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(res, d_out, 8, cudaMemcpyDeviceToHost));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
}

int main() {
    const uint32_t p = 32749, qbar = p - 1;
    const int64_t n = 1ll << 26, nvec = n / 8;
    // antilog table, SMALL layout: index s in [0, 2 qbar] -> 2^s mod p; 0xFFFF -> 0 (zero sentinel)
    std::vector<uint16_t> tab(65536, 0);
    uint32_t g = 1;
    for (uint32_t s = 0; s <= 2 * qbar; ++s) {
        tab[s] = (uint16_t)g;
        g = (g * 2) % p;
    }
    tab[0xFFFF] = 0;
    std::vector<uint16_t> a(n), b(n);
    uint64_t st = 0x0404008;
    auto rnd = [&]() { st += 0x9E3779B97F4A7C15ull; uint64_t z = st; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                       z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); };
    for (int64_t i = 0; i < n; ++i) {
        a[i] = rnd() % 10 == 0 ? 0 : (uint16_t)(1 + rnd() % qbar);
        b[i] = rnd() % 10 == 0 ? 0 : (uint16_t)(1 + rnd() % qbar);
    }
    uint16_t *da, *db, *dt;
    unsigned long long *d_out;
    CK(cudaMalloc(&da, n * 2));
    CK(cudaMalloc(&db, n * 2));
    CK(cudaMalloc(&dt, 65536 * 2));
    CK(cudaMalloc(&d_out, 8));
    CK(cudaMemcpy(da, a.data(), n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b.data(), n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dt, tab.data(), 65536 * 2, cudaMemcpyHostToDevice));
    KParams K{};
    K.p = p;
    K.mu = UINT64_MAX / p;
    K.qbar = qbar;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const auto av = reinterpret_cast<const uint4 *>(da), bv = reinterpret_cast<const uint4 *>(db);
    unsigned long long ref = 0, res = 0;
    const double bytes = 4.0 * n;
    {
        CK(cudaFuncSetAttribute(k_ldg<1024, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
        double ms = time_it([&] { k_ldg<1024, 2><<<sms, 1024, 131072>>>(av, bv, nvec, K, dt, d_out); }, 30, d_out, &ref);
        printf("%-36s %8.2f us  %7.1f GB/s  sum %llu\n", "ldg pipeline NT=1024 U=2", ms * 1e3, bytes / ms / 1e6, ref);
    }
#define TMA(NT, ST, CH)                                                                                           \
    {                                                                                                             \
        const size_t smem = 131072 + 2 * (size_t)(ST) * (CH);                                                    \
        CK(cudaFuncSetAttribute(k_tma<NT, ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
        double ms = time_it([&] { k_tma<NT, ST, CH><<<sms, NT, smem>>>(av, bv, nvec, K, dt, d_out); }, 30, d_out, &res); \
        printf("tma NT=%4d stages=%d chunk=%5dB       %8.2f us  %7.1f GB/s  %s\n", NT, ST, CH, ms * 1e3,         \
               bytes / ms / 1e6, res == ref ? "ok" : "MISMATCH");                                                 \
    }
    TMA(1024, 3, 16384)
    TMA(1024, 2, 16384)
    TMA(1024, 4, 8192)
    TMA(1024, 6, 8192)
    TMA(512, 3, 16384)
    TMA(1024, 3, 12288)
    return 0;
}
