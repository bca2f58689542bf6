// tune_dot.cu -- standalone B200 tuning harness for the streaming dot (not part of the product).
//
// Times variants of the C3 hot loop (Montgomery<2> policy from device.cuh, 2 x 1 GiB u32 operands):
// LDG.128 with different cache hints / unroll / block sizes, and a TMA 1-D bulk-copy pipeline
// (cp.async.bulk + mbarrier, STAGES deep) feeding shared memory.  Every variant's result is
// checked against the first one (mod p).  Build: make tune   Run: scripts/tune_dot [log2 n]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device.cuh"

using namespace gfp::dev;
using R = Montgomery<2>;

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

template <int KIND>
__device__ __forceinline__ uint4 ld(const uint4 *p) {
    uint4 r;
    if (KIND == 0)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (KIND == 1)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else if (KIND == 2)
        r = __ldcs(p);
    else if (KIND == 3)
        asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    else
        r = __ldg(p);
    return r;
}

__device__ __forceinline__ void finish_cta(R::Acc &acc, const KParams &K, unsigned long long *out) {
    __shared__ uint64_t red[32];
    uint64_t v = block_sum(R::finish(acc, K), red);
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)v);
}

template <int NT, int U, int KIND>
__global__ void __launch_bounds__(NT) v_ldg(const uint4 *av, const uint4 *bv, int64_t nvec, KParams K,
                                            unsigned long long *out) {
    R::Acc acc;
    R::init(acc);
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    for (; i0 + (U - 1) * NT < nvec; i0 += step) {
        uint4 xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xa[u] = ld<KIND>(av + i0 + u * NT);
            xb[u] = ld<KIND>(bv + i0 + u * NT);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) R::vec(acc, xa[u], xb[u], K, nullptr);
    }
    for (int u = 0; u < U; ++u)
        if (i0 + u * NT < nvec) R::vec(acc, ld<KIND>(av + i0 + u * NT), ld<KIND>(bv + i0 + u * NT), K, nullptr);
    finish_cta(acc, K, out);
}

// 256-bit loads (LDG.E.256, sm_100): each thread streams 32 contiguous bytes per load and operand.
__device__ __forceinline__ void ld256(const uint4 *p, uint4 &lo, uint4 &hi) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}

template <int NT, int U>
__global__ void __launch_bounds__(NT) v_ldg256(const uint4 *av, const uint4 *bv, int64_t nvec, KParams K,
                                               unsigned long long *out) {
    R::Acc acc;
    R::init(acc);
    const int64_t npair = nvec / 2;  // 32-byte units
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    for (; i0 + (U - 1) * NT < npair; i0 += step) {
        uint4 xa[2 * U], xb[2 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ld256(av + 2 * (i0 + u * NT), xa[2 * u], xa[2 * u + 1]);
            ld256(bv + 2 * (i0 + u * NT), xb[2 * u], xb[2 * u + 1]);
        }
#pragma unroll
        for (int u = 0; u < 2 * U; ++u) R::vec(acc, xa[u], xb[u], K, nullptr);
    }
    for (int u = 0; u < U; ++u)
        if (i0 + u * NT < npair) {
            uint4 a0, a1, b0, b1;
            ld256(av + 2 * (i0 + u * NT), a0, a1);
            ld256(bv + 2 * (i0 + u * NT), b0, b1);
            R::vec(acc, a0, b0, K, nullptr);
            R::vec(acc, a1, b1, K, nullptr);
        }
    finish_cta(acc, K, out);
}

// Contiguous per-CTA ranges instead of grid-stride (each CTA streams one long run of DRAM pages).
template <int NT, int U>
__global__ void __launch_bounds__(NT) v_ldg_block(const uint4 *av, const uint4 *bv, int64_t nvec, KParams K,
                                                  unsigned long long *out) {
    R::Acc acc;
    R::init(acc);
    const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * per, end = min(nvec, beg + per);
    int64_t i0 = beg + threadIdx.x;
    for (; i0 + (U - 1) * NT < end; i0 += NT * U) {
        uint4 xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xa[u] = ld<0>(av + i0 + u * NT);
            xb[u] = ld<0>(bv + i0 + u * NT);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) R::vec(acc, xa[u], xb[u], K, nullptr);
    }
    for (int u = 0; u < U; ++u)
        if (i0 + u * NT < end) R::vec(acc, ld<0>(av + i0 + u * NT), ld<0>(bv + i0 + u * NT), K, nullptr);
    finish_cta(acc, K, out);
}

// TMA 1-D bulk pipeline: thread 0 keeps STAGES chunk pairs in flight into shared memory.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NT, int STAGES, int CH>
__global__ void __launch_bounds__(NT) v_tma(const uint4 *av, const uint4 *bv, int64_t nvec, KParams K,
                                            unsigned long long *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint4 *bufA = reinterpret_cast<uint4 *>(sm);
    uint4 *bufB = reinterpret_cast<uint4 *>(sm + STAGES * CH);
    __shared__ __align__(8) uint64_t full[STAGES];
    constexpr int VPC = CH / 16;  // vectors per chunk
    const int64_t nchunks = nvec / VPC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](int64_t c, int s) {
        uint32_t mb = smem_addr(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(2 * CH));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(bufA + s * VPC)),
            "l"(av + c * VPC), "r"(CH), "r"(mb)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(bufB + s * VPC)),
            "l"(bv + c * VPC), "r"(CH), "r"(mb)
            : "memory");
    };
    int64_t first = blockIdx.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s)
            if (first + (int64_t)s * gridDim.x < nchunks) issue(first + (int64_t)s * gridDim.x, s);
    R::Acc acc;
    R::init(acc);
    int it = 0;
    for (int64_t c = first; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % STAGES;
        const uint32_t parity = (it / STAGES) & 1;
        uint32_t mb = smem_addr(&full[s]);
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(mb), "r"(parity)
                : "memory");
#pragma unroll
        for (int v = threadIdx.x; v < VPC; v += NT) R::vec(acc, bufA[s * VPC + v], bufB[s * VPC + v], K, nullptr);
        __syncthreads();  // stage s fully consumed
        if (threadIdx.x == 0) {
            int64_t nc = c + (int64_t)STAGES * gridDim.x;
            if (nc < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;");
                issue(nc, s);
            }
        }
    }
    // tail vectors (not a full chunk) by the whole grid
    for (int64_t v = nchunks * VPC + (int64_t)blockIdx.x * NT + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * NT)
        R::vec(acc, av[v], bv[v], K, nullptr);
    finish_cta(acc, K, out);
}

__global__ void fill(uint32_t *x, int64_t n, uint32_t p, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        x[i] = (uint32_t)(h % p);
    }
}

template <typename F>
double time_it(F launch, int reps, unsigned long long *d_out, unsigned long long *result) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<float> ts;
    for (int r = 0; r < reps + 3; ++r) {
        CK(cudaMemset(d_out, 0, 8));
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r >= 3) ts.push_back(ms);
    }
    CK(cudaMemcpy(result, d_out, 8, cudaMemcpyDeviceToHost));
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main(int argc, char **argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 28;
    const int64_t n = 1ll << lg, nvec = n / 4;
    const uint32_t p = 2147483647u;
    KParams K{};
    K.p = p;
    K.mu = UINT64_MAX / p;
    K.n_im = 0x80000001u;
    uint32_t *a, *b;
    unsigned long long *d_out;
    CK(cudaMalloc(&a, n * 4));
    CK(cudaMalloc(&b, n * 4));
    CK(cudaMalloc(&d_out, 8));
    fill<<<1184, 256>>>(a, n, p, 1);
    fill<<<1184, 256>>>(b, n, p, 2);
    CK(cudaDeviceSynchronize());
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double bytes = 2.0 * n * 4;
    unsigned long long ref = 0, res = 0;
    bool have_ref = false;
    auto report = [&](const char *name, double ms) {
        const unsigned long long r = res % p;
        if (!have_ref) {
            ref = r;
            have_ref = true;
        }
        printf("%-40s %9.1f us  %7.1f GB/s  %s\n", name, ms * 1e3, bytes / ms / 1e6, r == ref ? "ok" : "MISMATCH");
    };
    const auto av = reinterpret_cast<const uint4 *>(a), bv = reinterpret_cast<const uint4 *>(b);
#define LDG(NT, U, KIND, MULT)                                                                            \
    {                                                                                                     \
        int bps;                                                                                          \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, v_ldg<NT, U, KIND>, NT, 0));               \
        int grid = sms * bps * MULT;                                                                      \
        double ms = time_it([&] { v_ldg<NT, U, KIND><<<grid, NT>>>(av, bv, nvec, K, d_out); }, 20, d_out, &res); \
        char nm[96];                                                                                      \
        snprintf(nm, sizeof nm, "ldg NT=%d U=%d kind=%d grid=%dx%d", NT, U, KIND, sms * bps, MULT);       \
        report(nm, ms);                                                                                   \
    }
    LDG(256, 4, 0, 1)
    LDG(256, 4, 1, 1)
    LDG(256, 4, 2, 1)
    LDG(256, 4, 3, 1)
    LDG(256, 4, 4, 1)
    LDG(256, 2, 0, 1)
    LDG(256, 8, 0, 1)
    LDG(512, 4, 0, 1)
    LDG(1024, 4, 0, 1)
    LDG(128, 4, 0, 1)
    LDG(256, 4, 0, 2)
    LDG(256, 4, 0, 8)
    LDG(256, 16, 0, 1)
    // many waves up to flat (one U-chunk per thread): the conversions gained 24% from a flat grid
    LDG(256, 4, 0, 4)
    LDG(256, 4, 0, 16)
    LDG(256, 4, 0, 80)
    LDG(256, 2, 0, 80)
    LDG(256, 1, 0, 160)
    LDG(512, 4, 0, 80)
    // waves x unroll x block (second pass)
    LDG(256, 2, 0, 4)
    LDG(256, 8, 0, 4)
    LDG(256, 8, 0, 16)
    LDG(256, 2, 0, 16)
    LDG(512, 4, 0, 4)
    LDG(512, 4, 0, 16)
    LDG(128, 4, 0, 16)
    LDG(256, 4, 0, 32)
    LDG(256, 4, 4, 16)
    LDG(256, 4, 2, 16)
#define LDG256(NT, U)                                                                                     \
    {                                                                                                     \
        int bps;                                                                                          \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, v_ldg256<NT, U>, NT, 0));                  \
        int grid = sms * bps;                                                                             \
        double ms = time_it([&] { v_ldg256<NT, U><<<grid, NT>>>(av, bv, nvec, K, d_out); }, 20, d_out, &res); \
        char nm[96];                                                                                      \
        snprintf(nm, sizeof nm, "ldg256 NT=%d U=%d grid=%d", NT, U, grid);                               \
        report(nm, ms);                                                                                   \
    }
    LDG256(256, 1)
    LDG256(256, 2)
    LDG256(256, 4)
    LDG256(512, 2)
    LDG256(128, 4)
    LDG(256, 4, 0, 1)
    {
        int bps;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, v_ldg_block<256, 4>, 256, 0));
        int grid = sms * bps;
        double ms = time_it([&] { v_ldg_block<256, 4><<<grid, 256>>>(av, bv, nvec, K, d_out); }, 20, d_out, &res);
        report("ldg contiguous-per-CTA NT=256 U=4", ms);
    }
#define TMA(NT, ST, CH)                                                                                     \
    {                                                                                                       \
        size_t smem = 2 * (size_t)ST * CH;                                                                  \
        CK(cudaFuncSetAttribute(v_tma<NT, ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        int bps;                                                                                            \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, v_tma<NT, ST, CH>, NT, smem));               \
        int grid = sms * bps;                                                                               \
        double ms = time_it([&] { v_tma<NT, ST, CH><<<grid, NT, smem>>>(av, bv, nvec, K, d_out); }, 20, d_out, &res); \
        char nm[96];                                                                                        \
        snprintf(nm, sizeof nm, "tma NT=%d stages=%d chunk=%dB bps=%d", NT, ST, CH, bps);                   \
        report(nm, ms);                                                                                     \
    }
    TMA(256, 4, 8192)
    TMA(256, 4, 16384)
    TMA(256, 8, 8192)
    TMA(512, 4, 16384)
    TMA(256, 3, 32768)
    TMA(128, 4, 8192)
    TMA(256, 6, 4096)
    return 0;
}
