// gather_peak.cu -- standalone B200 measurement (not part of the product): the achievable rate of random
// 16-bit shared-memory lookups, the binding ceiling of the Zech matrix-vector product and of the Zech
// conversions.  The analogue of MEASURED_PEAKS.json's copy bandwidth for HBM: a measured peak,
// not a datasheet figure.
//
//   k_lookup : every thread walks an LCG in registers (1 IMAD + 2 ALU per code), looks the code up in a
//              64 KB u16 table in shared memory and sums the values -- no global memory at all.  Reports
//              lookups/s and L1TEX data-pipe wavefronts per SM per clock, using the expected wavefronts of a
//              warp-wide random lookup (the most distinct 32-bit words one of the 32 banks serves, E = 3.52
//              for 32 active lanes, computed here by simulation of the same codes).
//   k_stream : the same plus the Zech batch's A stream (a 16-byte LDG per 8 lookups, L1::no_allocate), to
//              show what streaming A through the same pipe costs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gather_peak scripts/gather_peak.cu
// Run:   scripts/gather_peak            (one B200; prints one line per kernel and occupancy)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

constexpr uint32_t kQbar = 32748;            // GF(32749): codes in [0, qbar]
constexpr uint32_t kA = 1664525u, kC = 1013904223u;  // LCG (Numerical Recipes constants)

__device__ __forceinline__ uint32_t code_of(uint32_t x) { return min(x >> 17, kQbar); }

template <int NT, int ITERS>
__global__ void __launch_bounds__(NT, 1) k_lookup(const uint16_t *tabg, unsigned long long *out) {
    extern __shared__ __align__(16) uint16_t tab[];
    for (int i = threadIdx.x; i < (int)(kQbar + 8) / 8; i += NT)
        reinterpret_cast<uint4 *>(tab)[i] = reinterpret_cast<const uint4 *>(tabg)[i];
    __syncthreads();
    uint32_t x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (blockIdx.x * NT + threadIdx.x) * 2654435761u + j * 40503u;
    uint32_t s0 = 0, s1 = 0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x[j] = x[j] * kA + kC;
            const uint32_t v = tab[code_of(x[j])];
            if (j & 1) s1 += v; else s0 += v;
        }
    }
    if (s0 + s1 == 0xFFFFFFFFu) atomicAdd(out, 1ull);  // keeps the sums live
}

template <int NT, int ITERS>
__global__ void __launch_bounds__(NT, 1) k_stream(const uint16_t *tabg, const uint4 *A, int64_t nvec,
                                                   unsigned long long *out) {
    extern __shared__ __align__(16) uint16_t tab[];
    for (int i = threadIdx.x; i < (int)(kQbar + 8) / 8; i += NT)
        reinterpret_cast<uint4 *>(tab)[i] = reinterpret_cast<const uint4 *>(tabg)[i];
    __syncthreads();
    uint32_t x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (blockIdx.x * NT + threadIdx.x) * 2654435761u + j * 40503u;
    uint32_t s0 = 0, s1 = 0, sa = 0;
    int64_t v = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int it = 0; it < ITERS; ++it) {
        uint4 a;
        asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
            : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(A + v));
        v += stride;
        if (v >= nvec) v -= nvec;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x[j] = x[j] * kA + kC;
            const uint32_t val = tab[code_of(x[j])];
            if (j & 1) s1 += val; else s0 += val;
        }
        sa += a.x ^ a.y ^ a.z ^ a.w;
    }
    if (s0 + s1 + sa == 0xFFFFFFFFu) atomicAdd(out, 1ull);
}

// expected wavefronts of one warp-wide lookup of the codes thread t's LCG produces (the same sequence)
static double expected_wavefronts(int NT, int grid, int samples) {
    double tot = 0;
    int n = 0;
    for (int w = 0; w < samples; ++w) {
        const int warp = (w * 7919) % (grid * NT / 32);
        uint32_t x[32];
        for (int l = 0; l < 32; ++l) x[l] = (uint32_t)(warp * 32 + l) * 2654435761u + 0 * 40503u;
        for (int it = 0; it < 16; ++it) {
            std::vector<std::set<uint32_t>> bank(32);
            for (int l = 0; l < 32; ++l) {
                x[l] = x[l] * kA + kC;
                const uint32_t c = std::min(x[l] >> 17, kQbar);
                bank[(c >> 1) & 31].insert(c >> 1);
            }
            size_t mx = 0;
            for (auto &b : bank) mx = std::max(mx, b.size());
            tot += (double)mx;
            ++n;
        }
    }
    return tot / n;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    std::vector<uint16_t> h(kQbar + 8);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 7 + 1);
    uint16_t *tab = nullptr;
    unsigned long long *out = nullptr;
    CK(cudaMalloc(&tab, h.size() * 2));
    CK(cudaMemcpy(tab, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, 8));
    const int64_t nvec = (int64_t)1 << 27;  // 2 GiB of 16-byte vectors streamed cyclically
    uint4 *A = nullptr;
    CK(cudaMalloc(&A, nvec * 16));
    CK(cudaMemset(A, 1, nvec * 16));
    constexpr int NT = 1024, ITERS = 4096;
    const size_t smem = (kQbar + 8) * 2;
    CK(cudaFuncSetAttribute(k_lookup<NT, ITERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_stream<NT, ITERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double E = expected_wavefronts(NT, sms, 512);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int k = 0; k < 2; ++k) {
        for (int rep = 0; rep < 6; ++rep) {
            CK(cudaEventRecord(e0));
            if (k == 0) k_lookup<NT, ITERS><<<sms, NT, smem>>>(tab, out);
            else k_stream<NT, ITERS><<<sms, NT, smem>>>(tab, A, nvec, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double lookups = (double)sms * NT * ITERS * 8;
            const double warp_lookups = lookups / 32;
            const double wf = warp_lookups * E + (k == 1 ? (double)sms * NT * ITERS * 16 / 128 : 0.0);
            const double per_sm_clk = wf / sms / (ms * 1e-3) / 1e9;  // wavefronts per SM per ns
            printf("%s rep %d: %.3f ms, %.3f T lookups/s, E = %.3f wavefronts per warp lookup, "
                   "%.3f G wavefronts per SM per second (%.3f per clock at the %d MHz max clock)%s\n",
                   k == 0 ? "k_lookup (random u16 lookups, no global memory)" : "k_stream (+ a 16-byte LDG per 8 lookups)",
                   rep, ms, lookups / (ms * 1e-3) / 1e12, E, per_sm_clk, per_sm_clk / (clk_khz * 1e-6), clk_khz / 1000,
                   k == 1 ? " (stream wavefronts counted at 1 per 128 B)" : "");
        }
    }
    return 0;
}
