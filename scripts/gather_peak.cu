// gather_peak.cu -- standalone B200 measurement (not part of the product): the achievable rate of random
// 16-bit shared-memory lookups, the binding ceiling of the Zech matrix-vector product and of the Zech
// conversions.  The analogue of MEASURED_PEAKS.json's copy bandwidth for HBM: a measured peak,
// not a datasheet figure.
//
//   k_lookup : every thread holds 16 hashed codes in registers and, each iteration, looks up code ^ key (a
//              warp-uniform key: the same conflict degree, one LOP per lookup) in a 64 KB u16 table in shared
//              memory and sums the values -- no global memory at all.  Reports
//              lookups/s and L1TEX data-pipe wavefronts per SM per clock, using the expected wavefronts of a
//              warp-wide random lookup (the most distinct 32-bit words one of the 32 banks serves, E ~ 3.4
//              for hashed codes with 10% zeros, computed here by simulation of the same codes; ncu's own
//              wavefront count and pipe utilisation are the primary numbers).
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

constexpr uint32_t kTabEntries = 32768;  // a 64 KB u16 table (GF(32749)'s codes are 15-bit): every 15-bit index is valid
constexpr int kCodes = 16;               // codes held in registers per thread

// a thread's codes: hashed from its global index (independent across lanes: E ~ 3.4 wavefronts per warp lookup,
// as for the Zech matrix-vector product's uniform codes), the zero element (code 0) with probability ~1/10
__host__ __device__ __forceinline__ uint32_t code_of(uint32_t gid, uint32_t j) {
    uint32_t h = (gid * 16u + j) * 0x9E3779B1u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    return (h & 1023u) < 102u ? 0u : (h >> 17);
}
// iteration key, uniform over the warp: index = code ^ key permutes the banks (bank(c ^ k) = bank(c) ^ bank(k)),
// so every iteration's warp lookup has the same conflict degree as the codes themselves, for one LOP per lookup
__host__ __device__ __forceinline__ uint32_t key_of(uint32_t it) { return (it * 2654435761u) >> 17; }

template <int NT, int ITERS>
__global__ void __launch_bounds__(NT, 1) k_lookup(const uint16_t *tabg, unsigned long long *out) {
    extern __shared__ __align__(16) uint16_t tab[];
    for (int i = threadIdx.x; i < (int)kTabEntries / 8; i += NT)
        reinterpret_cast<uint4 *>(tab)[i] = reinterpret_cast<const uint4 *>(tabg)[i];
    __syncthreads();
    const uint32_t gid = blockIdx.x * NT + threadIdx.x;
    uint32_t c[kCodes];
#pragma unroll
    for (int j = 0; j < kCodes; ++j) c[j] = code_of(gid, j);
    uint32_t s0 = 0, s1 = 0;
    for (int it = 0; it < ITERS; ++it) {
        const uint32_t k = key_of(it);
#pragma unroll
        for (int j = 0; j < kCodes; ++j) {
            const uint32_t v = tab[c[j] ^ k];
            if (j & 1) s1 += v; else s0 += v;
        }
    }
    if (s0 + s1 == 0xFFFFFFFFu) atomicAdd(out, 1ull);  // keeps the sums live
}

template <int NT, int ITERS>
__global__ void __launch_bounds__(NT, 1) k_stream(const uint16_t *tabg, const uint4 *A, int64_t nvec,
                                                   unsigned long long *out) {
    extern __shared__ __align__(16) uint16_t tab[];
    for (int i = threadIdx.x; i < (int)kTabEntries / 8; i += NT)
        reinterpret_cast<uint4 *>(tab)[i] = reinterpret_cast<const uint4 *>(tabg)[i];
    __syncthreads();
    const uint32_t gid = blockIdx.x * NT + threadIdx.x;
    uint32_t c[kCodes];
#pragma unroll
    for (int j = 0; j < kCodes; ++j) c[j] = code_of(gid, j);
    uint32_t s0 = 0, s1 = 0, sa = 0;
    int64_t v = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int it = 0; it < ITERS; ++it) {
        const uint32_t k = key_of(it);
#pragma unroll
        for (int h = 0; h < kCodes / 8; ++h) {  // a 16-byte stream load per 8 lookups (the Zech batch's ratio)
            uint4 a;
            asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(A + v));
            v += stride;
            if (v >= nvec) v -= nvec;
#pragma unroll
            for (int j = 8 * h; j < 8 * h + 8; ++j) {
                const uint32_t val = tab[c[j] ^ k];
                if (j & 1) s1 += val; else s0 += val;
            }
            sa += a.x ^ a.y ^ a.z ^ a.w;
        }
    }
    if (s0 + s1 + sa == 0xFFFFFFFFu) atomicAdd(out, 1ull);
}

// the same lookups while each warp streams A through a TMA ring in shared memory instead of LDG: per 8 lookups per
// lane, lane 0 re-arms one stage (512 bytes, the warp's 16 bytes per lane) with cp.async.bulk and an mbarrier
// transaction count; READ = every lane also reads its 16 bytes back (LDS.128), as a consumer would.  Shows what the
// copy engine's shared-memory writes cost the lookups (a TMA-fed A stream for the Zech matrix-vector
// product).
constexpr int kStages = 4;
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NT, int ITERS, bool READ>
__global__ void __launch_bounds__(NT, 1) k_tma(const uint16_t *tabg, const uint4 *A, int64_t nvec,
                                                unsigned long long *out) {
    extern __shared__ __align__(16) uint16_t tab[];
    uint4 *ring = reinterpret_cast<uint4 *>(tab + kTabEntries);  // [warp][stage][32 lanes]
    __shared__ __align__(8) uint64_t mbar[NT / 32][kStages];
    for (int i = threadIdx.x; i < (int)kTabEntries / 8; i += NT)
        reinterpret_cast<uint4 *>(tab)[i] = reinterpret_cast<const uint4 *>(tabg)[i];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nch = nvec / 32;  // 512-byte chunks
    int64_t ch = (int64_t)blockIdx.x * (NT / 32) + w;
    const int64_t cstride = (int64_t)gridDim.x * (NT / 32);
    uint4 *wr = ring + (size_t)w * kStages * 32;
    auto issue = [&](int st) {
        const uint32_t mb = sa(&mbar[w][st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(512));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(wr + st * 32)), "l"(A + ch * 32), "r"(512), "r"(mb) : "memory");
        ch += cstride;
        if (ch >= nch) ch -= nch;
    };
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar[w][st])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int st = 0; st < kStages; ++st) issue(st);
    }
    __syncthreads();
    const uint32_t gid = blockIdx.x * NT + threadIdx.x;
    uint32_t c[kCodes];
#pragma unroll
    for (int j = 0; j < kCodes; ++j) c[j] = code_of(gid, j);
    uint32_t s0 = 0, s1 = 0, sa_ = 0;
    uint32_t step = 0;
    for (int it = 0; it < ITERS; ++it) {
        const uint32_t k = key_of(it);
#pragma unroll
        for (int h = 0; h < kCodes / 8; ++h, ++step) {
            const int st = step % kStages;
            const uint32_t par = (step / kStages) & 1, mb = sa(&mbar[w][st]);
            uint32_t done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(mb), "r"(par) : "memory");
            if (READ) {
                const uint4 a = wr[st * 32 + lane];
                sa_ += a.x ^ a.y ^ a.z ^ a.w;
            }
#pragma unroll
            for (int j = 8 * h; j < 8 * h + 8; ++j) {
                const uint32_t val = tab[c[j] ^ k];
                if (j & 1) s1 += val; else s0 += val;
            }
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(st);
            }
        }
    }
    if (lane == 0)  // drain the ring before the CTA exits
        for (int st = 0; st < kStages; ++st, ++step) {
            const uint32_t par = (step / kStages) & 1, mb = sa(&mbar[w][step % kStages]);
            uint32_t done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(mb), "r"(par) : "memory");
        }
    if (s0 + s1 + sa_ == 0xFFFFFFFFu) atomicAdd(out, 1ull);
}

// expected wavefronts of one warp-wide lookup, over the same codes and keys
static double expected_wavefronts(int NT, int grid, int samples) {
    double tot = 0;
    int n = 0;
    for (int w = 0; w < samples; ++w) {
        const uint32_t warp = (uint32_t)((w * 7919) % (grid * NT / 32));
        for (int j = 0; j < kCodes; ++j)
            for (int it = 0; it < 4; ++it) {
                std::vector<std::set<uint32_t>> bank(32);
                for (uint32_t l = 0; l < 32; ++l) {
                    const uint32_t c = code_of(warp * 32 + l, j) ^ key_of(it);
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
    std::vector<uint16_t> h(kTabEntries);
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
    const size_t smem = kTabEntries * 2;
    CK(cudaFuncSetAttribute(k_lookup<NT, ITERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_stream<NT, ITERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const size_t smem_tma = smem + (size_t)(NT / 32) * kStages * 512;
    CK(cudaFuncSetAttribute(k_tma<NT, ITERS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tma));
    CK(cudaFuncSetAttribute(k_tma<NT, ITERS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tma));
    const double E = expected_wavefronts(NT, sms, 512);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const char *names[4] = {"k_lookup (random u16 lookups, no global memory)", "k_stream (+ a 16-byte LDG per 8 lookups)",
                            "k_tma_read (+ the same bytes by TMA into smem, read back with LDS.128)",
                            "k_tma_noread (+ the same bytes by TMA into smem, not read)"};
    for (int k = 0; k < 4; ++k) {
        for (int rep = 0; rep < 6; ++rep) {
            CK(cudaEventRecord(e0));
            if (k == 0) k_lookup<NT, ITERS><<<sms, NT, smem>>>(tab, out);
            else if (k == 1) k_stream<NT, ITERS><<<sms, NT, smem>>>(tab, A, nvec, out);
            else if (k == 2) k_tma<NT, ITERS, true><<<sms, NT, smem_tma>>>(tab, A, nvec, out);
            else k_tma<NT, ITERS, false><<<sms, NT, smem_tma>>>(tab, A, nvec, out);
            CK(cudaGetLastError());
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double lookups = (double)sms * NT * ITERS * kCodes;
            const double warp_lookups = lookups / 32;
            const double wf = warp_lookups * E + (k >= 1 ? (double)sms * NT * ITERS * (kCodes / 8) * 16 / 128 : 0.0);
            const double per_sm_clk = wf / sms / (ms * 1e-3) / 1e9;  // wavefronts per SM per ns
            printf("%s rep %d: %.3f ms, %.3f T lookups/s, E = %.3f wavefronts per warp lookup, "
                   "%.3f G wavefronts per SM per second (%.3f per clock at the %d MHz max clock)%s\n",
                   names[k],
                   rep, ms, lookups / (ms * 1e-3) / 1e12, E, per_sm_clk, per_sm_clk / (clk_khz * 1e-6), clk_khz / 1000,
                   k >= 1 ? " (stream wavefronts counted at 1 per 128 B)" : "");
        }
    }
    return 0;
}
