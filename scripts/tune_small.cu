// tune_small.cu -- fixed per-launch cost of the single-launch dot (not part of the product).
//
// Times CUDA-graph replays of 200 back-to-back launches of: an empty kernel; the C1-shaped dot
// (n = 100000 u32, classical) with three cross-CTA combine strategies; and the C2 shape
// (n = 10^7 fp64).  Build: make tune   Run: scripts/tune_small
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "device.cuh"

using namespace gfp::dev;

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void empty_kernel(int *) {}

struct WS {
    unsigned long long *partials;
    unsigned int *counter;
    unsigned long long *out;
};

// COMBINE 0: partials[] + threadfence + atomicInc counter + last CTA sums (the library's scheme)
// COMBINE 1: atomicAdd of the CTA sum into one u64 + release/acquire counter; last CTA reads the sum
// COMBINE 2: atomicAdd only (no finalisation: lower bound)
template <class R, int NT, int U, int COMBINE>
__global__ void __launch_bounds__(NT) dotk(const typename R::elem *a, const typename R::elem *b, int64_t n,
                                           KParams K, WS ws) {
    __shared__ uint64_t red[32];
    __shared__ int s_last;
    typename R::Acc acc;
    R::init(acc);
    const int64_t nvec = n / R::W;
    const uint4 *av = reinterpret_cast<const uint4 *>(a), *bv = reinterpret_cast<const uint4 *>(b);
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    for (; i0 + (U - 1) * NT < nvec; i0 += step) {
        uint4 xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xa[u] = ld_stream(av + i0 + u * NT);
            xb[u] = ld_stream(bv + i0 + u * NT);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) R::vec(acc, xa[u], xb[u], K, nullptr);
    }
    for (int u = 0; u < U; ++u)
        if (i0 + u * NT < nvec) R::vec(acc, ld_stream(av + i0 + u * NT), ld_stream(bv + i0 + u * NT), K, nullptr);
    uint64_t v = block_sum(R::finish(acc, K), red);
    if (COMBINE == 0) {
        if (threadIdx.x == 0) {
            ws.partials[blockIdx.x] = v;
            __threadfence();
            unsigned t = atomicAdd(ws.counter, 1u);
            s_last = t == gridDim.x - 1;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        uint64_t s = 0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) s += __ldcg(ws.partials + i);
        s = block_sum(s, red);
        if (threadIdx.x == 0) {
            ws.out[0] = mod_p(s, K.p, K.mu);
            *ws.counter = 0;
        }
    } else if (COMBINE == 1) {
        if (threadIdx.x == 0) {
            atomicAdd(ws.partials, (unsigned long long)v);
            unsigned t;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ws.counter) : "memory");
            if (t == gridDim.x - 1) {
                unsigned long long s;
                asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(s) : "l"(ws.partials) : "memory");
                ws.out[0] = mod_p(s, K.p, K.mu);
                *ws.partials = 0;
                *ws.counter = 0;
            }
        }
    } else {
        if (threadIdx.x == 0) atomicAdd(ws.out, (unsigned long long)v);
    }
}


// software-pipelined variant: loads of step k+1 issued before step k computes
template <class R, int NT, int U>
__global__ void __launch_bounds__(NT) dotk_pipe(const typename R::elem *a, const typename R::elem *b, int64_t n,
                                                KParams K, WS ws) {
    __shared__ uint64_t red[32];
    typename R::Acc acc;
    R::init(acc);
    const int64_t nvec = n / R::W;
    const uint4 *av = reinterpret_cast<const uint4 *>(a), *bv = reinterpret_cast<const uint4 *>(b);
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    uint4 ca[U], cb[U];
    bool have = i0 + (U - 1) * NT < nvec;
    if (have)
        for (int u = 0; u < U; ++u) {
            ca[u] = ld_stream(av + i0 + u * NT);
            cb[u] = ld_stream(bv + i0 + u * NT);
        }
    while (have) {
        const int64_t nx = i0 + step;
        const bool more = nx + (U - 1) * NT < nvec;
        uint4 na[U], nb[U];
        if (more)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                na[u] = ld_stream(av + nx + u * NT);
                nb[u] = ld_stream(bv + nx + u * NT);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) R::vec(acc, ca[u], cb[u], K, nullptr);
        i0 = nx;
        have = more;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ca[u] = na[u];
            cb[u] = nb[u];
        }
    }
    for (int u = 0; u < U; ++u)
        if (i0 + u * NT < nvec) R::vec(acc, ld_stream(av + i0 + u * NT), ld_stream(bv + i0 + u * NT), K, nullptr);
    uint64_t v = block_sum(R::finish(acc, K), red);
    if (threadIdx.x == 0) {
        atomicAdd(ws.partials, (unsigned long long)v);
        unsigned t;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ws.counter) : "memory");
        if (t == gridDim.x - 1) {
            unsigned long long s;
            asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(s) : "l"(ws.partials) : "memory");
            ws.out[0] = mod_p(s, K.p, K.mu);
            *ws.partials = 0;
            *ws.counter = 0;
        }
    }
}

__global__ void fill_u32(uint32_t *x, int64_t n, uint32_t p) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (uint32_t)((i * 2654435761ull) % p);
}
__global__ void fill_f64(double *x, int64_t n, uint32_t p) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (double)((i * 2654435761ull) % p);
}

template <typename L>
float graph_us(L launch, int per_graph = 200) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    launch(s);
    CK(cudaStreamSynchronize(s));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < per_graph; ++i) launch(s);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    for (int r = 0; r < 5; ++r) CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms * 1e3f / (5 * per_graph);
}

int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    WS ws;
    CK(cudaMalloc(&ws.partials, 8 * 8192));
    CK(cudaMalloc(&ws.counter, 64));
    CK(cudaMalloc(&ws.out, 64));
    CK(cudaMemset(ws.partials, 0, 8 * 8192));
    CK(cudaMemset(ws.counter, 0, 64));
    int *dummy;
    CK(cudaMalloc(&dummy, 64));
    printf("empty kernel grid 98    : %6.2f us\n", graph_us([&](cudaStream_t s) { empty_kernel<<<98, 256, 0, s>>>(dummy); }));
    printf("empty kernel grid 888   : %6.2f us\n", graph_us([&](cudaStream_t s) { empty_kernel<<<888, 256, 0, s>>>(dummy); }));
    // C1 shape: classical u32, p = 65521, n = 100000, rotating over 400 copies (> 3x L2)
    const int64_t n1 = 100000, copies = 480;
    uint32_t *A1;
    CK(cudaMalloc(&A1, n1 * 4 * copies));
    fill_u32<<<1184, 256>>>(A1, n1 * copies, 65521);
    KParams K{};
    K.p = 65521;
    K.mu = UINT64_MAX / 65521;
    using C = ClassicalU32<CL_ALL>;
    int it = 0;
    auto c1 = [&](auto kern, int grid) {
        return graph_us([&](cudaStream_t s) {
            const uint32_t *a = A1 + (it++ % copies) * n1;
            kern<<<grid, 256, 0, s>>>(a, a, n1, K, ws);
        });
    };
    for (int grid : {98, 25, 148, 296}) {
        printf("C1 combine0 grid %4d U4 : %6.2f us\n", grid, c1(dotk<C, 256, 4, 0>, grid));
        printf("C1 combine1 grid %4d U4 : %6.2f us\n", grid, c1(dotk<C, 256, 4, 1>, grid));
        printf("C1 combine2 grid %4d U4 : %6.2f us\n", grid, c1(dotk<C, 256, 4, 2>, grid));
    }
    printf("C1 pipe U2 grid 98        : %6.2f us\n", c1(dotk_pipe<C, 256, 2>, 98));
    // C2 shape: fp64, p = 67108859, n = 1e7, 3 copies
    const int64_t n2 = 10000000;
    double *A2, *B2;
    CK(cudaMalloc(&A2, n2 * 8 * 3));
    CK(cudaMalloc(&B2, n2 * 8 * 3));
    fill_f64<<<1184, 256>>>(A2, n2 * 3, 67108859);
    fill_f64<<<1184, 256>>>(B2, n2 * 3, 67108858);
    KParams K2{};
    K2.p = 67108859;
    K2.mu = UINT64_MAX / K2.p;
    K2.pd = 67108859.0;
    K2.inv_p = 1.0 / 67108859.0;
    using F = Fp64<2>;
    auto c2 = [&](auto kern, int grid, int nt) {
        return graph_us([&](cudaStream_t s) {
            const int c = it++ % 3;
            kern<<<grid, nt, 0, s>>>(A2 + c * n2, B2 + c * n2, n2, K2, ws);
        }, 30);
    };
    for (int mult : {1, 2, 4}) {
        printf("C2 NT256 U4 combine0 grid %4d: %6.2f us\n", sms * 6 * mult, c2(dotk<F, 256, 4, 0>, sms * 6 * mult, 256));
        printf("C2 NT256 U4 combine1 grid %4d: %6.2f us\n", sms * 6 * mult, c2(dotk<F, 256, 4, 1>, sms * 6 * mult, 256));
        printf("C2 NT256 U2 combine1 grid %4d: %6.2f us\n", sms * 6 * mult, c2(dotk<F, 256, 2, 1>, sms * 6 * mult, 256));
        printf("C2 NT256 U8 combine1 grid %4d: %6.2f us\n", sms * 6 * mult, c2(dotk<F, 256, 8, 1>, sms * 6 * mult, 256));
        printf("C2 NT512 U4 combine1 grid %4d: %6.2f us\n", sms * 3 * mult, c2(dotk<F, 512, 4, 1>, sms * 3 * mult, 512));
        printf("C2 pipe NT256 U2 grid %4d     : %6.2f us\n", sms * 6 * mult, c2(dotk_pipe<F, 256, 2>, sms * 6 * mult, 256));
        printf("C2 pipe NT256 U4 grid %4d     : %6.2f us\n", sms * 4 * mult, c2(dotk_pipe<F, 256, 4>, sms * 4 * mult, 256));
    }
    printf("ideal C2 at 7.2 TB/s: %.2f us\n", 160e6 / 7.2e12 * 1e6);
    // C3 shape: Montgomery u32 n = 2^28
    const int64_t n3 = 1ll << 28;
    uint32_t *A3, *B3;
    CK(cudaMalloc(&A3, n3 * 4));
    CK(cudaMalloc(&B3, n3 * 4));
    fill_u32<<<1184, 256>>>(A3, n3, 2147483647u);
    fill_u32<<<1184, 256>>>(B3, n3, 2147483646u);
    KParams K3{};
    K3.p = 2147483647u;
    K3.mu = UINT64_MAX / K3.p;
    K3.n_im = 0x80000001u;
    using M = Montgomery<2>;
    auto c3 = [&](auto kern, int grid, int nt) {
        return graph_us([&](cudaStream_t s) { kern<<<grid, nt, 0, s>>>(A3, B3, n3, K3, ws); }, 10);
    };
    printf("C3 NT256 U4 combine1 grid %d : %7.2f us\n", sms * 6, c3(dotk<M, 256, 4, 1>, sms * 6, 256));
    printf("C3 pipe NT256 U2 grid %d     : %7.2f us\n", sms * 6, c3(dotk_pipe<M, 256, 2>, sms * 6, 256));
    printf("C3 pipe NT256 U4 grid %d     : %7.2f us\n", sms * 4, c3(dotk_pipe<M, 256, 4>, sms * 4, 256));
    printf("ideal C3 at 7.2 TB/s: %.2f us\n", 2147483648.0 / 7.2e12 * 1e6);
    return 0;
}
