// kernels_conv.cu -- representation conversions (to / from Montgomery form, to / from Zech
// codes with the log / antilog tables staged in shared memory, casts, centered) and the tuner's synthetic
// canonical inputs (fill_kernel, F4).
#include "kernels_common.cuh"

namespace gfp {

// ------------------------------------------------------------------------------ conversions
enum ConvOp { C_TO_MONT, C_FROM_MONT, C_TO_ZECH, C_FROM_ZECH_SMALL, C_FROM_ZECH_LARGE, C_CAST, C_TO_CENTERED,
              C_FROM_CENTERED };

template <int OP, typename TI, typename TO>
__device__ __forceinline__ TO conv1(TI v, const KParams &K, const uint16_t *tab) {
    if constexpr (OP == C_TO_MONT) {
        // a -> aB mod p = REDC(a * (B^2 mod p)) (sec. 2.2); T < p^2 <= pB
        uint32_t r = redc((uint64_t)(uint32_t)v * K.r2, (uint32_t)K.p, K.n_im);
        return (TO)(r >= K.p ? r - (uint32_t)K.p : r);
    } else if constexpr (OP == C_FROM_MONT) {
        uint32_t r = redc((uint64_t)(uint32_t)v, (uint32_t)K.p, K.n_im);  // T < p: result <= p
        return (TO)(r >= K.p ? r - (uint32_t)K.p : r);
    } else if constexpr (OP == C_TO_ZECH) {
        uint64_t e = (uint64_t)v;
        return (TO)tab[e < K.p ? e : K.p - 1];  // log table; log[0] = 0
    } else if constexpr (OP == C_FROM_ZECH_SMALL) {
        uint32_t c = (uint32_t)v;
        return (TO)(c == 0 ? 0u : (uint32_t)tab[min(c, K.qbar)]);  // antilog[c] = g^c; only [0, qbar] is staged
    } else if constexpr (OP == C_FROM_ZECH_LARGE) {
        uint32_t c = (uint32_t)v;
        return (TO)tab[c <= K.qbar ? c : K.qbar];  // antilog[0] = 0 sentinel
    } else if constexpr (OP == C_TO_CENTERED) {  // residue r -> r or r - p (sec. 3.2.2)
        const int64_t r = (int64_t)v;
        return (TO)(r > K.half ? r - (int64_t)K.p : r);
    } else if constexpr (OP == C_FROM_CENTERED) {  // c -> c or c + p
        const int64_t c = (int64_t)v;
        return (TO)(c < 0 ? c + (int64_t)K.p : c);
    } else {
        return (TO)v;
    }
}

template <typename T>
__device__ __forceinline__ void load8(const T *p, T (&v)[8]) {
    constexpr int NV = 8 * sizeof(T) / 16;
    uint4 r[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const uint4 *q = reinterpret_cast<const uint4 *>(p) + i;
        if (GFP_CONV_LD == 0)
            r[i] = __ldcs(q);
        else
            asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r[i].x), "=r"(r[i].y), "=r"(r[i].z), "=r"(r[i].w) : "l"(q));
    }
    memcpy(v, r, sizeof(v));
}
template <typename T>
__device__ __forceinline__ void store8(T *p, const T (&v)[8]) {
    constexpr int NV = 8 * sizeof(T) / 16;
    uint4 r[NV];
    memcpy(r, v, sizeof(v));
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        uint4 *q = reinterpret_cast<uint4 *>(p) + i;
        if (GFP_CONV_ST == 0)
            __stcs(q, r[i]);
        else if (GFP_CONV_ST == 1)
            *q = r[i];
        else
            asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};"
                         :: "l"(q), "r"(r[i].x), "r"(r[i].y), "r"(r[i].z), "r"(r[i].w) : "memory");
    }
}

// Elementwise conversion, streaming: each thread holds U chunks of 8 elements (all loads issued before
// any store, so in == out is safe: a chunk is read and written by one thread only), coalesced per u.
template <int OP, typename TI, typename TO, int NT, int U>
__global__ void __launch_bounds__(NT) convert_kernel(const TI *in, TO *out, int64_t n, bool vec_ok, KParams K,
                                                     const uint16_t *table, uint32_t table_entries) {
    extern __shared__ __align__(16) uint16_t s_tab[];
    const int64_t gtid = (int64_t)blockIdx.x * NT + threadIdx.x, gstride = (int64_t)gridDim.x * NT;
    const int64_t nchunk = vec_ok ? n / 8 : 0;
    int64_t c0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    if (GFP_STAGE_EARLY && table != nullptr) stage_table(s_tab, table, table_entries);  // library-owned table
    pdl_wait();  // stream order (launch_pdl; no prefetch: a long stream)
    const uint16_t *tab = nullptr;
    if (table != nullptr) {
        if (!GFP_STAGE_EARLY) stage_table(s_tab, table, table_entries);
        __syncthreads();
        tab = s_tab;
    }
    for (; c0 + (U - 1) * NT < nchunk; c0 += step) {
        TI v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) load8(in + 8 * (c0 + u * NT), v[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            TO w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = conv1<OP, TI, TO>(v[u][i], K, tab);
            store8(out + 8 * (c0 + u * NT), w);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + u * NT;
        if (c < nchunk) {
            TI v[8];
            TO w[8];
            load8(in + 8 * c, v);
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = conv1<OP, TI, TO>(v[i], K, tab);
            store8(out + 8 * c, w);
        }
    }
    for (int64_t i = nchunk * 8 + gtid; i < n; i += gstride) out[i] = conv1<OP, TI, TO>(in[i], K, tab);
    pdl_exit();
}

// ------------------------------------------------------------------------------ synthetic inputs (tuning)
// Canonical elements for the install-time tuner (tune.cpp): residues floor(h p / 2^64) of a SplitMix64
// hash of (seed, i) -- classical residues, Montgomery forms (every residue is one), exact binary64
// integers, or Zech codes in [0, qbar] (code 0, the zero element, with probability 1/p).
__global__ void fill_kernel(void *out, int dtype, uint64_t p, uint64_t seed, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const uint64_t v = __umul64hi(z, p);
        if (dtype == GFP_U16) ((uint16_t *)out)[i] = (uint16_t)v;
        else if (dtype == GFP_U32) ((uint32_t *)out)[i] = (uint32_t)v;
        else ((double *)out)[i] = (double)v;
    }
}

cudaError_t launch_fill(void *out, int dtype, uint64_t p, uint64_t seed, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms(dev) * 8);
    fill_kernel<<<(int)grid, 256, 0, s>>>(out, dtype, p, seed, n);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ conversion launch
template <int OP, typename TI, typename TO>
static cudaError_t launch_conv_t(const KParams &K, const void *in, void *out, int64_t n, const uint16_t *table,
                                 uint32_t entries, cudaStream_t s) {
    // table conversions (Zech): 1024-thread CTAs, so that the one or two CTAs whose 64 KB table fits an SM
    // still keep 2048 threads of loads in flight
    constexpr bool kTab = OP == C_TO_ZECH || OP == C_FROM_ZECH_SMALL || OP == C_FROM_ZECH_LARGE;
    constexpr int NT = kTab ? GFP_CONV_TAB_NT : 256, U = kTab ? GFP_CONV_TAB_U : GFP_CONV_U;
    const size_t smem = table ? (size_t)entries * 2 : 0;
    auto kern = convert_kernel<OP, TI, TO, NT, U>;
    int bps = occupancy(kern, NT, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    const bool vec = ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0);
    int64_t want = (n / 8 + NT * U - 1) / (NT * U) + 1;
    // table-free conversions: one tile per thread over the whole input (B200 A/B, profiles/r01_conv_ab.txt:
    // 6.9 TB/s read + write vs 5.6 TB/s for the resident grid-stride loop); table conversions stage the table
    // once per CTA, so they keep a resident grid
    const bool flat = GFP_CONV_FLAT && table == nullptr;
    int64_t grid = std::min<int64_t>(std::max<int64_t>(want, 1),
                                     flat ? (int64_t)INT32_MAX : (int64_t)GFP_CONV_WAVES * num_sms(dev) * bps);
    cudaError_t e = launch_pdl(kern, dim3((unsigned)grid), dim3(NT), smem, s, (const TI *)in, (TO *)out, n, vec, K,
                               table, entries);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

gfp_status launch_convert(const gfp_info &I, const KParams &K, int dir, gfp_dtype in_dt, const void *in,
                          gfp_dtype out_dt, void *out, int64_t n, cudaStream_t s, cudaError_t *err) {
    // residues side must be integer; representation side must be the rep's dtype
    const gfp_dtype res_dt = dir == 0 ? in_dt : out_dt, rep_dt = dir == 0 ? out_dt : in_dt;
    if (res_dt == GFP_F64 || rep_dt != (gfp_dtype)I.dtype) return GFP_E_UNSUPPORTED;
    if (res_dt == GFP_U16 && I.p > 65536) return GFP_E_UNSUPPORTED;
    *err = cudaSuccess;
    const bool in16 = in_dt == GFP_U16, out16 = out_dt == GFP_U16;
    switch (I.rep) {
    case GFP_REP_CLASSICAL:  // residues are the representation: a dtype cast
        if (in16 && out16) *err = launch_conv_t<C_CAST, uint16_t, uint16_t>(K, in, out, n, nullptr, 0, s);
        else if (in16) *err = launch_conv_t<C_CAST, uint16_t, uint32_t>(K, in, out, n, nullptr, 0, s);
        else if (out16) *err = launch_conv_t<C_CAST, uint32_t, uint16_t>(K, in, out, n, nullptr, 0, s);
        else *err = launch_conv_t<C_CAST, uint32_t, uint32_t>(K, in, out, n, nullptr, 0, s);
        break;
    case GFP_REP_FP64:  // exact integer <-> binary64 casts
        if (dir == 0)
            *err = in16 ? launch_conv_t<C_CAST, uint16_t, double>(K, in, out, n, nullptr, 0, s)
                        : launch_conv_t<C_CAST, uint32_t, double>(K, in, out, n, nullptr, 0, s);
        else
            *err = out16 ? launch_conv_t<C_CAST, double, uint16_t>(K, in, out, n, nullptr, 0, s)
                         : launch_conv_t<C_CAST, double, uint32_t>(K, in, out, n, nullptr, 0, s);
        break;
    case GFP_REP_MONTGOMERY:
        if (in_dt != GFP_U32 || out_dt != GFP_U32) return GFP_E_UNSUPPORTED;
        *err = dir == 0 ? launch_conv_t<C_TO_MONT, uint32_t, uint32_t>(K, in, out, n, nullptr, 0, s)
                        : launch_conv_t<C_FROM_MONT, uint32_t, uint32_t>(K, in, out, n, nullptr, 0, s);
        break;
    case GFP_REP_CENTERED:  // sec. 3.2.2: residues <-> signed values in [-h, h] (int16 / int32 / binary64)
        if (dir == 0) {
            if (out_dt == GFP_F64)
                *err = in16 ? launch_conv_t<C_TO_CENTERED, uint16_t, double>(K, in, out, n, nullptr, 0, s)
                            : launch_conv_t<C_TO_CENTERED, uint32_t, double>(K, in, out, n, nullptr, 0, s);
            else if (out16)
                *err = in16 ? launch_conv_t<C_TO_CENTERED, uint16_t, int16_t>(K, in, out, n, nullptr, 0, s)
                            : launch_conv_t<C_TO_CENTERED, uint32_t, int16_t>(K, in, out, n, nullptr, 0, s);
            else
                *err = in16 ? launch_conv_t<C_TO_CENTERED, uint16_t, int32_t>(K, in, out, n, nullptr, 0, s)
                            : launch_conv_t<C_TO_CENTERED, uint32_t, int32_t>(K, in, out, n, nullptr, 0, s);
        } else {
            if (in_dt == GFP_F64)
                *err = out16 ? launch_conv_t<C_FROM_CENTERED, double, uint16_t>(K, in, out, n, nullptr, 0, s)
                             : launch_conv_t<C_FROM_CENTERED, double, uint32_t>(K, in, out, n, nullptr, 0, s);
            else if (in16)
                *err = out16 ? launch_conv_t<C_FROM_CENTERED, int16_t, uint16_t>(K, in, out, n, nullptr, 0, s)
                             : launch_conv_t<C_FROM_CENTERED, int16_t, uint32_t>(K, in, out, n, nullptr, 0, s);
            else
                *err = out16 ? launch_conv_t<C_FROM_CENTERED, int32_t, uint16_t>(K, in, out, n, nullptr, 0, s)
                             : launch_conv_t<C_FROM_CENTERED, int32_t, uint32_t>(K, in, out, n, nullptr, 0, s);
        }
        break;
    case GFP_REP_ZECH: {
        const uint32_t log_entries = (uint32_t)((I.p + 7) & ~7ull);
        if (dir == 0) {
            *err = in16 ? launch_conv_t<C_TO_ZECH, uint16_t, uint16_t>(K, in, out, n, K.logt, log_entries, s)
                        : launch_conv_t<C_TO_ZECH, uint32_t, uint16_t>(K, in, out, n, K.logt, log_entries, s);
        } else if (zech_small_layout(I.p)) {
            // codes are in [0, qbar]: stage only that prefix of the doubled dot table (64 KB, not 128 KB)
            const uint32_t entries = std::min<uint32_t>(K.antilog_entries, (K.qbar + 1 + 7) & ~7u);
            *err = out16 ? launch_conv_t<C_FROM_ZECH_SMALL, uint16_t, uint16_t>(K, in, out, n, K.antilog, entries, s)
                         : launch_conv_t<C_FROM_ZECH_SMALL, uint16_t, uint32_t>(K, in, out, n, K.antilog, entries, s);
        } else {
            *err = out16 ? launch_conv_t<C_FROM_ZECH_LARGE, uint16_t, uint16_t>(K, in, out, n, K.antilog,
                                                                                  K.antilog_entries, s)
                         : launch_conv_t<C_FROM_ZECH_LARGE, uint16_t, uint32_t>(K, in, out, n, K.antilog,
                                                                                  K.antilog_entries, s);
        }
        break;
    }
    }
    return *err == cudaSuccess ? GFP_OK : GFP_E_CUDA;
}

}  // namespace gfp
