// device.cuh -- device-side building blocks for sm_100a: streaming loads, exact reductions, and one
// accumulation policy per representation of arXiv cs/0404008 sec. 2.
//
// A policy R provides
//   elem, W              element type, elements per 16-byte vector
//   Acc                  per-thread accumulator state
//   init(Acc&)           zero
//   vec(Acc&, x, y, K)   accumulate the W products of two 16-byte vectors
//   term(Acc&, a, b, K)  accumulate one product (head / tail / unaligned elements)
//   finish(Acc&, K)      -> uint64 contribution that can be summed across threads without wrap:
//                          the raw sum when the host proved the grand total fits ("ALL" modes),
//                          else a residue in [0, p)
// K is the kernel-constant block (KParams) with p and the precomputed constants of numtheory.cpp.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "params.h"



namespace gfp {
namespace dev {


// ------------------------------------------------------------------------------ memory access
// 16-byte streaming load: read-only path, no L1 allocation (each byte is used exactly once).
__device__ __forceinline__ uint4 ld_stream(const void *ptr) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr));
    return r;
}

// ------------------------------------------------------------------------------ exact reductions
// x mod p for any 64-bit x and p < 2^62: q = floor(x * mu / 2^64) is floor(x/p) - {0,1,2}.
__device__ __forceinline__ uint64_t mod_p(uint64_t x, uint64_t p, uint64_t mu) {
    uint64_t q = __umul64hi(x, mu);
    uint64_t r = x - q * p;
    r = r >= p ? r - p : r;
    r = r >= p ? r - p : r;
    return r;
}

// x mod p for a 32-bit x (p < 2^16 in the m = 32 strategies): q = floor(x mu32 / 2^32) >= floor(x/p) - 2.
__device__ __forceinline__ uint32_t mod_p32(uint32_t x, uint32_t p, uint32_t mu32) {
    uint32_t q = __umulhi(x, mu32);
    uint32_t r = x - q * p;
    r = r >= p ? r - p : r;
    r = r >= p ? r - p : r;
    return r;
}

// Montgomery reduction (sec. 2.2) with B = 2^32: U = T n_im mod B, returns (T + U p) / B,
// which is T B^{-1} mod p up to a multiple of p.  The caller guarantees T + U p < 2^64.
__device__ __forceinline__ uint32_t redc(uint64_t T, uint32_t p, uint32_t n_im) {
    uint32_t U = (uint32_t)T * n_im;
    return (uint32_t)((T + (uint64_t)U * p) >> 32);
}

// NTL's floating point reduction (sec. 2.3, listing P:112-117): T -= floor(T*invP)*P; one fix-up.
// Every intermediate is an integer below 2^53, so each step is exact (reading G8).
__device__ __forceinline__ double ntl_reduce(double T, double P, double invP) {
    double q = floor(__dmul_rn(T, invP));
    T = __fma_rn(-q, P, T);
    if (T >= P)
        T -= P;
    else if (T < 0.0)
        T += P;
    return T;
}

// ------------------------------------------------------------------------------ carry-flag accumulation
// The carry word of sec. 3.3 ("division on demand") with the hardware carry flag: the product x y
// is added to the accumulator with add-with-carry instructions and the carry out of the top word is counted
// in c -- no compare, no branch, no correction inside the loop; the thread's value c 2^m + s is reduced once
// at the end (c (2^m mod p) + s).  m = 64: s += x y as mad.lo.cc / madc.hi.cc on the two 32-bit halves of s
// (the multiply and the 64-bit add are one pair of multiply-adds), then c += carry.
__device__ __forceinline__ void mac_carry64(uint64_t &s, uint32_t &c, uint32_t x, uint32_t y) {
    asm("{\n\t.reg .u32 lo, hi;\n\t"
        "mov.b64 {lo, hi}, %0;\n\t"
        "mad.lo.cc.u32 lo, %2, %3, lo;\n\t"
        "madc.hi.cc.u32 hi, %2, %3, hi;\n\t"
        "addc.u32 %1, %1, 0;\n\t"
        "mov.b64 %0, {lo, hi};\n\t}"
        : "+l"(s), "+r"(c) : "r"(x), "r"(y));
}
// m = 32 (the product fits 32 bits: (p-1)^2 < 2^32, host-checked): s += x y with carry out, c += carry.
__device__ __forceinline__ void mac_carry32(uint32_t &s, uint32_t &c, uint32_t x, uint32_t y) {
    asm("mad.lo.cc.u32 %0, %2, %3, %0;\n\t"
        "addc.u32 %1, %1, 0;"
        : "+r"(s), "+r"(c) : "r"(x), "r"(y));
}

// ------------------------------------------------------------------------------ policies
enum ClassicalMode { CL_ALL = 0, CL_THREAD = 1, CL_OVERFLOW = 2 };

// Classical Z/pZ, u32 storage (sec. 2.1).  Products a*b < 2^64 are added to a u64 with no
// remainder (AXPY with the remainder delayed, sec. 3.1).  CL_OVERFLOW: the paper's overflow
// detection trick (sec. 3.3): sum += product; if (sum < product) sum += CORR.
template <int MODE>
struct ClassicalU32 {
    using elem = uint32_t;
    static constexpr int W = 4;
    static constexpr bool kTable = false;
    struct Acc { uint64_t s; };
    __device__ __forceinline__ static void init(Acc &A) { A.s = 0; }
    __device__ __forceinline__ static void term(Acc &A, uint32_t x, uint32_t y, const KParams &K,
                                                const uint16_t * = nullptr) {
        uint64_t prod = (uint64_t)x * y;
        if (MODE == CL_OVERFLOW) {
            uint64_t s = A.s + prod;
            A.s = s < prod ? s + K.corr : s;
        } else {
            A.s += prod;
        }
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *) {
        term(A, x.x, y.x, K);
        term(A, x.y, y.y, K);
        term(A, x.z, y.z, K);
        term(A, x.w, y.w, K);
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        return MODE == CL_ALL ? A.s : mod_p(A.s, K.p, K.mu);
    }
};

// Classical Z/pZ, u16 storage (p <= 65521): products < 2^32; CL_ALL or CL_THREAD only.
template <int MODE>
struct ClassicalU16 {
    using elem = uint16_t;
    static constexpr int W = 8;
    static constexpr bool kTable = false;
    struct Acc { uint64_t s; };
    __device__ __forceinline__ static void init(Acc &A) { A.s = 0; }
    __device__ __forceinline__ static void term(Acc &A, uint32_t x, uint32_t y, const KParams &,
                                                const uint16_t * = nullptr) {
        A.s += (uint64_t)(x * y);
    }
    __device__ __forceinline__ static void pair(Acc &A, uint32_t x, uint32_t y) {
        A.s += (uint64_t)((x & 0xFFFFu) * (y & 0xFFFFu));
        A.s += (uint64_t)((x >> 16) * (y >> 16));
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &, const uint16_t *) {
        pair(A, x.x, y.x);
        pair(A, x.y, y.y);
        pair(A, x.z, y.z);
        pair(A, x.w, y.w);
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        return MODE == CL_ALL ? A.s : mod_p(A.s, K.p, K.mu);
    }
};

// Montgomery, B = 2^32 (sec. 2.2 / 3.2.1).  Elements are aB mod p; a product is ab B^2, and KR of
// them are summed before one REDC (sec. 3.2.1: "the reduction can indeed be delayed").
// Each REDC output (< 2p) is in B^1 scale and goes into a separate u64 sum S (reading G6), whose
// residue S mod p is the Montgomery form of the dot.  KR <= the host's mont_k(p).
template <int KR>
struct Montgomery {
    using elem = uint32_t;
    static constexpr int W = 4;
    static constexpr bool kTable = false;
    struct Acc { uint64_t S; };
    __device__ __forceinline__ static void init(Acc &A) { A.S = 0; }
    __device__ __forceinline__ static void term(Acc &A, uint32_t x, uint32_t y, const KParams &K,
                                                const uint16_t * = nullptr) {
        A.S += redc((uint64_t)x * y, (uint32_t)K.p, K.n_im);
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *) {
        const uint32_t p = (uint32_t)K.p;
        if (KR >= 4) {
            uint64_t T = (uint64_t)x.x * y.x;
            T += (uint64_t)x.y * y.y;
            T += (uint64_t)x.z * y.z;
            T += (uint64_t)x.w * y.w;
            A.S += redc(T, p, K.n_im);
        } else if (KR >= 2) {
            uint64_t T0 = (uint64_t)x.x * y.x + (uint64_t)x.y * y.y;
            uint64_t T1 = (uint64_t)x.z * y.z + (uint64_t)x.w * y.w;
            A.S += redc(T0, p, K.n_im);
            A.S += redc(T1, p, K.n_im);
        } else {
            term(A, x.x, y.x, K);
            term(A, x.y, y.y, K);
            term(A, x.z, y.z, K);
            term(A, x.w, y.w, K);
        }
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        return mod_p(A.S, K.p, K.mu);
    }
};

// Floating point (sec. 2.3 / 3.1).  Exact integers in binary64; products are fused into the
// accumulator (exact: every value is an integer below 2^53) and NTL's reduction runs every
// KF terms, KF <= k of Eq. (1) at m = 53.  KF = 0: no reduction until the end of the thread
// (the host proved the thread's whole sum stays below 2^53).
template <int KF>
struct Fp64 {
    using elem = double;
    static constexpr int W = 2;
    static constexpr bool kTable = false;
    struct Acc { double T; };
    __device__ __forceinline__ static void init(Acc &A) { A.T = 0.0; }
    __device__ __forceinline__ static void term(Acc &A, double x, double y, const KParams &K,
                                                const uint16_t * = nullptr) {
        A.T = __fma_rn(x, y, A.T);
        if (KF != 0) A.T = ntl_reduce(A.T, K.pd, K.inv_p);
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 xv, uint4 yv, const KParams &K, const uint16_t *) {
        const double x0 = __hiloint2double(xv.y, xv.x), x1 = __hiloint2double(xv.w, xv.z);
        const double y0 = __hiloint2double(yv.y, yv.x), y1 = __hiloint2double(yv.w, yv.z);
        if (KF == 1) {
            term(A, x0, y0, K);
            term(A, x1, y1, K);
        } else {
            A.T = __fma_rn(x0, y0, A.T);
            A.T = __fma_rn(x1, y1, A.T);
            if (KF != 0) A.T = ntl_reduce(A.T, K.pd, K.inv_p);
        }
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        double T = KF == 0 ? ntl_reduce(A.T, K.pd, K.inv_p) : A.T;
        return (uint64_t)T;
    }
};

// Discrete logarithms (sec. 2.4).  The product of g^i and g^j is g^(i+j): one index addition
// (Table 1 row 1) and one antilog lookup in shared memory gives its classical value
// (< p), which is summed in an integer register with the remainder delayed (reading G11).
// Zero operands (code 0) map the index to the zero sentinel (reading G13).
//   SMALL (2(q-1) <= 65534): index i + j needs no "- qbar" correction; 65536-entry table.
//   LARGE: index folded once by qbar (Table 1's "(- qbar)"), clamped; p-entry table.
// ALL: the grand total fits u64 (host-checked); else each thread reduces its sum.
template <bool SMALL, bool ALL>
struct Zech {
    using elem = uint16_t;
    static constexpr int W = 8;
    static constexpr bool kTable = true;
    struct Acc { uint64_t s; };
    __device__ __forceinline__ static void init(Acc &A) { A.s = 0; }
    __device__ __forceinline__ static uint32_t index(uint32_t i, uint32_t j, uint32_t qbar) {
        if (SMALL) {
            return (i == 0 || j == 0) ? 0xFFFFu : i + j;
        } else {
            uint32_t s = i + j;
            s = s > qbar ? s - qbar : s;
            s = s > qbar ? qbar : s;  // non-canonical codes stay inside the table
            return (i == 0 || j == 0) ? 0u : s;
        }
    }
    __device__ __forceinline__ static uint32_t lookup(uint32_t i, uint32_t j, const KParams &K,
                                                      const uint16_t *tab) {
        return tab[index(i, j, K.qbar)];
    }
    __device__ __forceinline__ static void term(Acc &A, uint32_t i, uint32_t j, const KParams &K,
                                                const uint16_t *tab) {
        A.s += lookup(i, j, K, tab);
    }
    __device__ __forceinline__ static uint32_t pair(uint32_t x, uint32_t y, const KParams &K, const uint16_t *tab) {
        return lookup(x & 0xFFFFu, y & 0xFFFFu, K, tab) + lookup(x >> 16, y >> 16, K, tab);
    }
    // SMALL, two terms per 32-bit word (SWAR): canonical codes are < 2^15, so i + j < 2^16 and
    // v + 0x7FFF < 2^16 never carry across the 16-bit lanes.  Bit 15 of v + 0x7FFF is [v != 0].
    __device__ __forceinline__ static uint32_t pair_swar(uint32_t x, uint32_t y, const uint16_t *tab) {
        const uint32_t s = x + y;                                                  // i + j per lane
        const uint32_t nz = (x + 0x7FFF7FFFu) & (y + 0x7FFF7FFFu) & 0x80008000u;  // both operands nonzero
        const uint32_t keep = (nz >> 15) * 0xFFFFu;                                // lane mask
        const uint32_t idx = s | ~keep;                                            // zero -> sentinel 0xFFFF
        return (uint32_t)tab[idx & 0xFFFFu] + (uint32_t)tab[idx >> 16];
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *tab) {
        uint32_t s;
        if (SMALL)
            s = pair_swar(x.x, y.x, tab) + pair_swar(x.y, y.y, tab) + pair_swar(x.z, y.z, tab) +
                pair_swar(x.w, y.w, tab);
        else
            s = pair(x.x, y.x, K, tab) + pair(x.y, y.y, K, tab) + pair(x.z, y.z, K, tab) + pair(x.w, y.w, K, tab);
        A.s += s;  // 8 values < 2^16: no wrap in 32 bits
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        return ALL ? A.s : mod_p(A.s, K.p, K.mu);
    }
};


// Centered representation (sec. 3.2.2): residues stored between -h and h, h = (p-1)/2, as
// int16 / int32 / binary64; products |ab| <= h^2 summed in a signed accumulator, blocks of lambda_c
// products with lambda_c h^2 + h < 2^(m-1) (the doubled block of P:396-398).
// signed 64-bit T -> residue in [0, p): T + 2^63 is a nonnegative u64, from which 2^63 mod p is removed
__device__ __forceinline__ uint64_t smod_p(int64_t T, const KParams &K) {
    const uint64_t r = mod_p((uint64_t)T ^ 0x8000000000000000ull, K.p, K.mu);
    return r >= K.c63 ? r - K.c63 : r + K.p - K.c63;
}
__device__ __forceinline__ int64_t centered_of(int64_t T, const KParams &K) {
    const uint64_t r = smod_p(T, K);
    return r > (uint64_t)K.half ? (int64_t)r - (int64_t)K.p : (int64_t)r;
}

enum CenteredMode { CE_ALL = 0, CE_THREAD = 1, CE_BLOCKED = 2 };

// int16 / int32 storage, int64 accumulator.  CE_ALL: the host proved n h^2 < 2^63, the raw signed sum is
// returned (two's-complement sums across threads are exact); CE_THREAD: each thread reduces once at the
// end; CE_BLOCKED: reduce to the centered residue every K.kblk = lambda_c products.
template <typename E, int MODE>
struct CenteredI {
    using elem = E;
    static constexpr int W = 16 / sizeof(E);
    static constexpr bool kTable = false;
    struct Acc {
        int64_t s;
        uint32_t cnt;
    };
    __device__ __forceinline__ static void init(Acc &A) {
        A.s = 0;
        A.cnt = 0;
    }
    __device__ __forceinline__ static void term(Acc &A, int32_t x, int32_t y, const KParams &K,
                                                const uint16_t * = nullptr) {
        if (MODE == CE_BLOCKED) {
            if (A.cnt >= K.kblk) {
                A.s = centered_of(A.s, K);
                A.cnt = 0;
            }
            ++A.cnt;
        }
        A.s += (int64_t)x * y;
    }
    __device__ __forceinline__ static void raw(Acc &A, uint4 x, uint4 y) {
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if constexpr (sizeof(E) == 2) {  // two int16 lanes: |lo lo' + hi hi'| <= 2 h^2 < 2^31
                const int32_t xl = (int32_t)(xs[i] << 16) >> 16, xh = (int32_t)xs[i] >> 16;
                const int32_t yl = (int32_t)(ys[i] << 16) >> 16, yh = (int32_t)ys[i] >> 16;
                A.s += (int64_t)(xl * yl + xh * yh);
            } else {
                A.s += (int64_t)(int32_t)xs[i] * (int32_t)ys[i];
            }
        }
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *) {
        if (MODE == CE_BLOCKED) {
            if (K.kblk >= (uint64_t)W) {  // bookkeeping once per vector: close the block before it overflows
                if (A.cnt + W > K.kblk) {
                    A.s = centered_of(A.s, K);
                    A.cnt = 0;
                }
                raw(A, x, y);
                A.cnt += W;
            } else {
                const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if constexpr (sizeof(E) == 2) {
                        term(A, (int32_t)(xs[i] << 16) >> 16, (int32_t)(ys[i] << 16) >> 16, K);
                        term(A, (int32_t)xs[i] >> 16, (int32_t)ys[i] >> 16, K);
                    } else {
                        term(A, (int32_t)xs[i], (int32_t)ys[i], K);
                    }
                }
            }
            return;
        }
        raw(A, x, y);
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        return MODE == CE_ALL ? (uint64_t)A.s : smod_p(A.s, K);
    }
};

// binary64 storage: T = fma(x, y, T) is exact while |T| < 2^53; every KF products the centered
// reduction T -= rint(T invP) P (exact by FMA; the quotient is within 1 of round(T/p)) and one +-P
// fix-up bring T back to [-h, h].  KF = 0: no reduction before the end of the thread.
__device__ __forceinline__ double centered_reduce(double T, const KParams &K) {
    const double q = rint(__dmul_rn(T, K.inv_p));
    T = __fma_rn(-q, K.pd, T);
    if (T > K.hd)
        T -= K.pd;
    else if (T < -K.hd)
        T += K.pd;
    return T;
}

template <int KF>
struct Fp64C {
    using elem = double;
    static constexpr int W = 2;
    static constexpr bool kTable = false;
    struct Acc {
        double T;
        int c;
    };
    __device__ __forceinline__ static void init(Acc &A) {
        A.T = 0.0;
        A.c = 0;
    }
    __device__ __forceinline__ static void term(Acc &A, double x, double y, const KParams &K,
                                                const uint16_t * = nullptr) {
        if (KF != 0 && A.c >= KF) {
            A.T = centered_reduce(A.T, K);
            A.c = 0;
        }
        A.T = __fma_rn(x, y, A.T);
        ++A.c;
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 xv, uint4 yv, const KParams &K, const uint16_t *) {
        const double x0 = __hiloint2double(xv.y, xv.x), x1 = __hiloint2double(xv.w, xv.z);
        const double y0 = __hiloint2double(yv.y, yv.x), y1 = __hiloint2double(yv.w, yv.z);
        if (KF == 1) {
            term(A, x0, y0, K);
            term(A, x1, y1, K);
            return;
        }
        if (KF != 0 && A.c + 2 > KF) {  // close the block before it would exceed KF products
            A.T = centered_reduce(A.T, K);
            A.c = 0;
        }
        A.T = __fma_rn(x0, y0, A.T);
        A.T = __fma_rn(x1, y1, A.T);
        A.c += 2;
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        return smod_p((int64_t)A.T, K);  // |T| < 2^53: an exact integer
    }
};

// Pure-Zech arithmetic (sec. 2.4, Table 1).  A nonzero element
// g^e is held as v = S e with e in [0, qbar] (e = qbar is g^0 again: the code qbar of P:126-131), the
// zero element as kZ.  S = 2 makes v a byte offset into the u16 table (one register + the table base
// per address); S = 1 when 2 qbar does not fit the u16 entries.  With q = S qbar:
//   multiplication  g^i * g^j:  v = S (i + j) (- q)                           (Table 1 row 1)
//   addition        g^s + g^c = g^s (1 + g^(c - s)),  k = c - s (+ q),
//                   v = s + delta[k] (- q), delta[k] = S log(1 + g^k)           (Table 1 "Addition")
// with delta the t_plus1 table in scaled exponent form (numtheory.h), 0xFFFF where 1 + g^k = 0.
// Each "(+/- q)" test is one unsigned min: v = min(v, v - q) or min(k, k + q).
namespace zadd {
template <int S>
struct Ops {
    static constexpr uint32_t kZ = 0u - (uint32_t)S;  // the zero element (-S: index math stays in the table)
    static constexpr uint32_t kDZero = 0xFFFFu;        // delta sentinel: 1 + g^k = 0 (odd: never a scaled delta)

    __device__ __forceinline__ static uint32_t fold(uint32_t v, uint32_t q) { return min(v, v - q); }
    __device__ __forceinline__ static uint32_t lookup(const uint16_t *delta, uint32_t k) {
        return *reinterpret_cast<const uint16_t *>(reinterpret_cast<const char *>(delta) + k * (2 / S));
    }

    // product of two codes (each in [0, qbar]); a zero operand gives kZ.  Result in [0, q].
    __device__ __forceinline__ static uint32_t mul(uint32_t ci, uint32_t cj, uint32_t q) {
        const uint32_t v = min(fold((uint32_t)S * (ci + cj), q), q);  // clamp: non-canonical codes stay in range
        return (ci == 0 || cj == 0) ? kZ : v;
    }

    // s + c, either operand possibly kZ, values in [0, q].  The index stays in [0, q] in every case
    // (s = kZ: k = c + S; c = kZ: k = q - S - s), so the lookup never leaves the table.
    __device__ __forceinline__ static uint32_t add(uint32_t s, uint32_t c, uint32_t q, const uint16_t *delta) {
        uint32_t k = c - s;
        k = min(k, k + q);
        const uint32_t d = lookup(delta, k);
        uint32_t r = fold(s + d, q);
        r = d == kDZero ? kZ : r;  // g^s (1 + g^k) = 0
        r = s == kZ ? c : r;
        r = c == kZ ? s : r;
        return r;
    }

    // exponent in [1, qbar] (qbar for g^0) of a nonzero value: the Zech code of P:126-131
    __device__ __forceinline__ static uint32_t code_nz(uint32_t v, uint32_t qbar) {
        const uint32_t e = v / S;
        return e == 0 ? qbar : e;
    }
    __device__ __forceinline__ static uint32_t to_code(uint32_t v, uint32_t qbar) { return v == kZ ? 0u : code_nz(v, qbar); }
};
}  // namespace zadd

// ------------------------------------------------------------------------------ explicit strategies
// The paper's section-3 accumulation algorithms, selectable through gfp_dot_ex / gfp_dot_batch_ex for
// classical storage E (u16 / u32) with an m-bit accumulator ACC (u32 or u64).  Every variant is exact;
// the host checks (p-1)^2 < 2^m and each strategy's bound.  Per thread (the paper's loop is per dot):
//   S_DELAYED  sec. 3.1, Eq. (1): no reduction until the end (host: the whole dot has n <= k terms)
//   S_BLOCKED  sec. 3.2 listing P:361-370: reduce every K.kblk = k products (reading G1/G7)
//   S_OVERFLOW sec. 3.3 listing P:414-422: sum += product; if (sum < product) sum += CORR
//   S_HYBRID   sec. 3.4, Eq. (2): one wrap test per block of K.kblk = lambda products,
//              lambda p (p-1) < 2^m; the block sum cannot wrap twice nor re-wrap after CORR
//   S_CARRY    sec. 3.3 with the correction deferred: the carry flag of the m-bit addition is counted in a
//              second word (mac_carry64 / mac_carry32; Acc::cnt holds the count);
//              the thread's value is carry 2^m + sum = carry (2^m mod p) + sum (mod p)
enum Strategy { S_DELAYED = 1, S_BLOCKED = 2, S_OVERFLOW = 3, S_HYBRID = 4, S_CARRY = 6 };

template <typename ACC, typename E, int STRAT>
struct ClassicalS {
    using elem = E;
    static constexpr int W = 16 / sizeof(E);
    static constexpr bool kTable = false;
    struct Acc {
        ACC s, base;
        uint32_t cnt;
    };
    __device__ __forceinline__ static void init(Acc &A) {
        A.s = 0;
        A.base = 0;
        A.cnt = 0;
    }
    __device__ __forceinline__ static ACC corr(const KParams &K) {
        return sizeof(ACC) == 4 ? (ACC)K.corr32 : (ACC)K.corr;
    }
    __device__ __forceinline__ static ACC reduce(ACC s, const KParams &K) {
        if constexpr (sizeof(ACC) == 4)
            return mod_p32(s, (uint32_t)K.p, K.mu32);
        else
            return mod_p(s, K.p, K.mu);
    }
    __device__ __forceinline__ static void term(Acc &A, uint32_t x, uint32_t y, const KParams &K,
                                                const uint16_t * = nullptr) {
        const ACC prod = (ACC)x * (ACC)y;
        if (STRAT == S_DELAYED) {
            A.s += prod;
        } else if (STRAT == S_BLOCKED) {
            if (A.cnt >= K.kblk) {
                A.s = reduce(A.s, K);  // res %= P after each block (G1)
                A.cnt = 0;
            }
            A.s += prod;
            ++A.cnt;
        } else if (STRAT == S_OVERFLOW) {
            A.s += prod;
            if (A.s < prod) A.s += corr(K);
        } else if (STRAT == S_CARRY) {  // carry flag of the m-bit add counted in cnt (the carry word)
            if constexpr (sizeof(ACC) == 8) mac_carry64(A.s, A.cnt, x, y);
            else mac_carry32(A.s, A.cnt, x, y);
        } else {  // S_HYBRID: close the block (its one wrap test) before it would exceed lambda products
            if (A.cnt >= K.kblk) {
                if (A.s < A.base) A.s += corr(K);
                A.base = A.s;
                A.cnt = 0;
            }
            A.s += prod;
            ++A.cnt;
        }
    }
    __device__ __forceinline__ static void raw(Acc &A, uint4 x, uint4 y) {
        if constexpr (sizeof(E) == 4) {
            A.s += (ACC)x.x * (ACC)y.x;
            A.s += (ACC)x.y * (ACC)y.y;
            A.s += (ACC)x.z * (ACC)y.z;
            A.s += (ACC)x.w * (ACC)y.w;
        } else {
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                A.s += (ACC)(xs[i] & 0xFFFFu) * (ACC)(ys[i] & 0xFFFFu);
                A.s += (ACC)(xs[i] >> 16) * (ACC)(ys[i] >> 16);
            }
        }
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *) {
        if ((STRAT == S_BLOCKED || STRAT == S_HYBRID) && K.kblk >= (uint64_t)W) {
            // block bookkeeping once per 16-byte vector: close the block first if W more products
            // would exceed k (BLOCKED: reduce; HYBRID: the one wrap test of the block)
            if (A.cnt + W > K.kblk) {
                if (STRAT == S_BLOCKED) {
                    A.s = reduce(A.s, K);
                } else {
                    if (A.s < A.base) A.s += corr(K);
                    A.base = A.s;
                }
                A.cnt = 0;
            }
            raw(A, x, y);
            A.cnt += W;
            return;
        }
        if (STRAT == S_DELAYED) {
            raw(A, x, y);
            return;
        }
        if constexpr (sizeof(E) == 4) {
            term(A, x.x, y.x, K);
            term(A, x.y, y.y, K);
            term(A, x.z, y.z, K);
            term(A, x.w, y.w, K);
        } else {
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                term(A, xs[i] & 0xFFFFu, ys[i] & 0xFFFFu, K);
                term(A, xs[i] >> 16, ys[i] >> 16, K);
            }
        }
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        if (STRAT == S_CARRY) {  // carry 2^m + s: carry < 2^32 terms per thread, (2^m mod p) < p < 2^32
            const uint64_t c = mod_p((uint64_t)A.cnt, K.p, K.mu) * (sizeof(ACC) == 4 ? (uint64_t)K.corr32 : K.corr);
            return mod_p(mod_p(c, K.p, K.mu) + (uint64_t)reduce(A.s, K), K.p, K.mu);
        }
        if (STRAT == S_HYBRID && A.s < A.base) A.s += corr(K);  // the last, partial block
        return (uint64_t)reduce(A.s, K);
    }
};

// Overflow-Montgomery (sec. 3.3): the products x~ y~ = ab B^2 are summed with the
// overflow trick (CORR = 2^64 mod p); each thread then reduces its sum mod p and applies ONE REDC
// to return to B^1 scale ("one reduction ... to mod out the result, and an additional one to divide
// the element by B").  The result is the Montgomery form of the dot, like Montgomery<KR>.
struct MontgomeryOverflow {
    using elem = uint32_t;
    static constexpr int W = 4;
    static constexpr bool kTable = false;
    struct Acc { uint64_t S; };
    __device__ __forceinline__ static void init(Acc &A) { A.S = 0; }
    __device__ __forceinline__ static void term(Acc &A, uint32_t x, uint32_t y, const KParams &K,
                                                const uint16_t * = nullptr) {
        const uint64_t prod = (uint64_t)x * y;
        A.S += prod;
        if (A.S < prod) A.S += K.corr;
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *) {
        term(A, x.x, y.x, K);
        term(A, x.y, y.y, K);
        term(A, x.z, y.z, K);
        term(A, x.w, y.w, K);
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        const uint32_t p = (uint32_t)K.p;
        const uint32_t r = redc(mod_p(A.S, K.p, K.mu), p, K.n_im);  // T < p <= pB: r <= p
        return r >= p ? r - p : r;
    }
};

// Montgomery with the carry word: products x~ y~ = ab B^2 summed in a u64 with the wraps counted in a
// second word; the thread's value carry 2^64 + S reduces to (carry CORR + S) mod p, then ONE REDC returns
// to B^1 scale (as overflow-Montgomery, with the corrections deferred to the end).
struct MontgomeryCarry {
    using elem = uint32_t;
    static constexpr int W = 4;
    static constexpr bool kTable = false;
    struct Acc { uint64_t S; uint32_t carry; };
    __device__ __forceinline__ static void init(Acc &A) { A.S = 0; A.carry = 0; }
    __device__ __forceinline__ static void term(Acc &A, uint32_t x, uint32_t y, const KParams &,
                                                const uint16_t * = nullptr) {
        mac_carry64(A.S, A.carry, x, y);  // carry flag of the 64-bit add counted (sec. 3.3 carry word)
    }
    __device__ __forceinline__ static void vec(Acc &A, uint4 x, uint4 y, const KParams &K, const uint16_t *) {
        term(A, x.x, y.x, K);
        term(A, x.y, y.y, K);
        term(A, x.z, y.z, K);
        term(A, x.w, y.w, K);
    }
    __device__ __forceinline__ static uint64_t finish(Acc &A, const KParams &K) {
        const uint32_t p = (uint32_t)K.p;
        const uint64_t T = mod_p(mod_p(A.carry, K.p, K.mu) * K.corr + mod_p(A.S, K.p, K.mu), K.p, K.mu);
        const uint32_t r = redc(T, p, K.n_im);  // T < p <= pB: r <= p
        return r >= p ? r - p : r;
    }
};

// ------------------------------------------------------------------------------ combination
__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// Sum over the CTA; the result is valid in thread 0.  `red` holds >= 32 entries.
__device__ __forceinline__ uint64_t block_sum(uint64_t v, uint64_t *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();  // `red` may still be read by a previous call
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = 0;
    if (warp == 0) {
        v = lane < nw ? red[lane] : 0;
        v = warp_sum(v);
    }
    return v;
}

}  // namespace dev
}  // namespace gfp
