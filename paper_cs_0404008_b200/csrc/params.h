// params.h -- the kernel-constant block shared by host launchers and device code (plain C++).
#pragma once
#include <cstdint>

namespace gfp {
namespace dev {

struct KParams {
    uint64_t p;
    uint64_t mu;        // floor((2^64 - 1) / p): Barrett constant for the final reductions
    uint64_t corr;      // 2^64 mod p (sec. 3.3 CORR)
    double pd;          // p as binary64
    double inv_p;       // RN(1/p)
    uint64_t r2;        // Montgomery B^2 mod p
    uint32_t n_im;      // -p^{-1} mod 2^32
    uint32_t qbar;      // Zech q - 1
    const uint16_t *antilog;  // Zech antilog table (global; staged to shared memory by the kernel)
    const uint16_t *logt;     // Zech log table (global; read once by the finaliser)
    uint32_t antilog_entries;
    const uint16_t *zplus1;   // Zech t_plus1 table in exponent form (numtheory.h zech_plus1_delta), global
    const uint16_t *zplus1s;  // small fields: 2 delta[e mod qbar] for e in [0, 2 qbar], then 0 entries
    uint32_t zplus1s_entries; // 65536 (padding: any 16-bit lane sum indexes inside)
    uint32_t zplus1_entries;  // qbar + 1, padded to a multiple of 8
    // explicit-strategy kernels (gfp_dot_ex): block length for BLOCKED / HYBRID, 32-bit constants
    uint64_t kblk;
    uint32_t corr32;    // 2^32 mod p
    uint32_t mu32;      // floor((2^32 - 1) / p)
    // centered representation (sec. 3.2.2)
    int64_t half;       // h = (p - 1) / 2
    double hd;          // h as binary64
    uint64_t c63;       // 2^63 mod p
};

}  // namespace dev
}  // namespace gfp
