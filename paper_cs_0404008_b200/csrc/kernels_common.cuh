// kernels_common.cuh -- shared by the kernel translation units (kernels_dot.cu: single dots, the pure-Zech dot,
// finalize, the dot planner; kernels_batch.cu: the batched / matrix-vector kernels; kernels_conv.cu:
// representation conversions and the tuner's input fill): the policy enumeration, output encoding, the fused
// multi-GPU exchange, table staging, programmatic-dependent-launch helpers, the tuning knobs, the launch helpers
// and the explicit-strategy policy tables.  Device functions and templates only (plus inline host helpers), so
// every translation unit compiles on its own (make -j).
#pragma once
#include <algorithm>
#include <mutex>
#include <string>
#include <type_traits>
#include <unordered_map>

#include "device.cuh"
#include "internal.h"
#include "numtheory.h"

namespace gfp {

using namespace dev;

enum Policy {
    P_CL32_ALL, P_CL32_THREAD, P_CL32_OVF,
    P_CL16_ALL, P_CL16_THREAD,
    P_MONT1, P_MONT2, P_MONT4,
    P_FP_THREAD, P_FP_K1, P_FP_K2,
    P_ZS_ALL, P_ZS_THREAD, P_ZL_ALL, P_ZL_THREAD,
    // explicit strategies (gfp_dot_ex): P_CS + 10*acc64 + 5*elem32 + (strategy - 1), strategies 1..4 and
    // the carry word (slot 4)
    P_CS = 32, P_CS_END = P_CS + 20,
    P_MONT_CARRY = 63,  // Montgomery with the carry word
    P_MONT_OVF = 64,
    P_ZECH_ADD = 65,  // pure-Zech accumulation (F3)
    // centered representation (sec. 3.2.2): int16 / int32 storage x {ALL, THREAD, BLOCKED}, binary64 x KF
    P_CE16_ALL = 66, P_CE16_THREAD, P_CE16_BLK, P_CE32_ALL, P_CE32_THREAD, P_CE32_BLK,
    P_FC0, P_FC1, P_FC2, P_FC4, P_FC8,
    P_COUNT
};
constexpr int cs_slot(int strat) { return strat == GFP_STRAT_CARRY ? 4 : strat - 1; }
constexpr int cs_policy(bool acc64, bool e32, int strat) { return P_CS + 10 * acc64 + 5 * e32 + cs_slot(strat); }
constexpr int cs_strategy(int pol) { return (pol - P_CS) % 5 == 4 ? GFP_STRAT_CARRY : (pol - P_CS) % 5 + 1; }

uint64_t launches(int reset);  // kernels_dot.cu (gfp_launch_count)

// ------------------------------------------------------------------------------ output encoding
__device__ __forceinline__ void write_result(uint64_t r, const OutSpec &O, const KParams &K, int64_t idx) {
    if (O.mode == OUT_PARTIAL) {
        ((uint64_t *)O.out)[idx] = r;
        return;
    }
    if (O.mode == OUT_ACCUMULATE) {
        ((uint64_t *)O.out)[idx] += r;  // single writer, stream-ordered
        return;
    }
    switch (O.rep) {
    case GFP_REP_FP64:
        ((double *)O.out)[idx] = (double)r;  // exact, never -0.0
        break;
    case GFP_REP_ZECH:
        ((uint16_t *)O.out)[idx] = r == 0 ? (uint16_t)0 : K.logt[r];
        break;
    case GFP_REP_CENTERED: {  // sec. 3.2.2: residues above h are stored as r - p
        const int64_t c = r > (uint64_t)K.half ? (int64_t)r - (int64_t)K.p : (int64_t)r;
        if (O.dtype == GFP_U16) ((int16_t *)O.out)[idx] = (int16_t)c;
        else if (O.dtype == GFP_U32) ((int32_t *)O.out)[idx] = (int32_t)c;
        else ((double *)O.out)[idx] = (double)c;  // exact, +0.0 for 0
        break;
    }
    default:  // classical residue, or Montgomery form (the sum of aB-forms is the aB-form)
        if (O.dtype == GFP_U16)
            ((uint16_t *)O.out)[idx] = (uint16_t)r;
        else
            ((uint32_t *)O.out)[idx] = (uint32_t)r;
    }
}

// ------------------------------------------------------------------------------ fused multi-GPU combine
// gfp_dot_allreduce (gfp.h protocol): called by ONE thread of the last CTA with this rank's partial residue
// r (additive form, < p < 2^32); returns the residue of the sum over all ranks.  Peer buffers are other
// GPUs' memory mapped over NVLink (CUDA IPC).  Each rank stores ONE tagged word (epoch << 32 | r) into
// slot [e mod 2][rank] of every rank's buffer and polls its own slots until every rank's word carries
// epoch e: the data and its flag are one aligned 64-bit store (single-copy atomic), so no release /
// acquire fence is needed at system scope -- the fences of a separate flag cost ~2.5 us per launch
// (profiles/r01_fused_ab.txt).  Slots for epoch e + 2 are only written after every rank has published
// e + 1, i.e. after every rank has read epoch e's slots (two parities suffice).
__device__ __forceinline__ uint64_t xchg_allreduce(uint64_t r, uint64_t *own, uint64_t p, uint64_t mu) {
    const uint64_t e = own[0] + 1;  // this rank's epoch: only this rank's kernels touch word 0, in stream order
    const int rank = (int)own[1], world = (int)own[2];
    uint64_t *const *peers = reinterpret_cast<uint64_t *const *>(own + kXPeers);
    const int par = (int)(e & 1);
    const uint64_t tag = e & 0xFFFFFFFFull;
    const uint64_t word = (tag << 32) | r;
    for (int q = 0; q < world; ++q) {
        uint64_t *slot = peers[q] + kXSlots + par * GFP_XCHG_MAX_WORLD + rank;
        asm volatile("st.relaxed.sys.u64 [%0], %1;" ::"l"(slot), "l"(word) : "memory");
    }
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    // a peer that never arrives: trap after ~30 s (fail loudly, do not hang); with a soft timeout armed in
    // word [kXSoft] (gfp_xchg_soft_timeout: connectivity checks) record it in [kXTimedOut] and return instead
    const uint64_t soft = own[kXSoft], limit = soft ? soft : 30000000000ull;
    bool late = false;
    uint64_t sum = 0;
    for (int q = 0; q < world && !late; ++q) {
        const uint64_t *slot = own + kXSlots + par * GFP_XCHG_MAX_WORLD + q;
        for (;;) {
            uint64_t v;
            asm volatile("ld.relaxed.sys.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
            if ((v >> 32) == tag) {
                sum += v & 0xFFFFFFFFull;  // world <= 16 residues < 2^32: no wrap
                break;
            }
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > limit) {
                if (!soft) __trap();
                late = true;
                break;
            }
            __nanosleep(32);
        }
    }
    own[0] = e;
    if (late) {
        own[kXTimedOut] = 1;
        return 0;
    }
    return mod_p(sum, p, mu);
}

// gfp_dot_allreduce_mc (gfp.h protocol): the fused combine through an NVLS multicast buffer.  ONE thread of the
// last CTA adds this rank's partial residue r (< 2^32) to the parity slot's running sum on every rank at once
// (multimem.red: the switch applies it to each member's copy), then -- release -- one arrival to the slot's
// counter; it polls its own copy of the counter (acquire) until world x (uses of this parity) arrivals are in,
// and this epoch's group sum is the slot's running total minus its total at the parity's previous use
// (wrapping u64 arithmetic: exact).  A rank can only add to parity e mod 2 at epoch e + 2 after every rank
// arrived at epoch e + 1, i.e. after every rank read epoch e's total: two parities suffice.  A missing peer
// traps after ~30 s instead of hanging.
__device__ __forceinline__ uint64_t mc_allreduce(uint64_t r, uint64_t *uc, uint64_t *mc, uint64_t p, uint64_t mu) {
    const uint64_t e = uc[0] + 1;  // only this rank's kernels touch its private words, in stream order
    const int par = (int)(e & 1);
    const uint64_t world = uc[1], uses = uc[2 + par] + 1;
    asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc + kMcSum + par), "l"(r) : "memory");
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc + kMcCnt + par), "l"(1ull) : "memory");
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint64_t c;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(c) : "l"(uc + kMcCnt + par) : "memory");
        if (c >= world * uses) break;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 30000000000ull) __trap();  // a peer never arrived: fail loudly, do not hang
        __nanosleep(32);
    }
    uint64_t total;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(total) : "l"(uc + kMcSum + par) : "memory");
    const uint64_t sum = total - uc[4 + par];  // this epoch's sum of world residues < 2^36
    uc[4 + par] = total;
    uc[2 + par] = uses;
    uc[0] = e;
    return mod_p(sum, p, mu);
}

// Bytes [sh, sh + 16) of the 32-byte concatenation lo:hi (sh in {2, 4, ..., 14}, a whole number of elements):
// the 16-byte window of an operand that is not co-aligned with the other one, from the two aligned vectors it
// straddles.  Word k of the window is word q + k funnel-shifted with word q + k + 1 (q = sh / 4).
__device__ __forceinline__ uint4 realign16(uint4 lo, uint4 hi, int sh) {
    const int q = sh >> 2, r = (sh & 3) * 8;
    const uint32_t w0 = lo.x, w1 = lo.y, w2 = lo.z, w3 = lo.w, w4 = hi.x, w5 = hi.y, w6 = hi.z, w7 = hi.w;
    const uint32_t s0 = q == 0 ? w0 : q == 1 ? w1 : q == 2 ? w2 : w3;
    const uint32_t s1 = q == 0 ? w1 : q == 1 ? w2 : q == 2 ? w3 : w4;
    const uint32_t s2 = q == 0 ? w2 : q == 1 ? w3 : q == 2 ? w4 : w5;
    const uint32_t s3 = q == 0 ? w3 : q == 1 ? w4 : q == 2 ? w5 : w6;
    const uint32_t s4 = q == 0 ? w4 : q == 1 ? w5 : q == 2 ? w6 : w7;
    return make_uint4(__funnelshift_r(s0, s1, r), __funnelshift_r(s1, s2, r), __funnelshift_r(s2, s3, r),
                      __funnelshift_r(s3, s4, r));
}

// Stage a u16 table (entries padded to a multiple of 8) from global into shared memory.
__device__ __forceinline__ void stage_table(uint16_t *dst, const uint16_t *src, uint32_t entries) {
    const uint4 *s = reinterpret_cast<const uint4 *>(src);
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    for (uint32_t i = threadIdx.x; i < entries / 8; i += blockDim.x) d[i] = __ldg(s + i);
}

// ------------------------------------------------------------------------------ programmatic dependent launch
// Every hot kernel is launched with programmatic stream serialization (launch_pdl): the next kernel's
// launch is staged while this one runs.  Each kernel waits (griddepcontrol.wait: every earlier kernel in
// the stream has completed and its writes are visible) before its first load, so memory order is the
// stream order, and each CTA signals its dependents after its last global write.
// Dots whose threads stream at most kPrefetchMaxIters chunks (the launcher sets O.prefetch) and batches
// first prefetch the thread's first chunk of both operands into L2, so the DRAM round trip of the first
// loads overlaps the previous kernel's drain (its last CTA's combine and the memory flush).  An L2
// prefetch cannot observe stale data: L2 is the device's point of coherence and nothing is loaded into
// registers or L1 before the wait.  A/B on the B200 (scripts/ab_secondary.sh, scripts/ab_head.sh,
// profiles/r01_pdl_ab.txt): prefetch -6% at C2, -1.5% at C4 / F3 / C5, -0.2% at C3 (16 waves: ~5 chunks
// per thread); conversions are flat grids with one tile per thread and no prefetch.  Signalling the
// dependents at CTA entry instead (GFP_PDL_EARLY=1) was slower on every config.
#ifndef GFP_PDL_EARLY
#define GFP_PDL_EARLY 0
#endif
#ifndef GFP_PDL_PREFETCH
#define GFP_PDL_PREFETCH 1
#endif
// prefetch when each thread streams at most this many U-chunks
constexpr int64_t kPrefetchMaxIters = 32;
__device__ __forceinline__ void prefetch_l2(const void *ptr) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}
template <int U, int NT>
__device__ __forceinline__ void pdl_prefetch(const uint4 *av, const uint4 *bv, int64_t i0, int64_t nvec, bool pf) {
    if (GFP_PDL_PREFETCH && pf) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * NT < nvec) {
                prefetch_l2(av + i0 + u * NT);
                prefetch_l2(bv + i0 + u * NT);
            }
    }
}
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // stream order (no-op without a programmatic launch)
    if (GFP_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <int U, int NT>
__device__ __forceinline__ void pdl_enter(const uint4 *av, const uint4 *bv, int64_t i0, int64_t nvec, bool pf) {
    pdl_prefetch<U, NT>(av, bv, i0, nvec, pf);
    pdl_wait();
}
// The Zech tables are library-owned device memory, written once (synchronously) when a (device, p) cache
// entry is built and never by stream work: the table kernels stage them into shared memory BEFORE
// griddepcontrol.wait, so under PDL the copy overlaps the previous kernel's drain (GFP_STAGE_EARLY).
#ifndef GFP_STAGE_EARLY
#define GFP_STAGE_EARLY 1
#endif
#ifndef GFP_ZADD_STAGE_EARLY
#define GFP_ZADD_STAGE_EARLY 0
#endif
__device__ __forceinline__ void pdl_exit() {
    if (!GFP_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // after the last write
}

// ------------------------------------------------------------------------------ tuning knobs (A/B builds: make variant)
#ifndef GFP_CONV_FLAT
#define GFP_CONV_FLAT 1  // 1: one U-chunk tile per thread, grid not capped at the resident CTAs (no table)
#endif
#ifndef GFP_ZBATCH_U
#define GFP_ZBATCH_U 4  // 16-byte vectors per lane in flight in the Zech batch (doubled table)
#endif
#ifndef GFP_ZBATCH_DECODE
#define GFP_ZBATCH_DECODE 1  // 1: Zech matrix-vector by decode + DP2A (batch_zech_kernel); 0: index-add batch_kernel
#endif
#ifndef GFP_ZSPLIT
#define GFP_ZSPLIT 1  // 1: Zech matrix-vector by split-exponent lookups (batch_zsplit_kernel) where it applies
#endif
#ifndef GFP_ZS_NT
#define GFP_ZS_NT 1024  // threads per CTA of the split-exponent batch (one CTA per SM: 128 KB of shared memory)
#endif
#ifndef GFP_ZS_U
#define GFP_ZS_U 2  // 16-byte A vectors per row and lane in flight in the split-exponent batch
#endif
#ifndef GFP_ZS_RP
#define GFP_ZS_RP 2  // rows a warp of the split-exponent batch walks at once
#endif
#ifndef GFP_ZDEC_RP
#define GFP_ZDEC_RP 2  // rows a warp of the decode batch walks at once (each staged x read serves RP rows)
#endif
#ifndef GFP_ZDEC_NT
#define GFP_ZDEC_NT 1024  // threads per CTA of the decode batch (one CTA per SM)
#endif
#ifndef GFP_ZDEC_U
#define GFP_ZDEC_U 4  // 16-byte A vectors per row and lane in flight in the decode batch
#endif
#ifndef GFP_ZBATCH_UL
#define GFP_ZBATCH_UL 8  // the same for the large-field (q-entry, folded index) table
#endif
#ifndef GFP_ZADD_U
#define GFP_ZADD_U 2  // 16-byte vectors per operand per step of the pure-Zech dot
#endif
#ifndef GFP_ZECH_NT
#define GFP_ZECH_NT 1024  // threads per CTA of the integer Zech dot (one CTA per SM: the table fills smem)
#endif
#ifndef GFP_ZECH_U
#define GFP_ZECH_U 2  // 16-byte vectors per operand per step of the integer Zech dot
#endif
#ifndef GFP_CL16_U
#define GFP_CL16_U 16  // C5 batch: 16-byte A vectors per lane in flight (long rows)
#endif
#ifndef GFP_BATCH_WAVES
#define GFP_BATCH_WAVES 4  // C5 batch grid: waves of resident CTAs (B200 A/B, profiles/r01_waves_ab.txt)
#endif
#ifndef GFP_DOT_WAVES
#define GFP_DOT_WAVES 16  // most waves of resident CTAs for a long table-free dot (see plan_dot)
#endif
#ifndef GFP_WAVE_LOG2
#define GFP_WAVE_LOG2 25  // one wave per 2^25 bytes (32 MiB) of operands (plan_dot)
#endif
#ifndef GFP_CONV_WAVES
#define GFP_CONV_WAVES 1  // resident-grid conversions: grid = waves x the resident CTAs
#endif
#ifndef GFP_CONV_TAB_U
#define GFP_CONV_TAB_U 4  // table (Zech) conversions: 8-element chunks per thread in flight
#endif
#ifndef GFP_CONV_TAB_NT
#define GFP_CONV_TAB_NT 512  // table (Zech) conversions: threads per CTA (B200 A/B, scripts/ab_zconv.py: C4's two
                              // operands from_zech / to_zech 95.0 / 94.1 us at 1024 threads x U = 2, 88.8 / 90.4 here)
#endif
#ifndef GFP_CONV_LD
#define GFP_CONV_LD 1  // 0: ld.global.cs (streaming), 1: ld.global.L1::no_allocate (coherent: in == out is fine)
#endif
#ifndef GFP_CONV_ST
#define GFP_CONV_ST 0  // 0: st.global.cs (streaming), 1: plain st.global, 2: st.global.L1::no_allocate
#endif
// ------------------------------------------------------------------------------ launch helpers
// Programmatic dependent launch for the dot kernels: the launch of dot N+1 is staged while dot N runs.
// The kernel waits (griddepcontrol.wait) before doing anything and each CTA signals its dependents
// (griddepcontrol.launch_dependents) only after its last global write, so memory order is exactly the
// stream order; what overlaps is the launch latency of the next dot.
#ifndef GFP_PDL
#define GFP_PDL 1
#endif
template <typename Kern, typename... Args>
static cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = GFP_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename F>
static int occupancy(F kernel, int block, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<std::string, int> cache;       // per (device, kernel, dynamic smem)
    static std::unordered_map<std::string, size_t> allowed;  // per (device, kernel): the smem opt-in so far
    std::lock_guard<std::mutex> g(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const uintptr_t kp = (uintptr_t)reinterpret_cast<const void *>(kernel);
    const std::string fkey = std::to_string(dev) + ":" + std::to_string(kp);
    // the opt-in is a per-function attribute of the current device's context: only ever raise it (a kernel
    // launched with several table sizes, e.g. Zech at several primes, must keep the largest one it has been
    // allowed), and once per device (a process driving several GPUs opts in on each)
    if (smem > 48 * 1024 && smem > allowed[fkey]) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        allowed[fkey] = smem;
    }
    const std::string key = fkey + ":" + std::to_string(smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int bps = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, block, smem) != cudaSuccess || bps < 1) bps = 1;
    cache[key] = bps;
    return bps;
}

// Measured on B200 (scripts/ab_bench.sh, scripts/ab_head.sh, scripts/tune_*.cu): unpipelined loads beat
// the register-pipelined variant (80 regs) by 2% on C3 (U = 2 with multi-wave grids; U = 4 was best with
// one wave); fp64 is best at U = 2; Zech (1024 threads, 64-register cap) needs the pipeline to keep
// loads in flight across its table lookups.
#ifndef GFP_DOT_PIPE
#define GFP_DOT_PIPE 0
#endif
#ifndef GFP_FP_U
#define GFP_FP_U 2
#endif
#ifndef GFP_DOT_U
#define GFP_DOT_U 2  // Montgomery and explicit strategies; with the multi-wave grids U 2: 290.6 -> 289.4 us at C3
#endif
#ifndef GFP_CL_U
#define GFP_CL_U 4  // built-in classical dots: 4 loads per operand in flight serve C1's DRAM-latency-bound 10^5
#endif          // terms from fewer CTAs (2.68 vs 2.84 us with U 2; scripts/ab_sec2.sh)
#ifndef GFP_CONV_U
#define GFP_CONV_U 2  // B200 A/B, flat grid: U = 1 / 2 / 4 -> 6.97 / 6.94 / 6.60 TB/s (to_montgomery, 4 GiB)
#endif
constexpr int kClU = GFP_CL_U;  // built-in classical dots
constexpr int kDotNT = 256, kDotU = GFP_DOT_U, kFpU = GFP_FP_U, kZechNT = GFP_ZECH_NT, kZechU = GFP_ZECH_U, kZaddNT = 1024, kZaddU = GFP_ZADD_U;
constexpr bool kPipe = GFP_DOT_PIPE != 0;

// explicit-strategy policy type for (acc64, e32, strategy)
#define GFP_CS_CASES(M)                                                                     \
    M(cs_policy(0, 0, 1), ClassicalS<uint32_t, uint16_t, S_DELAYED>)                        \
    M(cs_policy(0, 0, 2), ClassicalS<uint32_t, uint16_t, S_BLOCKED>)                        \
    M(cs_policy(0, 0, 3), ClassicalS<uint32_t, uint16_t, S_OVERFLOW>)                       \
    M(cs_policy(0, 0, 4), ClassicalS<uint32_t, uint16_t, S_HYBRID>)                         \
    M(cs_policy(0, 0, GFP_STRAT_CARRY), ClassicalS<uint32_t, uint16_t, S_CARRY>)            \
    M(cs_policy(0, 1, 1), ClassicalS<uint32_t, uint32_t, S_DELAYED>)                        \
    M(cs_policy(0, 1, 2), ClassicalS<uint32_t, uint32_t, S_BLOCKED>)                        \
    M(cs_policy(0, 1, 3), ClassicalS<uint32_t, uint32_t, S_OVERFLOW>)                       \
    M(cs_policy(0, 1, 4), ClassicalS<uint32_t, uint32_t, S_HYBRID>)                         \
    M(cs_policy(0, 1, GFP_STRAT_CARRY), ClassicalS<uint32_t, uint32_t, S_CARRY>)            \
    M(cs_policy(1, 0, 1), ClassicalS<uint64_t, uint16_t, S_DELAYED>)                        \
    M(cs_policy(1, 0, 2), ClassicalS<uint64_t, uint16_t, S_BLOCKED>)                        \
    M(cs_policy(1, 0, 3), ClassicalS<uint64_t, uint16_t, S_OVERFLOW>)                       \
    M(cs_policy(1, 0, 4), ClassicalS<uint64_t, uint16_t, S_HYBRID>)                         \
    M(cs_policy(1, 0, GFP_STRAT_CARRY), ClassicalS<uint64_t, uint16_t, S_CARRY>)            \
    M(cs_policy(1, 1, 1), ClassicalS<uint64_t, uint32_t, S_DELAYED>)                        \
    M(cs_policy(1, 1, 2), ClassicalS<uint64_t, uint32_t, S_BLOCKED>)                        \
    M(cs_policy(1, 1, 3), ClassicalS<uint64_t, uint32_t, S_OVERFLOW>)                       \
    M(cs_policy(1, 1, 4), ClassicalS<uint64_t, uint32_t, S_HYBRID>)                         \
    M(cs_policy(1, 1, GFP_STRAT_CARRY), ClassicalS<uint64_t, uint32_t, S_CARRY>)            \
    M(P_MONT_OVF, MontgomeryOverflow)                                                         \
    M(P_MONT_CARRY, MontgomeryCarry)                                                          \
    M(P_CE16_ALL, CenteredI<int16_t, CE_ALL>)                                                 \
    M(P_CE16_THREAD, CenteredI<int16_t, CE_THREAD>)                                           \
    M(P_CE16_BLK, CenteredI<int16_t, CE_BLOCKED>)                                             \
    M(P_CE32_ALL, CenteredI<int32_t, CE_ALL>)                                                 \
    M(P_CE32_THREAD, CenteredI<int32_t, CE_THREAD>)                                           \
    M(P_CE32_BLK, CenteredI<int32_t, CE_BLOCKED>)

// binary64 centered policies (unroll kFpU like Fp64)
#define GFP_FC_CASES(M)      \
    M(P_FC0, Fp64C<0>)       \
    M(P_FC1, Fp64C<1>)       \
    M(P_FC2, Fp64C<2>)       \
    M(P_FC4, Fp64C<4>)       \
    M(P_FC8, Fp64C<8>)

inline size_t elem_size(int dt) { return dt == GFP_U16 ? 2 : (dt == GFP_U32 ? 4 : 8); }

// binary64 centered: the largest compiled block KF in {8, 4, 2, 1} not above lambda_c
inline int fc_policy(uint64_t lambda_c) {
    return lambda_c >= 8 ? P_FC8 : (lambda_c >= 4 ? P_FC4 : (lambda_c >= 2 ? P_FC2 : P_FC1));
}
inline uint64_t fc_block(int pol) { return pol == P_FC8 ? 8 : (pol == P_FC4 ? 4 : (pol == P_FC2 ? 2 : (pol == P_FC1 ? 1 : 0))); }

// Explicit strategy (gfp_options) -> policy and block length; GFP_OK or the reason it is not admissible
// (kernels_dot.cu; the batch launcher resolves the same options).
gfp_status resolve_strategy(const gfp_info &I, int64_t n, const gfp_options *opt, int *pol, uint64_t *kblk,
                            int *acc_bits);

}  // namespace gfp
