// kernels.cu -- the hot-path kernels for sm_100a and their launchers.
//
//   dot_kernel      single dot product: persistent grid-stride streaming of both operands with
//                   16-byte loads, per-thread delayed-modulus accumulation (policy R, device.cuh),
//                   warp-shuffle + CTA tree, per-CTA partial, last-CTA-done final reduction and
//                   encoding -- one launch per dot.
//                   With OUT_XCHG the last CTA also exchanges the partial with the peer GPUs over
//                   NVLink peer memory and finalizes (gfp_dot_allreduce, a9 fused).
//   zech_add_dot_kernel  the pure-Zech dot (F3): Table-1 products, t_plus1 additions in shared memory.
//   batch_cl16      C5 matrix-vector over classical u16: warp per row, x byte-split in shared
//                   memory, two DP2A per pair of terms (a8).
//   batch_kernel    generic batch (any policy): LPR lanes per row, x staged in shared memory.
//   convert_kernel  representation conversions (a2).
//   finalize_kernel sum of partial residues -> mod p -> encode (a7/a9).
//   fill_kernel     synthetic canonical inputs for the install-time tuner (F4, tune.cpp).
//   xchg_setup_kernel  writes a fused-combine group description into an exchange buffer.
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

static thread_local uint64_t t_launches = 0;
void count_launch() { ++t_launches; }
uint64_t launches(int reset) {
    uint64_t v = t_launches;
    if (reset) t_launches = 0;
    return v;
}

int num_sms(int device) {
    static std::mutex mu;
    static std::unordered_map<int, int> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    cache[device] = v;
    return v;
}

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
    uint64_t sum = 0;
    for (int q = 0; q < world; ++q) {
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
            if (t - t0 > 30000000000ull) __trap();  // a peer never arrived: fail loudly, do not hang
            __nanosleep(32);
        }
    }
    own[0] = e;
    return mod_p(sum, p, mu);
}

struct XchgDesc {
    uint64_t *peers[GFP_XCHG_MAX_WORLD];
};
__global__ void xchg_setup_kernel(uint64_t *own, int rank, int world, XchgDesc d) {
    own[1] = (uint64_t)rank;
    own[2] = (uint64_t)world;
    for (int r = 0; r < GFP_XCHG_MAX_WORLD; ++r) own[kXPeers + r] = r < world ? (uint64_t)(uintptr_t)d.peers[r] : 0;
}

cudaError_t launch_xchg_setup(uint64_t *own, int rank, int world, uint64_t *const *peers, cudaStream_t s) {
    XchgDesc d;
    for (int r = 0; r < GFP_XCHG_MAX_WORLD; ++r) d.peers[r] = r < world ? peers[r] : nullptr;
    xchg_setup_kernel<<<1, 1, 0, s>>>(own, rank, world, d);
    count_launch();
    return cudaGetLastError();
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

// ------------------------------------------------------------------------------ single dot

template <class R, int NT, int U, bool PIPE>
__global__ void __launch_bounds__(NT) dot_kernel(const typename R::elem *__restrict__ a,
                                                 const typename R::elem *__restrict__ b, int64_t n,
                                                 int64_t head, KParams K, Workspace ws, OutSpec O) {
    extern __shared__ __align__(16) uint16_t s_tab[];
    __shared__ uint64_t red[32];
    typename R::Acc acc;
    R::init(acc);
    const int64_t gtid = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * NT;
    const int64_t nvec = (n - head) / R::W;
    const uint4 *av = reinterpret_cast<const uint4 *>(a + head);
    const uint4 *bv = reinterpret_cast<const uint4 *>(b + head);
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    pdl_prefetch<U, NT>(av, bv, i0, nvec, O.prefetch != 0);
    if constexpr (R::kTable && GFP_STAGE_EARLY) stage_table(s_tab, K.antilog, K.antilog_entries);
    pdl_wait();
    const int64_t step = (int64_t)gridDim.x * (NT * U);
    const uint16_t *tab = nullptr;

    // Software-pipelined stream (PIPE): the U loads of each operand for step k+1 are in flight while
    // step k computes, so every thread keeps between U and 2U 16-byte loads outstanding per operand.
    // Without GFP_STAGE_EARLY the first loads are issued before the Zech antilog table is staged, so the
    // stream's DRAM latency overlaps the table copy from L2 into shared memory.
    uint4 ca[U], cb[U];
    bool have = PIPE && i0 + (U - 1) * NT < nvec;
    if (PIPE && have) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ca[u] = ld_stream(av + i0 + u * NT);
            cb[u] = ld_stream(bv + i0 + u * NT);
        }
    }
    if constexpr (R::kTable) {
        if (!GFP_STAGE_EARLY) stage_table(s_tab, K.antilog, K.antilog_entries);
        __syncthreads();
        tab = s_tab;
    }
    if constexpr (PIPE) {
        // two register sets in ping-pong: the next step's loads land in the set not being consumed
        uint4 na[U], nb[U];
        auto step_once = [&](uint4 (&cx)[U], uint4 (&cy)[U], uint4 (&nx_a)[U], uint4 (&nx_b)[U]) {
            const int64_t nx = i0 + step;
            const bool more = nx + (U - 1) * NT < nvec;
            if (more) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    nx_a[u] = ld_stream(av + nx + u * NT);
                    nx_b[u] = ld_stream(bv + nx + u * NT);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) R::vec(acc, cx[u], cy[u], K, tab);
            i0 = nx;
            have = more;
        };
        while (have) {
            step_once(ca, cb, na, nb);
            if (!have) break;
            step_once(na, nb, ca, cb);
        }
    }

    // scalar head (the whole input when a and b are not co-aligned)
    for (int64_t i = gtid; i < head; i += gstride) R::term(acc, a[i], b[i], K, tab);

    // 16-byte vector body (!PIPE): U independent loads of each operand in flight per thread
    for (; i0 + (U - 1) * NT < nvec; i0 += step) {
        uint4 xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xa[u] = ld_stream(av + i0 + u * NT);
            xb[u] = ld_stream(bv + i0 + u * NT);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) R::vec(acc, xa[u], xb[u], K, tab);
    }
    if (i0 < nvec) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * NT < nvec) R::vec(acc, ld_stream(av + i0 + u * NT), ld_stream(bv + i0 + u * NT), K, tab);
    }
    // scalar tail (< W elements)
    for (int64_t i = head + nvec * R::W + gtid; i < n; i += gstride) R::term(acc, a[i], b[i], K, tab);

    // combine: warp shuffle -> CTA tree -> one u64 atomic per CTA; the CTA whose arrival on the
    // counter is last (acq_rel orders every earlier CTA's atomic before its own read) reduces mod p
    // once and encodes -- "A single machine remaindering is needed at the end".
    // Exact and order-independent: integer sums, no wrap (host-checked bounds).
    const uint64_t v = block_sum(R::finish(acc, K), red);
    if (threadIdx.x == 0) {
        // Packed combine (the plan keeps grids below 2^(64 - kPackShift) CTAs): the CTA's sum is reduced to its
        // residue c < p < 2^32 (centered sums are signed two's complement: smod_p), and ONE atomic adds c and
        // one arrival to a single word; the CTA that sees every other arrival in the old value holds the
        // complete total -- one L2 round trip, where a sum atomic + acq_rel counter + reload took three.  The
        // word holds nothing but the sums, so relaxed order suffices.
        const uint64_t c = O.rep == GFP_REP_CENTERED ? smod_p((int64_t)v, K) : mod_p(v, K.p, K.mu);
        unsigned long long *word = reinterpret_cast<unsigned long long *>(ws.partials);
        unsigned long long old;
        asm volatile("atom.relaxed.gpu.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(word),
                     "l"((unsigned long long)c + (1ull << kPackShift)) : "memory");
        if ((old >> kPackShift) == gridDim.x - 1) {
            uint64_t r = mod_p((old & ((1ull << kPackShift) - 1)) + c, K.p, K.mu);
            if (O.mode == OUT_XCHG) r = xchg_allreduce(r, O.xchg, K.p, K.mu);  // fused multi-GPU combine
            write_result(r, O, K, 0);
            *word = 0;  // self-reset for the next launch on this stream
        }
        pdl_exit();
    }
}

// ------------------------------------------------------------------------------ pure-Zech dot (F3)
// Every product and every partial sum stays in the discrete-log representation (sec. 2.4, Table 1):
// a product is an index addition, a sum one lookup in the t_plus1 table (staged in shared memory).
// Eight independent Zech accumulators per thread (one per u16 lane of a 16-byte vector) hide the
// lookup latency of the dependent additions; they are merged by Zech additions in the thread, the
// warp (shuffles) and the CTA, and each CTA's merged value goes to the workspace, where the last CTA
// to arrive on the counter merges them all and encodes.  No integer sum, no remainder anywhere.
template <int S>
__device__ __forceinline__ uint32_t zech_warp_merge(uint32_t v, uint32_t q, const uint16_t *D) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = zadd::Ops<S>::add(v, __shfl_xor_sync(0xFFFFFFFFu, v, o), q, D);
    return v;
}

// Merge over the CTA; valid in thread 0.
template <int S>
__device__ __forceinline__ uint32_t zech_block_merge(uint32_t v, uint32_t *red, uint32_t q, const uint16_t *D) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = zech_warp_merge<S>(v, q, D);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = zadd::Ops<S>::kZ;
    if (warp == 0) v = zech_warp_merge<S>(lane < nw ? red[lane] : zadd::Ops<S>::kZ, q, D);
    return v;
}

template <int S>
__device__ __forceinline__ void zech_add_pair(uint32_t (&acc)[8], int j, uint32_t x, uint32_t y, uint32_t q,
                                              const uint16_t *D) {
    using Z = zadd::Ops<S>;
    acc[2 * j] = Z::add(acc[2 * j], Z::mul(x & 0xFFFFu, y & 0xFFFFu, q), q, D);
    acc[2 * j + 1] = Z::add(acc[2 * j + 1], Z::mul(x >> 16, y >> 16, q), q, D);
}

template <int S>
__device__ __forceinline__ void zech_add_vec(uint32_t (&acc)[8], uint4 x, uint4 y, uint32_t q, const uint16_t *D) {
    zech_add_pair<S>(acc, 0, x.x, y.x, q, D);
    zech_add_pair<S>(acc, 1, x.y, y.y, q, D);
    zech_add_pair<S>(acc, 2, x.z, y.z, q, D);
    zech_add_pair<S>(acc, 3, x.w, y.w, q, D);
}

// Fast path (S = 2, odd p, 2 qbar < 2^16): the running sums never hold the zero element, so the
// additions need no zero tests.  Each sum starts at the element 1 (v = 0) and `corr` (checked
// arithmetic) books -1 for it.  A zero product is steered to the table's "add nothing" entry (byte
// offset kzero, delta 0).  A sum that cancels (delta sentinel 0xFFFF) becomes odd -- every valid v is
// even -- and is repaired once per vector: restart at 1, book -1 in corr.  The product index
// 2 (ci + cj) - s is not folded first: the table is doubled (indices [0, 2q]) instead.
// Per term: lane extract, one multiply-add for the index, one index fold, one select, one lookup,
// one add and one fold for the sum.
__device__ __forceinline__ uint32_t zech_fast_add(uint32_t s, uint32_t lane_sum, bool zero, uint32_t q,
                                                  uint32_t kzero, uint32_t tab) {
    uint32_t k = 2u * lane_sum - s;  // 2 (ci + cj) - s in (4 - q, 2q] for canonical codes
    k = min(k, k + q);                // in [0, 2^17 - 2] for any 16-bit lane: the staged table is padded to
    k = zero ? kzero : k;             // 2^16 entries, so non-canonical codes never leave it (gfp.h)
    uint16_t d;
    asm("ld.shared.u16 %0, [%1];" : "=h"(d) : "r"(tab + k));
    return zadd::Ops<2>::fold(s + d, q);
}

__device__ __forceinline__ void zech_fast_pair(uint32_t (&acc)[8], int j, uint32_t x, uint32_t y, uint32_t q,
                                               uint32_t kzero, uint32_t tab) {
    const uint32_t P = x + y;             // codes < 2^15: both 16-bit lane sums fit, no carry between lanes
    const uint32_t m = __vminu2(x, y);    // per lane min(ci, cj): zero iff the lane's product is zero
    acc[2 * j] = zech_fast_add(acc[2 * j], P & 0xFFFFu, (m & 0xFFFFu) == 0, q, kzero, tab);
    acc[2 * j + 1] = zech_fast_add(acc[2 * j + 1], P >> 16, m < 0x10000u, q, kzero, tab);
}

__device__ __forceinline__ void zech_repair(uint32_t (&acc)[8], uint32_t &corr, uint32_t q, const uint16_t *D) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (acc[j] & 1u) {  // this sum cancelled to zero: restart it at 1 (v = 0), book -1 (v = q/2) in corr
            acc[j] = 0u;
            corr = zadd::Ops<2>::add(corr, q / 2u, q, D);
        }
    }
}

__device__ __forceinline__ void zech_fast_vec(uint32_t (&acc)[8], uint32_t &corr, uint4 x, uint4 y, uint32_t q,
                                              uint32_t kzero, const uint16_t *D) {
    const uint32_t tab = (uint32_t)__cvta_generic_to_shared(D);  // table base as a shared-window offset
    zech_fast_pair(acc, 0, x.x, y.x, q, kzero, tab);
    zech_fast_pair(acc, 1, x.y, y.y, q, kzero, tab);
    zech_fast_pair(acc, 2, x.z, y.z, q, kzero, tab);
    zech_fast_pair(acc, 3, x.w, y.w, q, kzero, tab);
    if ((acc[0] | acc[1] | acc[2] | acc[3] | acc[4] | acc[5] | acc[6] | acc[7]) & 1u) zech_repair(acc, corr, q, D);
}

template <int NT, int U, int S, bool FAST>
__global__ void __launch_bounds__(NT) zech_add_dot_kernel(const uint16_t *__restrict__ a,
                                                          const uint16_t *__restrict__ b, int64_t n, int64_t head,
                                                          KParams K, Workspace ws, OutSpec O) {
    using Z = zadd::Ops<S>;
    extern __shared__ __align__(16) uint16_t s_delta[];
    __shared__ uint32_t red[32];
    __shared__ int s_last;
    const uint32_t q = (uint32_t)S * K.qbar;
    const int64_t gtid = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * NT;
    const int64_t nvec = (n - head) / 8;
    const uint4 *av = reinterpret_cast<const uint4 *>(a + head);
    const uint4 *bv = reinterpret_cast<const uint4 *>(b + head);
    int64_t i0 = (int64_t)blockIdx.x * (NT * U) + threadIdx.x;
    pdl_prefetch<U, NT>(av, bv, i0, nvec, O.prefetch != 0);
    // (staging this table before the wait, as the other table kernels do, was 1% slower here: B200 A/B,
    // profiles/r01_pdl_ab.txt; its first loads go out before the staging instead)
    if (GFP_ZADD_STAGE_EARLY)
        stage_table(s_delta, FAST ? K.zplus1s : K.zplus1, FAST ? K.zplus1s_entries : K.zplus1_entries);
    pdl_wait();
    const int64_t step = (int64_t)gridDim.x * (NT * U);

    // first loads in flight while the table is staged from L2
    uint4 ca[U], cb[U];
    bool have = i0 + (U - 1) * NT < nvec;
    if (have) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ca[u] = ld_stream(av + i0 + u * NT);
            cb[u] = ld_stream(bv + i0 + u * NT);
        }
    }
    if (!GFP_ZADD_STAGE_EARLY)
        stage_table(s_delta, FAST ? K.zplus1s : K.zplus1, FAST ? K.zplus1s_entries : K.zplus1_entries);
    const uint32_t kzero = 2u * q + 2u;  // fast path: byte offset of the "add nothing" entry
    __syncthreads();
    const uint16_t *D = s_delta;

    uint32_t acc[8], corr = Z::kZ;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        acc[j] = FAST ? 0u : Z::kZ;  // fast path: start at the element 1 (v = 0), booked as -1 in corr
        if (FAST) corr = Z::add(corr, q / 2u, q, D);
    }
    // Two register sets in ping-pong (no copies between iterations): while one set is consumed, the
    // loads of the next step land in the other.
    uint4 na[U], nb[U];
    auto step_once = [&](uint4 (&cx)[U], uint4 (&cy)[U], uint4 (&nx_a)[U], uint4 (&nx_b)[U]) {
        const int64_t nx = i0 + step;
        const bool more = nx + (U - 1) * NT < nvec;
        if (more) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                nx_a[u] = ld_stream(av + nx + u * NT);
                nx_b[u] = ld_stream(bv + nx + u * NT);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (FAST) zech_fast_vec(acc, corr, cx[u], cy[u], q, kzero, D);
            else zech_add_vec<S>(acc, cx[u], cy[u], q, D);
        }
        i0 = nx;
        have = more;
    };
    while (have) {
        step_once(ca, cb, na, nb);
        if (!have) break;
        step_once(na, nb, ca, cb);
    }
    // ragged vectors (< U per thread), scalar head and tail
    for (int u = 0; u < U; ++u) {
        if (i0 + u * NT < nvec) {
            const uint4 x = ld_stream(av + i0 + u * NT), y = ld_stream(bv + i0 + u * NT);
            if constexpr (FAST) zech_fast_vec(acc, corr, x, y, q, kzero, D);
            else zech_add_vec<S>(acc, x, y, q, D);
        }
    }
    for (int64_t i = gtid; i < head; i += gstride) acc[0] = Z::add(acc[0], Z::mul(a[i], b[i], q), q, D);
    for (int64_t i = head + nvec * 8 + gtid; i < n; i += gstride)
        acc[1] = Z::add(acc[1], Z::mul(a[i], b[i], q), q, D);

    // merge: thread (tree over its 8 accumulators) -> warp -> CTA -> workspace -> last CTA
    acc[0] = Z::add(acc[0], acc[1], q, D);
    acc[2] = Z::add(acc[2], acc[3], q, D);
    acc[4] = Z::add(acc[4], acc[5], q, D);
    acc[6] = Z::add(acc[6], acc[7], q, D);
    acc[6] = Z::add(acc[6], corr, q, D);  // only nonzero on the fast path (corr starts at zero)
    acc[0] = Z::add(acc[0], acc[2], q, D);
    acc[4] = Z::add(acc[4], acc[6], q, D);
    uint32_t v = zech_block_merge<S>(Z::add(acc[0], acc[4], q, D), red, q, D);
    if (threadIdx.x == 0) {
        ws.partials[1 + blockIdx.x] = v;
        unsigned int t;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ws.counter) : "memory");
        s_last = t == gridDim.x - 1;
        if (!s_last) pdl_exit();
    }
    __syncthreads();
    if (!s_last) return;
    v = Z::kZ;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) {
        unsigned long long w;
        asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(w) : "l"(ws.partials + 1 + i) : "memory");
        v = Z::add(v, (uint32_t)w, q, D);
    }
    v = zech_block_merge<S>(v, red, q, D);
    if (threadIdx.x == 0) {
        if (O.mode == OUT_ENCODE) {
            ((uint16_t *)O.out)[0] = (uint16_t)Z::to_code(v, K.qbar);  // already a Zech code: no log lookup
        } else {  // additive (classical) form for the multi-GPU sum: g^(u+1) from the antilog table
            uint64_t r = v == Z::kZ ? 0 : K.antilog[Z::code_nz(v, K.qbar)];  // g^code, both layouts
            // fused multi-GPU combine: exchange the classical value with the peers, then encode the sum
            // (write_result: log table) -- the group's sum of Zech elements is not a sum of codes
            if (O.mode == OUT_XCHG) r = xchg_allreduce(r, O.xchg, K.p, K.mu);
            write_result(r, O, K, 0);
        }
        *ws.counter = 0;
        pdl_exit();
    }
}

// ------------------------------------------------------------------------------ finalize
__global__ void finalize_kernel(const uint64_t *summed, int count, KParams K, OutSpec O) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t r = 0;
    for (int i = 0; i < count; ++i) r = mod_p(r + mod_p(summed[i], K.p, K.mu), K.p, K.mu);
    write_result(r, O, K, 0);
}

// ------------------------------------------------------------------------------ batch: C5 fast path
// Classical u16, p <= 65521.  A row r is A[r*lda .. +n); x is staged once per CTA into shared
// memory as byte-split words w_j = (x_{2j} lo, x_{2j+1} lo, x_{2j} hi, x_{2j+1} hi), so that for a
// packed pair of A entries  dp2a_lo(A2, w) = a0 x0_lo + a1 x1_lo  and  dp2a_hi(A2, w) = a0 x0_hi + a1 x1_hi,
// each < 2^25.  Row value = sum lo + 256 * sum hi, accumulated in u64 per lane (no reduction, the
// row total n (p-1)^2 < 2^64 is host-checked; Eq. (1)), then one mod p per row.
// Segmented sum over aligned groups of L lanes (L a power of two <= 32).
template <int L>
__device__ __forceinline__ uint64_t group_sum(uint64_t v) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// Batch kernels under programmatic dependent launch (see pdl_enter): when pf, prefetch into
// L2 the first chunk of this lane's first row (U 16-byte vectors, LPR lanes per row; A16 is the row base
// in u16 units, lda16 the row stride in u16 units), then wait for the stream's earlier kernels.
template <int U, int LPR, int NT>
__device__ __forceinline__ void batch_pdl_enter(const void *A, int64_t lda16, int64_t rows, int64_t nvec, bool pf) {
    if (GFP_PDL_PREFETCH && pf) {
        const int lane = threadIdx.x & 31;
        const int64_t row = ((int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5)) * (32 / LPR) + lane / LPR;
        if (row < rows) {
            const uint4 *av = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint16_t *>(A) + row * lda16);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (lane % LPR + u * LPR < nvec) prefetch_l2(av + lane % LPR + u * LPR);
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (GFP_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// LPR lanes per row (32: a warp per long row; 8: four short rows per warp, so DIM = 512 rows still
// keep 8 vectors per lane in flight and pay a 3-step instead of a 5-step shuffle per row).
template <int NT, int U, int LPR>
__global__ void __launch_bounds__(NT) batch_cl16_kernel(const uint16_t *__restrict__ A, int64_t lda,
                                                        const uint16_t *__restrict__ x, int64_t rows, int64_t n,
                                                        KParams K, OutSpec O) {
    extern __shared__ __align__(16) uint32_t s_xw[];
    batch_pdl_enter<U, LPR, NT>(A, lda, rows, n / 8, O.prefetch != 0);
    const int64_t nw = (n + 1) / 2;
    const int64_t nwpad = (nw + 3) & ~int64_t(3);
    for (int64_t j = threadIdx.x; j < nwpad; j += NT) {
        uint32_t x0 = 2 * j < n ? x[2 * j] : 0u, x1 = 2 * j + 1 < n ? x[2 * j + 1] : 0u;
        s_xw[j] = (x0 & 0xFFu) | ((x1 & 0xFFu) << 8) | ((x0 >> 8) << 16) | ((x1 >> 8) << 24);
    }
    __syncthreads();
    constexpr int RPW = 32 / LPR;  // rows per warp
    const int lane = threadIdx.x & 31, g = lane % LPR;
    const int64_t nvec = n / 8;
    const uint4 *xv = reinterpret_cast<const uint4 *>(s_xw);
    const int64_t warp0 = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
    const int64_t wstride = (int64_t)gridDim.x * (NT / 32);
    for (int64_t rbase = warp0 * RPW; rbase < rows; rbase += wstride * RPW) {
        const int64_t row = rbase + lane / LPR;
        const bool valid = row < rows;
        const uint16_t *Ar = A + (valid ? row : 0) * lda;
        const uint4 *av = reinterpret_cast<const uint4 *>(Ar);
        uint64_t tot = 0;
        int64_t v0 = g;
        if (valid) {
            // full chunks: U unpredicated 16-byte loads per lane in flight, then 8 DP2A per vector
            for (; v0 + LPR * (U - 1) < nvec; v0 += LPR * U) {
                uint4 ra[U];
#pragma unroll
                for (int u = 0; u < U; ++u) ra[u] = ld_stream(av + v0 + u * LPR);
                uint32_t lo = 0, hi = 0;  // <= 4U dp2a of < 2^25 each: no wrap for U <= 32
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint4 w = xv[v0 + u * LPR];
                    lo = __dp2a_lo(ra[u].x, w.x, lo);
                    hi = __dp2a_hi(ra[u].x, w.x, hi);
                    lo = __dp2a_lo(ra[u].y, w.y, lo);
                    hi = __dp2a_hi(ra[u].y, w.y, hi);
                    lo = __dp2a_lo(ra[u].z, w.z, lo);
                    hi = __dp2a_hi(ra[u].z, w.z, hi);
                    lo = __dp2a_lo(ra[u].w, w.w, lo);
                    hi = __dp2a_hi(ra[u].w, w.w, hi);
                }
                tot += (uint64_t)lo + ((uint64_t)hi << 8);
            }
            for (; v0 < nvec; v0 += LPR) {  // remaining vectors of the row
                const uint4 ra = ld_stream(av + v0), w = xv[v0];
                uint32_t lo = __dp2a_lo(ra.x, w.x, 0u), hi = __dp2a_hi(ra.x, w.x, 0u);
                lo = __dp2a_lo(ra.y, w.y, lo);
                hi = __dp2a_hi(ra.y, w.y, hi);
                lo = __dp2a_lo(ra.z, w.z, lo);
                hi = __dp2a_hi(ra.z, w.z, hi);
                lo = __dp2a_lo(ra.w, w.w, lo);
                hi = __dp2a_hi(ra.w, w.w, hi);
                tot += (uint64_t)lo + ((uint64_t)hi << 8);
            }
            for (int64_t j = nvec * 8 + g; j < n; j += LPR) tot += (uint64_t)Ar[j] * x[j];
        }
        tot = group_sum<LPR>(tot);
        if (valid && g == 0) write_result(mod_p(tot, K.p, K.mu), O, K, row);
    }
    pdl_exit();
}

// ------------------------------------------------------------------------------ batch: Zech matrix-vector
// Zech codes (sec. 2.4), A row-major, x shared by every row.  The product of g^i and g^j costs ONE
// shared-memory lookup per term in either design; this kernel decodes instead of adding indices: each code c
// of A is decoded with one lookup T[c] (T = the antilog table on [0, qbar], T[0] = 0 for the zero element), x
// is decoded once per CTA and staged byte-split as in batch_cl16, and each pair of decoded terms costs two
// DP2A (as C5).  The table holds q entries instead of the 2q - 1 an index sum needs, and there is no zero test
// and no index add or fold per term (the large-field index-add kernel was ALU-bound, 89% ALU pipe).  A warp
// walks RP rows at once, so each staged x read serves RP rows (x reads are a quarter-warp LDS.128: 4
// wavefronts per 256 terms, against ~27 for the random lookups).  The shared-memory gather is the binding
// ceiling.  Row value = sum lo + 256 sum hi, one mod p, log-table encoding.
template <int NT, int U, int MINB, int RP>
__global__ void __launch_bounds__(NT, MINB) batch_zech_kernel(const uint16_t *__restrict__ A, int64_t lda,
                                                              const uint16_t *__restrict__ x, int64_t rows, int64_t n,
                                                              KParams K, OutSpec O, uint32_t tab_entries) {
    extern __shared__ __align__(16) uint16_t s_tab[];
    stage_table(s_tab, K.antilog, tab_entries);  // library-owned table: staged before the PDL wait
    batch_pdl_enter<U, 32, NT>(A, lda, rows, n / 8, O.prefetch != 0);
    uint32_t *s_xw = reinterpret_cast<uint32_t *>(s_tab + tab_entries);  // tab_entries: a multiple of 8
    __syncthreads();
    if (threadIdx.x == 0) s_tab[0] = 0;  // code 0 is the zero element (the doubled layout holds g^0 there)
    __syncthreads();
    const uint32_t qbar = K.qbar, qq = qbar | (qbar << 16);
    // x decoded and byte-split: w_j = (x_{2j} lo, x_{2j+1} lo, x_{2j} hi, x_{2j+1} hi) of the decoded values
    const int64_t nw = (n + 1) / 2, nwpad = (nw + 3) & ~int64_t(3);
    for (int64_t j = threadIdx.x; j < nwpad; j += NT) {
        const uint32_t c0 = 2 * j < n ? min((uint32_t)x[2 * j], qbar) : 0u;
        const uint32_t c1 = 2 * j + 1 < n ? min((uint32_t)x[2 * j + 1], qbar) : 0u;
        const uint32_t x0 = s_tab[c0], x1 = s_tab[c1];
        s_xw[j] = (x0 & 0xFFu) | ((x1 & 0xFFu) << 8) | ((x0 >> 8) << 16) | ((x1 >> 8) << 24);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nvec = n / 8;
    const uint4 *xv = reinterpret_cast<const uint4 *>(s_xw);
    // two decoded codes of one 32-bit word (clamped: non-canonical codes never leave the table) -> packed u16 pair
    auto dec2 = [&](uint32_t w) -> uint32_t {
        const uint32_t c = __vminu2(w, qq);
        return (uint32_t)s_tab[c & 0xFFFFu] | ((uint32_t)s_tab[c >> 16] << 16);
    };
    // one 16-byte vector of 8 codes against the staged x words: 2 DP2A per pair of terms
    auto vec8 = [&](const uint4 a, const uint4 w, uint32_t &lo, uint32_t &hi) {
        uint32_t d = dec2(a.x);
        lo = __dp2a_lo(d, w.x, lo);
        hi = __dp2a_hi(d, w.x, hi);
        d = dec2(a.y);
        lo = __dp2a_lo(d, w.y, lo);
        hi = __dp2a_hi(d, w.y, hi);
        d = dec2(a.z);
        lo = __dp2a_lo(d, w.z, lo);
        hi = __dp2a_hi(d, w.z, hi);
        d = dec2(a.w);
        lo = __dp2a_lo(d, w.w, lo);
        hi = __dp2a_hi(d, w.w, hi);
    };
    const int64_t warp0 = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
    const int64_t wstride = (int64_t)gridDim.x * (NT / 32);
    for (int64_t r0 = warp0 * RP; r0 < rows; r0 += wstride * RP) {
        const uint4 *av[RP];
        uint64_t tot[RP];
#pragma unroll
        for (int k = 0; k < RP; ++k) {
            av[k] = reinterpret_cast<const uint4 *>(A + (r0 + k < rows ? r0 + k : r0) * lda);
            tot[k] = 0;
        }
        int64_t v0 = lane;
        // full chunks: U 16-byte loads per row per lane in flight, then the lookups; x read once per RP rows
        for (; v0 + 32 * (U - 1) < nvec; v0 += 32 * U) {
            uint4 ra[RP][U];
#pragma unroll
            for (int k = 0; k < RP; ++k)
#pragma unroll
                for (int u = 0; u < U; ++u) ra[k][u] = ld_stream(av[k] + v0 + u * 32);
            uint32_t lo[RP], hi[RP];  // <= 4U dp2a of < 2^25 each: no wrap for U <= 32
#pragma unroll
            for (int k = 0; k < RP; ++k) lo[k] = hi[k] = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint4 w = xv[v0 + u * 32];
#pragma unroll
                for (int k = 0; k < RP; ++k) vec8(ra[k][u], w, lo[k], hi[k]);
            }
#pragma unroll
            for (int k = 0; k < RP; ++k) tot[k] += (uint64_t)lo[k] + ((uint64_t)hi[k] << 8);
        }
        for (; v0 < nvec; v0 += 32) {  // remaining vectors of the rows
            const uint4 w = xv[v0];
#pragma unroll
            for (int k = 0; k < RP; ++k) {
                uint32_t lo = 0, hi = 0;
                vec8(ld_stream(av[k] + v0), w, lo, hi);
                tot[k] += (uint64_t)lo + ((uint64_t)hi << 8);
            }
        }
        for (int64_t j = nvec * 8 + lane; j < n; j += 32) {  // scalar tail: decoded x from the byte-split words
            const uint32_t w = s_xw[j >> 1], sh = (j & 1) * 8;
            const uint32_t xvj = ((w >> sh) & 0xFFu) | (((w >> (16 + sh)) & 0xFFu) << 8);
#pragma unroll
            for (int k = 0; k < RP; ++k)
                tot[k] += (uint64_t)s_tab[min((uint32_t)reinterpret_cast<const uint16_t *>(av[k])[j], qbar)] * xvj;
        }
#pragma unroll
        for (int k = 0; k < RP; ++k) {
            const uint64_t t = warp_sum(tot[k]);  // row total < n (p-1)^2 < 2^64 (host-checked)
            if (lane == 0 && r0 + k < rows) write_result(mod_p(t, K.p, K.mu), O, K, r0 + k);
        }
    }
    pdl_exit();
}

// ------------------------------------------------------------------------------ batch: generic
// Row loads: with L >= 8 lanes per row a warp's 16-byte loads cover whole 128-byte lines (streamed past L1);
// with one lane per row each lane walks its own row, so its loads may allocate in L1: the second half of a
// 32-byte sector is then served from L1 instead of a second L2 request.
// 32-byte load (LDG.E.256) of two consecutive 16-byte vectors (32-byte aligned): one lane walking its own row
// fetches a whole sector per request
__device__ __forceinline__ void ld_row256(const uint4 *ptr, uint4 &a, uint4 &b) {
    asm("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(ptr));
}
template <int LPR>
__device__ __forceinline__ uint4 ld_row(const uint4 *ptr) {
    if constexpr (LPR == 1) {
        uint4 r;
        asm("ld.global.nc.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
        return r;
    } else {
        return ld_stream(ptr);
    }
}

// Warp per row with policy R.  x read through the read-only path (L1-resident, reused by every
// row).  VEC: rows and x are 16-byte aligned (A, lda*sizeof, x) -> 16-byte loads.
template <class R, int NT, int U, bool VEC, int LPR, bool XS>
__global__ void __launch_bounds__(NT) batch_kernel(const typename R::elem *__restrict__ A, int64_t lda,
                                                   const typename R::elem *__restrict__ x, int64_t rows,
                                                   int64_t n, KParams K, OutSpec O) {
    extern __shared__ __align__(16) uint16_t s_tab[];
    if constexpr (R::kTable && GFP_STAGE_EARLY) stage_table(s_tab, K.antilog, K.antilog_entries);  // library-owned
    batch_pdl_enter<U, LPR, NT>(A, lda * (int64_t)sizeof(typename R::elem) / 2, rows, VEC ? n / R::W : 0,
                                O.prefetch != 0);
    const uint16_t *tab = nullptr;
    const uint32_t tab_bytes = R::kTable ? ((K.antilog_entries * 2 + 15) & ~15u) : 0;
    if constexpr (R::kTable) {
        if (!GFP_STAGE_EARLY) stage_table(s_tab, K.antilog, K.antilog_entries);
        tab = s_tab;
    }
    // XS: x staged once per CTA in shared memory (16-byte vectors; every row reuses it)
    const uint4 *xs = reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(s_tab) + tab_bytes);
    if constexpr (XS) {
        const int64_t nxv = n / R::W;
        uint4 *d = reinterpret_cast<uint4 *>(reinterpret_cast<char *>(s_tab) + tab_bytes);
        const uint4 *src = reinterpret_cast<const uint4 *>(x);
        for (int64_t i = threadIdx.x; i < nxv; i += NT) d[i] = __ldg(src + i);
    }
    if constexpr (R::kTable || XS) __syncthreads();
    constexpr int RPW = 32 / LPR;
    const int lane = threadIdx.x & 31, g = lane % LPR;
    const int64_t warp0 = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
    const int64_t wstride = (int64_t)gridDim.x * (NT / 32);
    for (int64_t rbase = warp0 * RPW; rbase < rows; rbase += wstride * RPW) {
        const int64_t row = rbase + lane / LPR;
        const bool valid = row < rows;
        const typename R::elem *Ar = A + (valid ? row : 0) * lda;
        typename R::Acc acc;
        R::init(acc);
        if (valid) {
            int64_t done = 0;
            if (VEC) {
                // U 16-byte loads per lane in flight per chunk; the launcher sizes U so that a short row
                // is one chunk (its epilogue then costs one round trip per row, not per chunk)
                const int64_t nvec = n / R::W;
                const uint4 *av = reinterpret_cast<const uint4 *>(Ar);
                const uint4 *xv = XS ? xs : reinterpret_cast<const uint4 *>(x);
                int64_t v0 = g;
                // one lane per row: 32-byte loads when the row is 32-byte aligned (v0 advances by U vectors)
                const bool wide = LPR == 1 && U % 2 == 0 && ((uintptr_t)av & 31) == 0;
                for (; v0 + LPR * (U - 1) < nvec; v0 += LPR * U) {
                    uint4 ra[U];
                    if (LPR == 1 && U % 2 == 0 && wide) {
#pragma unroll
                        for (int u = 0; u < U; u += 2) ld_row256(av + v0 + u, ra[u], ra[u + 1]);
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) ra[u] = ld_row<LPR>(av + v0 + u * LPR);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) R::vec(acc, ra[u], XS ? xv[v0 + u * LPR] : __ldg(xv + v0 + u * LPR), K, tab);
                }
                if (v0 < nvec) {  // a partial chunk: predicated loads, all still in flight together
                    uint4 ra[U];
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (v0 + u * LPR < nvec) ra[u] = ld_row<LPR>(av + v0 + u * LPR);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (v0 + u * LPR < nvec)
                            R::vec(acc, ra[u], XS ? xv[v0 + u * LPR] : __ldg(xv + v0 + u * LPR), K, tab);
                }
                done = nvec * R::W;
            }
            for (int64_t j = done + g; j < n; j += LPR) R::term(acc, Ar[j], x[j], K, tab);
        }
        uint64_t v = group_sum<LPR>(valid ? R::finish(acc, K) : 0);
        if (valid && g == 0)
            write_result(O.rep == GFP_REP_CENTERED ? smod_p((int64_t)v, K) : mod_p(v, K.p, K.mu), O, K, row);
    }
    pdl_exit();
}

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

#ifndef GFP_CONV_FLAT
#define GFP_CONV_FLAT 1  // 1: one U-chunk tile per thread, grid not capped at the resident CTAs (no table)
#endif
#ifndef GFP_ZBATCH_U
#define GFP_ZBATCH_U 4  // 16-byte vectors per lane in flight in the Zech batch (doubled table)
#endif
#ifndef GFP_ZBATCH_DECODE
#define GFP_ZBATCH_DECODE 1  // 1: Zech matrix-vector by decode + DP2A (batch_zech_kernel); 0: index-add batch_kernel
#endif
#ifndef GFP_ZDEC_RP
#define GFP_ZDEC_RP 2  // rows a warp of the decode batch walks at once (each staged x read serves RP rows)
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

template <class R, int NT, int U, bool PIPE>
static cudaError_t launch_dot_t(const DotPlan &P, const KParams &K, const void *a, const void *b, int64_t n,
                                Workspace ws, OutSpec O, cudaStream_t s) {
    auto kern = dot_kernel<R, NT, U, PIPE>;
    occupancy(kern, NT, P.smem);  // sets the smem attribute once
    cudaError_t e = launch_pdl(kern, dim3(P.grid), dim3(NT), P.smem, s, (const typename R::elem *)a,
                               (const typename R::elem *)b, n, P.head, K, ws, O);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <class R, int NT, int U, bool PIPE>
static int dot_occupancy(size_t smem) {
    return occupancy(dot_kernel<R, NT, U, PIPE>, NT, smem);
}

// pure-Zech fast path: small fields (2 qbar < 2^16, byte-offset table) of odd characteristic
static bool zech_add_fast(uint64_t p) { return zech_small_layout(p) && p > 2; }
static bool is_zech(int pol) { return pol >= P_ZS_ALL && pol <= P_ZL_THREAD; }
static bool is_fc(int pol) { return pol >= P_FC0 && pol <= P_FC8; }
static int policy_block(int pol) { return pol == P_ZECH_ADD ? kZaddNT : (is_zech(pol) ? kZechNT : kDotNT); }
static int policy_unroll(int pol) {
    if (pol == P_ZECH_ADD) return kZaddU;
    if (is_fc(pol)) return kFpU;
    if (pol >= P_CL32_ALL && pol <= P_CL16_THREAD) return kClU;
    return is_zech(pol) ? kZechU : ((pol >= P_FP_THREAD && pol <= P_FP_K2) ? kFpU : kDotU);
}
static int policy_width(int pol) {
    if (pol >= P_CS && pol < P_CS_END) return ((pol - P_CS) % 10 >= 5) ? 4 : 8;
    if (pol >= P_CE16_ALL && pol <= P_CE16_BLK) return 8;
    if (pol >= P_CE32_ALL && pol <= P_CE32_BLK) return 4;
    if (is_fc(pol)) return 2;
    if (pol <= P_CL32_OVF || (pol >= P_MONT1 && pol <= P_MONT4) || pol == P_MONT_OVF) return 4;
    if (pol >= P_FP_THREAD && pol <= P_FP_K2) return 2;
    return 8;
}

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

static int policy_occupancy(int pol, size_t smem) {
    switch (pol) {
    case P_CL32_ALL: return dot_occupancy<ClassicalU32<CL_ALL>, kDotNT, kClU, kPipe>(smem);
    case P_CL32_THREAD: return dot_occupancy<ClassicalU32<CL_THREAD>, kDotNT, kClU, kPipe>(smem);
    case P_CL32_OVF: return dot_occupancy<ClassicalU32<CL_OVERFLOW>, kDotNT, kClU, kPipe>(smem);
    case P_CL16_ALL: return dot_occupancy<ClassicalU16<CL_ALL>, kDotNT, kClU, kPipe>(smem);
    case P_CL16_THREAD: return dot_occupancy<ClassicalU16<CL_THREAD>, kDotNT, kClU, kPipe>(smem);
    case P_MONT1: return dot_occupancy<Montgomery<1>, kDotNT, kDotU, kPipe>(smem);
    case P_MONT2: return dot_occupancy<Montgomery<2>, kDotNT, kDotU, kPipe>(smem);
    case P_MONT4: return dot_occupancy<Montgomery<4>, kDotNT, kDotU, kPipe>(smem);
    case P_FP_THREAD: return dot_occupancy<Fp64<0>, kDotNT, kFpU, false>(smem);
    case P_FP_K1: return dot_occupancy<Fp64<1>, kDotNT, kFpU, false>(smem);
    case P_FP_K2: return dot_occupancy<Fp64<2>, kDotNT, kFpU, false>(smem);
    case P_ZS_ALL: return dot_occupancy<Zech<true, true>, kZechNT, kZechU, true>(smem);
    case P_ZS_THREAD: return dot_occupancy<Zech<true, false>, kZechNT, kZechU, true>(smem);
    case P_ZL_ALL: return dot_occupancy<Zech<false, true>, kZechNT, kZechU, true>(smem);
    case P_ZL_THREAD: return dot_occupancy<Zech<false, false>, kZechNT, kZechU, true>(smem);
#define GFP_OCC(pol, ...) \
    case pol: return dot_occupancy<__VA_ARGS__, kDotNT, kDotU, false>(smem);
        GFP_CS_CASES(GFP_OCC)
#undef GFP_OCC
#define GFP_OCC_FC(pol, ...) \
    case pol: return dot_occupancy<__VA_ARGS__, kDotNT, kFpU, false>(smem);
        GFP_FC_CASES(GFP_OCC_FC)
#undef GFP_OCC_FC
    case P_ZECH_ADD: return occupancy(zech_add_dot_kernel<kZaddNT, kZaddU, 2, true>, kZaddNT, smem);
    }
    return 1;
}

cudaError_t launch_dot(const DotPlan &P, const KParams &K0, const void *a, const void *b, int64_t n, Workspace ws,
                       OutSpec O, cudaStream_t s) {
    KParams K = K0;
    K.kblk = P.kblk;
    {  // L2 prefetch of the first chunk before the PDL wait: short streams only (see pdl_enter)
        const int64_t nvec = (n - P.head) / policy_width(P.policy);
        const int64_t per_sweep = (int64_t)std::max(P.grid, 1) * policy_block(P.policy) * policy_unroll(P.policy);
        O.prefetch = nvec <= kPrefetchMaxIters * per_sweep;
    }
    switch (P.policy) {
    case P_CL32_ALL: return launch_dot_t<ClassicalU32<CL_ALL>, kDotNT, kClU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_CL32_THREAD: return launch_dot_t<ClassicalU32<CL_THREAD>, kDotNT, kClU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_CL32_OVF: return launch_dot_t<ClassicalU32<CL_OVERFLOW>, kDotNT, kClU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_CL16_ALL: return launch_dot_t<ClassicalU16<CL_ALL>, kDotNT, kClU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_CL16_THREAD: return launch_dot_t<ClassicalU16<CL_THREAD>, kDotNT, kClU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_MONT1: return launch_dot_t<Montgomery<1>, kDotNT, kDotU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_MONT2: return launch_dot_t<Montgomery<2>, kDotNT, kDotU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_MONT4: return launch_dot_t<Montgomery<4>, kDotNT, kDotU, kPipe>(P, K, a, b, n, ws, O, s);
    case P_FP_THREAD: return launch_dot_t<Fp64<0>, kDotNT, kFpU, false>(P, K, a, b, n, ws, O, s);
    case P_FP_K1: return launch_dot_t<Fp64<1>, kDotNT, kFpU, false>(P, K, a, b, n, ws, O, s);
    case P_FP_K2: return launch_dot_t<Fp64<2>, kDotNT, kFpU, false>(P, K, a, b, n, ws, O, s);
    case P_ZS_ALL: return launch_dot_t<Zech<true, true>, kZechNT, kZechU, true>(P, K, a, b, n, ws, O, s);
    case P_ZS_THREAD: return launch_dot_t<Zech<true, false>, kZechNT, kZechU, true>(P, K, a, b, n, ws, O, s);
    case P_ZL_ALL: return launch_dot_t<Zech<false, true>, kZechNT, kZechU, true>(P, K, a, b, n, ws, O, s);
    case P_ZL_THREAD: return launch_dot_t<Zech<false, false>, kZechNT, kZechU, true>(P, K, a, b, n, ws, O, s);
#define GFP_LAUNCH(pol, ...) \
    case pol: return launch_dot_t<__VA_ARGS__, kDotNT, kDotU, false>(P, K, a, b, n, ws, O, s);
        GFP_CS_CASES(GFP_LAUNCH)
#undef GFP_LAUNCH
#define GFP_LAUNCH_FC(pol, ...) \
    case pol: return launch_dot_t<__VA_ARGS__, kDotNT, kFpU, false>(P, K, a, b, n, ws, O, s);
        GFP_FC_CASES(GFP_LAUNCH_FC)
#undef GFP_LAUNCH_FC
    case P_ZECH_ADD: {
        // fast path for small odd-characteristic fields (p = 2 has qbar = 1: the checked kernel)
        auto kern = zech_add_fast(K.p) ? zech_add_dot_kernel<kZaddNT, kZaddU, 2, true>
                                                        : zech_add_dot_kernel<kZaddNT, kZaddU, 1, false>;
        occupancy(kern, kZaddNT, P.smem);
        cudaError_t e = launch_pdl(kern, dim3(P.grid), dim3(kZaddNT), P.smem, s, (const uint16_t *)a,
                                   (const uint16_t *)b, n, P.head, K, ws, O);
        if (e != cudaSuccess) return e;
        count_launch();
        return cudaGetLastError();
    }
    }
    return cudaErrorInvalidValue;
}

static size_t elem_size(int dt) { return dt == GFP_U16 ? 2 : (dt == GFP_U32 ? 4 : 8); }

// binary64 centered: the largest compiled block KF in {8, 4, 2, 1} not above lambda_c
static int fc_policy(uint64_t lambda_c) {
    return lambda_c >= 8 ? P_FC8 : (lambda_c >= 4 ? P_FC4 : (lambda_c >= 2 ? P_FC2 : P_FC1));
}
static uint64_t fc_block(int pol) { return pol == P_FC8 ? 8 : (pol == P_FC4 ? 4 : (pol == P_FC2 ? 2 : (pol == P_FC1 ? 1 : 0))); }

// Explicit strategy (gfp_options) -> policy and block length; GFP_OK or the reason it is not admissible.
static gfp_status resolve_strategy(const gfp_info &I, int64_t n, const gfp_options *opt, int *pol, uint64_t *kblk,
                                   int *acc_bits) {
    const int strat = opt ? opt->strategy : GFP_STRAT_AUTO;
    const int bits = opt ? opt->acc_bits : 0;
    *kblk = 0;
    *acc_bits = I.acc_bits;
    if (strat < GFP_STRAT_AUTO || strat > GFP_STRAT_CARRY) return GFP_E_INVAL;
    if (strat == GFP_STRAT_ZECH_ADD) {
        if (I.rep != GFP_REP_ZECH || (bits != 0 && bits != 64)) return GFP_E_UNSUPPORTED;
        *pol = P_ZECH_ADD;
        return GFP_OK;
    }
    if (strat == GFP_STRAT_AUTO && bits == 0) return GFP_OK;
    const uint64_t pm1 = I.p - 1;
    const u128 q2 = (u128)pm1 * pm1;
    switch (I.rep) {
    case GFP_REP_CLASSICAL: {
        if (bits != 0 && bits != 32 && bits != 64) return GFP_E_INVAL;
        const int m = bits ? bits : 64;
        const u128 wmax = m == 64 ? (~(u128)0 >> 64) : (((u128)1 << 32) - 1);  // 2^m - 1
        if (q2 + pm1 > wmax) return GFP_E_BOUND;  // an AXPY must fit the m-bit word
        const int s = strat == GFP_STRAT_AUTO ? GFP_STRAT_BLOCKED : strat;
        if (s == GFP_STRAT_DELAYED && (u128)n * q2 > wmax) return GFP_E_BOUND;  // Eq. (1): n <= k
        if (s == GFP_STRAT_BLOCKED) *kblk = q2 == 0 ? UINT64_MAX : (uint64_t)std::min<u128>((wmax - pm1) / q2, UINT64_MAX);
        if (s == GFP_STRAT_HYBRID) {
            const u128 pp = (u128)I.p * pm1;  // Eq. (2): lambda p (p-1) < 2^m
            *kblk = (uint64_t)std::min<u128>(wmax / pp, UINT64_MAX);
            if (*kblk == 0) return GFP_E_BOUND;
        }
        *pol = cs_policy(m == 64, I.dtype == GFP_U32, s);
        *acc_bits = m;
        return GFP_OK;
    }
    case GFP_REP_MONTGOMERY:
        if (bits != 0 && bits != 64) return GFP_E_INVAL;
        if (strat == GFP_STRAT_OVERFLOW) *pol = P_MONT_OVF;
        else if (strat == GFP_STRAT_CARRY) *pol = P_MONT_CARRY;
        else if (strat != GFP_STRAT_AUTO && strat != GFP_STRAT_BLOCKED) return GFP_E_UNSUPPORTED;
        return GFP_OK;
    case GFP_REP_FP64:
        if (bits != 0 && bits != 53) return GFP_E_INVAL;
        if (strat == GFP_STRAT_DELAYED) {
            if ((u128)n * q2 >= ((u128)1 << 53)) return GFP_E_BOUND;
            *pol = P_FP_THREAD;
        } else if (strat == GFP_STRAT_BLOCKED) {
            *pol = I.k >= 2 ? P_FP_K2 : P_FP_K1;
        } else if (strat != GFP_STRAT_AUTO) {
            return GFP_E_UNSUPPORTED;
        }
        return GFP_OK;
    case GFP_REP_ZECH:
        return (strat == GFP_STRAT_AUTO && (bits == 0 || bits == 64)) ? GFP_OK : GFP_E_UNSUPPORTED;
    case GFP_REP_CENTERED: {  // sec. 3.2.2: DELAYED (one reduction at the end) or BLOCKED (lambda_c)
        const bool f64 = I.dtype == GFP_F64;
        if (bits != 0 && bits != (f64 ? 53 : 64)) return GFP_E_INVAL;
        const u128 h = (u128)(I.p - 1) / 2, h2 = h * h;
        if (strat == GFP_STRAT_DELAYED) {
            if (f64 ? (u128)n * h2 + h >= ((u128)1 << 53) : (u128)n * h2 + h > (((u128)1 << 63) - 1))
                return GFP_E_BOUND;
            *pol = f64 ? P_FC0 : (I.dtype == GFP_U16 ? P_CE16_ALL : P_CE32_ALL);
        } else if (strat == GFP_STRAT_BLOCKED || (strat == GFP_STRAT_AUTO && bits != 0)) {
            *pol = f64 ? fc_policy(I.k) : (I.dtype == GFP_U16 ? P_CE16_BLK : P_CE32_BLK);
            *kblk = f64 ? fc_block(*pol) : I.k;
        } else if (strat != GFP_STRAT_AUTO) {
            return GFP_E_UNSUPPORTED;  // the signed overflow trick / hybrid centered
        }
        *acc_bits = f64 ? 53 : 64;
        return GFP_OK;
    }
    }
    return GFP_E_INVAL;
}

static const char *policy_name(int pol) {
    switch (pol) {
    case P_CL32_ALL: return "dot_kernel<ClassicalU32<ALL>>";
    case P_CL32_THREAD: return "dot_kernel<ClassicalU32<THREAD>>";
    case P_CL32_OVF: return "dot_kernel<ClassicalU32<OVERFLOW>>";
    case P_CL16_ALL: return "dot_kernel<ClassicalU16<ALL>>";
    case P_CL16_THREAD: return "dot_kernel<ClassicalU16<THREAD>>";
    case P_MONT1: return "dot_kernel<Montgomery<1>>";
    case P_MONT2: return "dot_kernel<Montgomery<2>>";
    case P_MONT4: return "dot_kernel<Montgomery<4>>";
    case P_FP_THREAD: return "dot_kernel<Fp64<0>>";
    case P_FP_K1: return "dot_kernel<Fp64<1>>";
    case P_FP_K2: return "dot_kernel<Fp64<2>>";
    case P_ZS_ALL: return "dot_kernel<Zech<SMALL,ALL>>";
    case P_ZS_THREAD: return "dot_kernel<Zech<SMALL,THREAD>>";
    case P_ZL_ALL: return "dot_kernel<Zech<LARGE,ALL>>";
    case P_ZL_THREAD: return "dot_kernel<Zech<LARGE,THREAD>>";
    case P_MONT_OVF: return "dot_kernel<MontgomeryOverflow>";
    case P_MONT_CARRY: return "dot_kernel<MontgomeryCarry>";
    case P_ZECH_ADD: return "zech_add_dot_kernel";
    case P_CE16_ALL: return "dot_kernel<CenteredI<i16,ALL>>";
    case P_CE16_THREAD: return "dot_kernel<CenteredI<i16,THREAD>>";
    case P_CE16_BLK: return "dot_kernel<CenteredI<i16,BLOCKED>>";
    case P_CE32_ALL: return "dot_kernel<CenteredI<i32,ALL>>";
    case P_CE32_THREAD: return "dot_kernel<CenteredI<i32,THREAD>>";
    case P_CE32_BLK: return "dot_kernel<CenteredI<i32,BLOCKED>>";
    case P_FC0: return "dot_kernel<Fp64C<0>>";
    case P_FC1: return "dot_kernel<Fp64C<1>>";
    case P_FC2: return "dot_kernel<Fp64C<2>>";
    case P_FC4: return "dot_kernel<Fp64C<4>>";
    case P_FC8: return "dot_kernel<Fp64C<8>>";
    }
    if (pol >= P_CS && pol < P_CS_END) {
        static const char *slot[5] = {"DELAYED", "BLOCKED", "OVERFLOW", "HYBRID", "CARRY"};
        static std::string names[20];
        static std::once_flag once;
        std::call_once(once, [] {
            for (int i = 0; i < 20; ++i)
                names[i] = std::string("ClassicalS<") + (i >= 10 ? "u64acc," : "u32acc,") + (i % 10 >= 5 ? "u32," : "u16,") +
                           slot[i % 5] + ">";
        });
        return names[pol - P_CS].c_str();
    }
    return "?";
}

gfp_status plan_dot(const gfp_info &I, const KParams &K, const void *a, const void *b, int64_t n,
                    const gfp_options *opt, DotPlan *P) {
    if (opt != nullptr && opt->lanes_per_row != 0) return GFP_E_INVAL;  // a batch option (gfp.h)
    gfp_options tuned{};  // AUTO follows the install-time table when it has an admissible entry (F4)
    if ((opt == nullptr || (opt->strategy == GFP_STRAT_AUTO && opt->acc_bits == 0)) &&
        tuned_options(I, 0, n, 0, &tuned) && plan_dot(I, K, a, b, n, &tuned, P) == GFP_OK)
        return GFP_OK;
    const size_t es = elem_size(I.dtype);
    const uint64_t pm1 = I.p - 1;
    const u128 q2 = (u128)pm1 * pm1;
    const u128 max64 = ~(u128)0 >> 64;
    size_t smem = I.rep == GFP_REP_ZECH ? (size_t)K.antilog_entries * 2 : 0;

    // provisional policy (the mode refinement below only depends on per-thread counts)
    int pol = 0;
    switch (I.rep) {
    case GFP_REP_CLASSICAL: pol = I.dtype == GFP_U16 ? P_CL16_THREAD : P_CL32_THREAD; break;
    case GFP_REP_MONTGOMERY: pol = I.mont_kr >= 4 ? P_MONT4 : (I.mont_kr >= 2 ? P_MONT2 : P_MONT1); break;
    case GFP_REP_FP64: pol = I.k >= 2 ? P_FP_K2 : P_FP_K1; break;
    case GFP_REP_ZECH: pol = zech_small_layout(I.p) ? P_ZS_ALL : P_ZL_ALL; break;
    case GFP_REP_CENTERED:
        pol = I.dtype == GFP_F64 ? fc_policy(I.k) : (I.dtype == GFP_U16 ? P_CE16_THREAD : P_CE32_THREAD);
        break;
    }
    int xpol = -1, acc_bits = I.acc_bits;
    uint64_t kblk = 0;
    gfp_status st = resolve_strategy(I, n, opt, &xpol, &kblk, &acc_bits);
    if (st != GFP_OK) return st;
    if (xpol >= 0) pol = xpol;
    if (pol == P_ZECH_ADD) smem = (size_t)(zech_add_fast(I.p) ? K.zplus1s_entries : K.zplus1_entries) * 2;
    const int NT = policy_block(pol), U = policy_unroll(pol), W = policy_width(pol);
    const uintptr_t pa = (uintptr_t)a, pb = (uintptr_t)b;
    int64_t head = n;
    if (pa % 16 == pb % 16) head = std::min<int64_t>(n, (int64_t)(((16 - pa % 16) % 16) / es));
    const int64_t nvec = (n - head) / W;
    const int dev_sms = [] {
        int d = 0;
        cudaGetDevice(&d);
        return num_sms(d);
    }();
    const int bps = policy_occupancy(pol, smem);
    // at least one 16-byte vector per thread before capping at the resident grid: small inputs are
    // latency-bound, so spread them over as many SMs as possible (one DRAM round trip per thread)
    int64_t want = std::max<int64_t>((nvec + NT - 1) / NT, (head + NT - 1) / NT);
    // Long table-free streams run several waves of resident CTAs: one wave per 2^GFP_WAVE_LOG2 bytes of
    // operands, up to GFP_DOT_WAVES (B200 A/B, profiles/r01_waves_ab.txt: C3's 2 GiB 301 -> 291 us with 16
    // waves, C2's 160 MB 22.9 -> 22.1 us with 4); every CTA ends with one packed atomic on one word, so very
    // many CTAs of a short kernel ending together would queue on it.  Centered (signed) dots finish each
    // thread with a signed reduction and keep one wave per 128 MiB.  Table kernels stage their table once per
    // CTA: one wave.  The pure-Zech kernel keeps one workspace slot per CTA after slot 0.
    const bool tab_kernel = is_zech(pol) || pol == P_ZECH_ADD;
    const int wave_log2 = I.rep == GFP_REP_CENTERED ? 27 : GFP_WAVE_LOG2;
    const int64_t waves =
        tab_kernel ? 1 : std::max<int64_t>(1, std::min<int64_t>(GFP_DOT_WAVES, (int64_t)(((u128)n * es * 2) >> wave_log2)));
    const int64_t cap = tab_kernel ? (int64_t)kMaxGrid - (pol == P_ZECH_ADD ? 1 : 0) : (int64_t)INT32_MAX;
    // (dot_kernel's packed combine counts CTA arrivals in 64 - kPackShift bits)
    int64_t grid = std::min<int64_t>({(int64_t)dev_sms * bps * waves, std::max<int64_t>(want, 1), cap,
                                      ((int64_t)1 << (64 - kPackShift)) - 1});
    const int64_t threads = grid * NT;
    const int64_t iters = (nvec + threads * U - 1) / (threads * U);
    const u128 per_thread = (u128)iters * U * W + (head + threads - 1) / threads + 1;

    int acc = GFP_ACC_DELAYED, strat = GFP_STRAT_DELAYED;
    int64_t reductions = 1;  // per thread, bound (delayed: the one final reduction)
    if (xpol < 0) {
        switch (I.rep) {
        case GFP_REP_CLASSICAL:
            if ((u128)n * q2 <= max64) {
                pol = I.dtype == GFP_U16 ? P_CL16_ALL : P_CL32_ALL;  // Eq. (1): k > n, one final remainder
                reductions = 0;
            } else if (per_thread * q2 <= max64) {
                pol = I.dtype == GFP_U16 ? P_CL16_THREAD : P_CL32_THREAD;
            } else if (const uint64_t lam = (uint64_t)std::min<u128>(max64 / ((u128)I.p * pm1), UINT64_MAX);
                       lam >= 4) {
                // sec. 3.4 hybrid, Eq. (2): one wrap test per block of lambda products, lambda p (p-1) < 2^64
                // (B200: 1.07x (dot) / 1.4x (DIM=512 batch) over a test per product at lambda = 4; slower at 2)
                pol = cs_policy(true, true, GFP_STRAT_HYBRID);
                acc = GFP_ACC_OVERFLOW;
                strat = GFP_STRAT_HYBRID;
                kblk = lam;
                reductions = (int64_t)(per_thread / lam) + 1;
            } else {
                // sec. 3.3 division on demand with the carry word (lambda < 4: p > ~2^31.5, u32 storage): the
                // carry flag of each 64-bit add counted, one reduction per thread (B200: replaces a wrap test
                // + CORR per product, 1.15 T terms/s at p = 4294967291)
                pol = cs_policy(true, true, GFP_STRAT_CARRY);
                acc = GFP_ACC_OVERFLOW;
                strat = GFP_STRAT_CARRY;
                reductions = 1;
            }
            break;
        case GFP_REP_MONTGOMERY:
            acc = GFP_ACC_BLOCKED;
            strat = GFP_STRAT_BLOCKED;
            kblk = pol == P_MONT4 ? 4 : (pol == P_MONT2 ? 2 : 1);
            reductions = (int64_t)(per_thread / kblk) + 1;  // REDCs
            break;
        case GFP_REP_FP64:
            if (per_thread * q2 < ((u128)1 << 53)) {
                pol = P_FP_THREAD;
            } else {
                acc = GFP_ACC_BLOCKED;
                strat = GFP_STRAT_BLOCKED;
                kblk = pol == P_FP_K2 ? 2 : 1;
                reductions = (int64_t)(per_thread / kblk) + 1;
            }
            break;
        case GFP_REP_ZECH: {
            const bool small = zech_small_layout(I.p);
            if ((u128)n * pm1 <= max64) {
                pol = small ? P_ZS_ALL : P_ZL_ALL;
                reductions = 0;
            } else {
                pol = small ? P_ZS_THREAD : P_ZL_THREAD;
            }
            break;
        }
        case GFP_REP_CENTERED: {  // sec. 3.2.2: the doubled block, lambda_c h^2 + h < 2^(m-1)
            const u128 h = (u128)(I.p - 1) / 2, h2 = h * h, w63 = ((u128)1 << 63) - 1;
            if (I.dtype == GFP_F64) {
                if (per_thread * h2 + h < ((u128)1 << 53)) {
                    pol = P_FC0;
                } else {
                    acc = GFP_ACC_BLOCKED;
                    strat = GFP_STRAT_BLOCKED;
                    kblk = fc_block(pol);
                    reductions = (int64_t)(per_thread / kblk) + 1;
                }
            } else if ((u128)n * h2 + h <= w63) {
                pol = I.dtype == GFP_U16 ? P_CE16_ALL : P_CE32_ALL;  // one final reduction
                reductions = 0;
            } else if (per_thread * h2 + h <= w63) {
                pol = I.dtype == GFP_U16 ? P_CE16_THREAD : P_CE32_THREAD;
            } else {
                pol = I.dtype == GFP_U16 ? P_CE16_BLK : P_CE32_BLK;
                acc = GFP_ACC_BLOCKED;
                strat = GFP_STRAT_BLOCKED;
                kblk = I.k;
                reductions = (int64_t)(per_thread / kblk) + 1;
            }
            break;
        }
        }
    } else {
        strat = (pol >= P_CS && pol < P_CS_END) ? cs_strategy(pol)
                : (pol == P_MONT_OVF ? GFP_STRAT_OVERFLOW
                   : (pol == P_MONT_CARRY ? GFP_STRAT_CARRY : (opt ? opt->strategy : GFP_STRAT_AUTO)));
        if (strat == GFP_STRAT_AUTO) strat = GFP_STRAT_BLOCKED;
        if (pol == P_ZECH_ADD) strat = GFP_STRAT_ZECH_ADD;  // no integer accumulator at all

        acc = strat == GFP_STRAT_OVERFLOW || strat == GFP_STRAT_HYBRID || strat == GFP_STRAT_CARRY ? GFP_ACC_OVERFLOW
              : (strat == GFP_STRAT_BLOCKED ? GFP_ACC_BLOCKED : GFP_ACC_DELAYED);
        if (pol == P_FP_K2 || pol == P_FP_K1) kblk = pol == P_FP_K2 ? 2 : 1;
        if (is_fc(pol)) kblk = fc_block(pol);
        if (strat == GFP_STRAT_OVERFLOW || strat == GFP_STRAT_ZECH_ADD) {
            reductions = (int64_t)per_thread;  // one wrap test / one Zech addition (table lookup) per term
            if (pol == P_ZECH_ADD) acc_bits = 0;
        } else if (strat == GFP_STRAT_CARRY) {
            reductions = 1;  // the carry flag is counted, never tested: one reduction per thread at the end
        } else if (strat == GFP_STRAT_BLOCKED || strat == GFP_STRAT_HYBRID)
            reductions = (int64_t)(kblk ? per_thread / kblk : 0) + 1;
    }
    P->policy = pol;
    P->grid = (int)grid;
    P->block = NT;
    P->smem = smem;
    P->head = head;
    P->acc = acc;
    P->strategy = strat;
    P->acc_bits = acc_bits;
    P->kblk = kblk;
    P->per_thread = (int64_t)per_thread;
    P->reductions = reductions;
    P->name = policy_name(pol);
    return GFP_OK;
}

cudaError_t launch_finalize(const KParams &K, const uint64_t *summed, int count, OutSpec O, cudaStream_t s) {
    finalize_kernel<<<1, 32, 0, s>>>(summed, count, K, O);
    count_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ batch launch
constexpr size_t kBatchSmemX = 200 * 1024;  // table + staged x, per CTA
#ifndef GFP_BATCH_U
#define GFP_BATCH_U 4
#endif
constexpr int kBatchU = GFP_BATCH_U;  // 16-byte A vectors in flight per lane (generic batch kernel)

template <class R, int NT, int U, int LPR>
static cudaError_t launch_batch_lpr(const KParams &K, const void *A, int64_t lda, const void *x, int64_t rows,
                                   int64_t n, bool vec, int64_t grid, OutSpec O, cudaStream_t s) {
    using E = typename R::elem;
    const size_t tab = R::kTable ? (((size_t)K.antilog_entries * 2 + 15) & ~size_t(15)) : 0;
    const size_t xbytes = (size_t)(n / R::W) * 16;
    // x in shared memory when it fits beside the table (every row reuses it; L1 is not needed for it)
    const bool xs = vec && (R::kTable ? tab + xbytes <= kBatchSmemX : xbytes <= 32 * 1024);
    const size_t smem = tab + (xs ? xbytes : 0);
    auto kern = vec ? (xs ? batch_kernel<R, NT, U, true, LPR, true> : batch_kernel<R, NT, U, true, LPR, false>)
                    : batch_kernel<R, NT, U, false, LPR, false>;
    occupancy(kern, NT, smem);  // sets the shared-memory opt-in
    cudaError_t e = launch_pdl(kern, dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(NT), smem, s, (const E *)A, lda,
                               (const E *)x, rows, n, K, O);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <class R, int NT, int U, int LPR>
static int batch_occupancy(const KParams &K, int64_t n, bool vec) {
    const size_t tab = R::kTable ? (((size_t)K.antilog_entries * 2 + 15) & ~size_t(15)) : 0;
    const size_t xbytes = (size_t)(n / R::W) * 16;
    const bool xs = vec && (R::kTable ? tab + xbytes <= kBatchSmemX : xbytes <= 32 * 1024);
    const size_t smem = tab + (xs ? xbytes : 0);
    auto kern = vec ? (xs ? batch_kernel<R, NT, U, true, LPR, true> : batch_kernel<R, NT, U, true, LPR, false>)
                    : batch_kernel<R, NT, U, false, LPR, false>;
    return occupancy(kern, NT, smem);
}

// Lanes per row and grid.  A row is summed by LPR lanes (RPW = 32 / LPR rows per warp) with U 16-byte loads per
// lane in flight per chunk (U = 4: larger U makes the heavier policies spill into fewer resident warps).  The
// grid spreads the rows over as few CTAs as the resident sweeps need (no partially filled last sweep).
template <class R, int NT, int U, int LPR>
static cudaError_t launch_batch_shape(const KParams &K, const void *A, int64_t lda, const void *x, int64_t rows,
                                      int64_t n, bool vec, OutSpec O, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int bps = batch_occupancy<R, NT, U, LPR>(K, n, vec);
    const int64_t rpb = (NT / 32) * (32 / LPR), gmax = (int64_t)num_sms(dev) * bps;
    const int64_t sweeps = std::max<int64_t>((rows + gmax * rpb - 1) / (gmax * rpb), 1);
    const int64_t grid = (rows + sweeps * rpb - 1) / (sweeps * rpb);
    return launch_batch_lpr<R, NT, U, LPR>(K, A, lda, x, rows, n, vec, grid, O, s);
}

// Lanes per row of the generic batch kernel: the caller's gfp_options.lanes_per_row, else a full warp per
// long row (>= 256 vectors) or per table-kernel row, else 8 lanes (4 rows per warp).
static int batch_lanes(int64_t n, int W, bool table, int want) {
    if (want != 0) return want;
    return (n / W >= 256 || table) ? 32 : 8;
}
// Upper bound on the terms ONE lane of a row sums in batch_kernel with L lanes per row: vectors g, g + L, ...
// of W terms each plus every L-th scalar tail term, or (unvectorised rows) every L-th term.  The built-in
// plan's per-lane overflow tests (Eq. (1) per accumulator) use it with the L the launch will use.
static u128 batch_per_lane(int64_t n, int W, int L) {
    const int64_t nvec = n / W;
    const u128 v = (u128)((nvec + L - 1) / L) * W + (u128)((n - nvec * W + L - 1) / L);
    return std::max<u128>(v, (u128)((n + L - 1) / L));
}
// policies a single lane may own a whole row for (integer storage; gfp.h lanes_per_row = 1)
template <class R>
constexpr bool kOneLaneOk = !R::kTable && !std::is_same<typename R::elem, double>::value;

template <class R, int NT, int U>
static cudaError_t launch_batch_t(const KParams &K, const void *A, int64_t lda, const void *x, int64_t rows,
                                  int64_t n, bool vec, int lanes, OutSpec O, cudaStream_t s) {
    switch (batch_lanes(n, R::W, R::kTable, lanes)) {
    case 1:
        if constexpr (kOneLaneOk<R>) return launch_batch_shape<R, NT, U, 1>(K, A, lda, x, rows, n, vec, O, s);
        return cudaErrorInvalidValue;  // excluded by launch_batch
    case 8: return launch_batch_shape<R, NT, U, 8>(K, A, lda, x, rows, n, vec, O, s);
    default: return launch_batch_shape<R, NT, U, 32>(K, A, lda, x, rows, n, vec, O, s);
    }
}

gfp_status launch_batch(const gfp_info &I, const KParams &K, const void *A, int64_t lda, const void *x, int64_t rows,
                        int64_t n, const gfp_options *opt, OutSpec O, cudaStream_t s, cudaError_t *err) {
    O.prefetch = 1;  // first row chunk into L2 before the PDL wait (B200 A/B: C5 -1.5%)
    const size_t es = elem_size(I.dtype);
    const bool vec = ((uintptr_t)A % 16 == 0) && ((uintptr_t)x % 16 == 0) && ((lda * (int64_t)es) % 16 == 0);
    const uint64_t pm1 = I.p - 1;
    const u128 q2 = (u128)pm1 * pm1, max64 = ~(u128)0 >> 64;
    const int lanes = opt ? opt->lanes_per_row : 0;
    if (lanes != 0 && lanes != 1 && lanes != 8 && lanes != 32) return GFP_E_INVAL;
    // one lane per row: integer storage only (no table, no binary64), gfp.h
    if (lanes == 1 && (I.rep == GFP_REP_ZECH || I.rep == GFP_REP_FP64 || I.dtype == GFP_F64)) return GFP_E_UNSUPPORTED;
    // terms one accumulator sums for a policy of W elements per vector (batch_lanes / batch_per_lane)
    auto per_lane = [&](int W) { return batch_per_lane(n, W, batch_lanes(n, W, false, lanes)); };
    int dev = 0;
    cudaGetDevice(&dev);
    *err = cudaSuccess;
    gfp_options tuned{};  // AUTO follows the install-time table when it has an admissible entry (F4)
    if ((opt == nullptr || (opt->strategy == GFP_STRAT_AUTO && opt->acc_bits == 0 && opt->lanes_per_row == 0)) &&
        tuned_options(I, 1, n, rows, &tuned)) {
        int xpol = -1, acc_bits = 0;
        uint64_t kblk = 0;
        if (resolve_strategy(I, n, &tuned, &xpol, &kblk, &acc_bits) == GFP_OK && xpol >= 0 && xpol != P_ZECH_ADD)
            opt = &tuned;
    }
    {  // explicit strategy (gfp_dot_batch_ex): the generic warp-per-row kernel with that policy
        int xpol = -1, acc_bits = 0;
        uint64_t kblk = 0;
        gfp_status st = resolve_strategy(I, n, opt, &xpol, &kblk, &acc_bits);
        if (st != GFP_OK) return st;
        if (xpol >= 0) {
            KParams K2 = K;
            K2.kblk = kblk;
            switch (xpol) {
#define GFP_BATCH(pol, ...) \
    case pol: *err = launch_batch_t<__VA_ARGS__, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s); break;
                GFP_CS_CASES(GFP_BATCH)
#undef GFP_BATCH
            case P_FP_THREAD: *err = launch_batch_t<Fp64<0>, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s); break;
            case P_FP_K2: *err = launch_batch_t<Fp64<2>, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s); break;
            case P_FP_K1: *err = launch_batch_t<Fp64<1>, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s); break;
#define GFP_BATCH_FC(pol, ...) \
    case pol: *err = launch_batch_t<__VA_ARGS__, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s); break;
                GFP_FC_CASES(GFP_BATCH_FC)
#undef GFP_BATCH_FC
            default: return GFP_E_UNSUPPORTED;
            }
            return *err == cudaSuccess ? GFP_OK : GFP_E_CUDA;
        }
    }
    switch (I.rep) {
    case GFP_REP_CLASSICAL:
        if (I.dtype == GFP_U16) {
            if (vec && lanes == 0 && (u128)n * q2 <= max64 && n <= 96 * 1024) {
                constexpr int NT = 256;
                const bool long_rows = n / 8 >= 256;
                auto kern = long_rows ? batch_cl16_kernel<NT, GFP_CL16_U, 32> : batch_cl16_kernel<NT, 8, 8>;
                const int64_t rpb = long_rows ? NT / 32 : NT / 8;  // rows per CTA per sweep
                const size_t smem = (size_t)(((n + 1) / 2 + 3) & ~int64_t(3)) * 4;
                int bps = occupancy(kern, NT, smem);
                int64_t grid = std::min<int64_t>((rows + rpb - 1) / rpb, (int64_t)num_sms(dev) * bps * GFP_BATCH_WAVES);
                cudaError_t le = launch_pdl(kern, dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(NT), smem, s,
                                            (const uint16_t *)A, lda, (const uint16_t *)x, rows, n, K, O);
                if (le != cudaSuccess) {
                    *err = le;
                    return GFP_E_CUDA;
                }
                count_launch();
                *err = cudaGetLastError();
            } else if (per_lane(8) * q2 <= max64) {
                *err = (u128)n * q2 <= max64
                           ? launch_batch_t<ClassicalU16<CL_ALL>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s)
                           : launch_batch_t<ClassicalU16<CL_THREAD>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
            } else {
                return GFP_E_UNSUPPORTED;
            }
        } else {
            const uint64_t lam = (uint64_t)std::min<u128>(max64 / ((u128)I.p * pm1), UINT64_MAX);
            KParams K2 = K;
            K2.kblk = lam;
            if ((u128)n * q2 <= max64)
                *err = launch_batch_t<ClassicalU32<CL_ALL>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
            else if (per_lane(4) * q2 <= max64)
                *err = launch_batch_t<ClassicalU32<CL_THREAD>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
            else if (lam >= 4)  // sec. 3.4 hybrid (Eq. (2)), as in plan_dot
                *err = launch_batch_t<ClassicalS<uint64_t, uint32_t, S_HYBRID>, 256, kBatchU>(K2, A, lda, x, rows, n,
                                                                                            vec, lanes, O, s);
            else  // lambda < 4: the carry word (as plan_dot)
                *err = launch_batch_t<ClassicalS<uint64_t, uint32_t, S_CARRY>, 256, kBatchU>(K, A, lda, x, rows, n, vec,
                                                                                           lanes, O, s);
        }
        break;
    case GFP_REP_MONTGOMERY:
        if (I.mont_kr >= 4)
            *err = launch_batch_t<Montgomery<4>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
        else if (I.mont_kr >= 2)
            *err = launch_batch_t<Montgomery<2>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
        else
            *err = launch_batch_t<Montgomery<1>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
        break;
    case GFP_REP_FP64:
        if (per_lane(2) * q2 < ((u128)1 << 53))
            *err = launch_batch_t<Fp64<0>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
        else if (I.k >= 2)
            *err = launch_batch_t<Fp64<2>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
        else
            *err = launch_batch_t<Fp64<1>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
        break;
    case GFP_REP_ZECH: {
        // decode kernel (batch_zech_kernel) for aligned rows: one lookup per term in a q-entry table; the row
        // total n (p-1)^2 must fit the u64 (always for n < 2^32)
        const uint32_t zentries = (uint32_t)((I.p + 7) & ~7ull);  // codes [0, qbar] = p entries
        const size_t zsmem = (size_t)zentries * 2 + (size_t)(((n + 1) / 2 + 3) & ~int64_t(3)) * 4;
        if (GFP_ZBATCH_DECODE && vec && lanes == 0 && (u128)n * q2 <= max64 && zsmem <= kBatchSmemX) {
            const uint32_t entries = zentries;
            const size_t smem = zsmem;
            // one 1024-thread CTA per SM (64 registers: U = 4 vectors per row and lane for RP = 2 rows in flight);
            // B200 A/B (scripts/ab_zbatch.py, GF(32749) / GF(65521)): three 512-thread CTAs at 40 registers
            // (U = 2) 152.7 / - us, RP = 1 137.8 / 138.1, RP = 4 (U = 1) 148.7 / 149.1, this 130.7 (65521);
            // a register ping-pong pipeline over (row, chunk) spilled and ran 173-190 us
            auto kern = batch_zech_kernel<1024, GFP_ZDEC_U, 1, GFP_ZDEC_RP>;
            const int bps = occupancy(kern, 1024, smem);
            const int64_t rpb = 32 * GFP_ZDEC_RP;  // rows per CTA per sweep (a warp per RP rows)
            const int64_t grid = std::min<int64_t>((rows + rpb - 1) / rpb, (int64_t)num_sms(dev) * bps);
            cudaError_t le = launch_pdl(kern, dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(1024), smem, s,
                                        (const uint16_t *)A, lda, (const uint16_t *)x, rows, n, K, O, entries);
            count_launch();
            *err = le != cudaSuccess ? le : cudaGetLastError();
            break;
        }
        // index-add kernel (batch_kernel<Zech>): unaligned rows or an explicit lanes_per_row.
        // unroll A/B (scripts/ab_zbatch.py): U = 4 for the doubled table, 8 for the folded large-field one
        if (zech_small_layout(I.p))
            *err = launch_batch_t<Zech<true, false>, 1024, GFP_ZBATCH_U>(K, A, lda, x, rows, n, vec, lanes, O, s);
        else
            *err = launch_batch_t<Zech<false, false>, 1024, GFP_ZBATCH_UL>(K, A, lda, x, rows, n, vec, lanes, O, s);
        break;
    }
    case GFP_REP_CENTERED: {  // sec. 3.2.2: per-row sums; one reduction per lane unless a row overflows
        const u128 h = (u128)(I.p - 1) / 2, h2 = h * h, w63 = ((u128)1 << 63) - 1;
        KParams K2 = K;
        K2.kblk = I.k;
        if (I.dtype == GFP_F64) {
            if (per_lane(2) * h2 + h < ((u128)1 << 53))
                *err = launch_batch_t<Fp64C<0>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s);
            else
                switch (fc_policy(I.k)) {
                case P_FC8: *err = launch_batch_t<Fp64C<8>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s); break;
                case P_FC4: *err = launch_batch_t<Fp64C<4>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s); break;
                case P_FC2: *err = launch_batch_t<Fp64C<2>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s); break;
                default: *err = launch_batch_t<Fp64C<1>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s); break;
                }
        } else if (I.dtype == GFP_U16) {
            *err = (u128)n * h2 + h <= w63 ? launch_batch_t<CenteredI<int16_t, CE_ALL>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s)
                                          : launch_batch_t<CenteredI<int16_t, CE_BLOCKED>, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s);
        } else {
            *err = (u128)n * h2 + h <= w63 ? launch_batch_t<CenteredI<int32_t, CE_ALL>, 256, kBatchU>(K, A, lda, x, rows, n, vec, lanes, O, s)
                                          : launch_batch_t<CenteredI<int32_t, CE_BLOCKED>, 256, kBatchU>(K2, A, lda, x, rows, n, vec, lanes, O, s);
        }
        break;
    }
    }
    return *err == cudaSuccess ? GFP_OK : GFP_E_CUDA;
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
