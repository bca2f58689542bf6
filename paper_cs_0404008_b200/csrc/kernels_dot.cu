// kernels_dot.cu -- single dots (SURVEY.md 8(a) a3-a7, a9 fused): dot_kernel (persistent grid-stride streaming
// of both operands with 16-byte loads, per-thread delayed-modulus accumulation by policy R of device.cuh,
// warp-shuffle + CTA tree, one packed atomic per CTA, last-CTA-done final reduction and encoding; with OUT_XCHG
// the last CTA also exchanges the partial with the peer GPUs over NVLink peer memory), the pure-Zech dot (F3),
// finalize, the exchange-buffer setup kernel, and the dot planner (plan_dot / launch_dot).
#include "kernels_common.cuh"

namespace gfp {

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

// ------------------------------------------------------------------------------ single dot

// CO: a and b co-aligned (bshift == 0, the common case: its code carries no realignment); !CO: the instance for
// operands whose 16-byte alignments differ (built-in policies only; see plan_dot)
template <class R, int NT, int U, bool PIPE, bool CO = true>
__global__ void __launch_bounds__(NT) dot_kernel(const typename R::elem *__restrict__ a,
                                                 const typename R::elem *__restrict__ b, int64_t n,
                                                 int64_t head, int bshift, KParams K, Workspace ws, OutSpec O) {
    extern __shared__ __align__(16) uint16_t s_tab[];
    __shared__ uint64_t red[32];
    typename R::Acc acc;
    R::init(acc);
    const int64_t gtid = (int64_t)blockIdx.x * NT + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * NT;
    // bshift != 0: b is not co-aligned with a (its element `head` sits bshift bytes past a 16-byte boundary):
    // every 16-byte window of b is re-assembled from the two aligned vectors it straddles (realign16), and the
    // last vector goes to the scalar tail, so that no load reaches past b's last element
    const int64_t nvec = (!CO && (n - head) / R::W > 0) ? (n - head) / R::W - 1 : (n - head) / R::W;
    const uint4 *av = reinterpret_cast<const uint4 *>(a + head);
    const uint4 *bv = CO ? reinterpret_cast<const uint4 *>(b + head)
                         : reinterpret_cast<const uint4 *>(reinterpret_cast<uintptr_t>(b + head) & ~uintptr_t(15));
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
    bool have = PIPE && CO && i0 + (U - 1) * NT < nvec;  // (not co-aligned: the plain loop below)
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
    if constexpr (PIPE && CO) {
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

    // scalar head (the elements before a's first 16-byte boundary)
    for (int64_t i = gtid; i < head; i += gstride) R::term(acc, a[i], b[i], K, tab);

    // 16-byte vector body (!PIPE, or b not co-aligned): U independent loads of each operand in flight per thread
    auto ldb = [&](int64_t i) -> uint4 {
        if constexpr (CO) return ld_stream(bv + i);
        else return realign16(ld_stream(bv + i), ld_stream(bv + i + 1), bshift);
    };
    for (; i0 + (U - 1) * NT < nvec; i0 += step) {
        uint4 xa[U], xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xa[u] = ld_stream(av + i0 + u * NT);
            xb[u] = ldb(i0 + u * NT);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) R::vec(acc, xa[u], xb[u], K, tab);
    }
    if (i0 < nvec) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * NT < nvec) R::vec(acc, ld_stream(av + i0 + u * NT), ldb(i0 + u * NT), K, tab);
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
            else if (O.mode == OUT_MC) r = mc_allreduce(r, O.xchg, O.mc, K.p, K.mu);  // the same over NVLS
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
            else if (O.mode == OUT_MC) r = mc_allreduce(r, O.xchg, O.mc, K.p, K.mu);
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

// policies with a non-co-aligned instance (the built-in plans; explicit strategies take the scalar path then)
template <class R>
struct MisOk : std::false_type {};
template <int M>
struct MisOk<ClassicalU32<M>> : std::true_type {};
template <int M>
struct MisOk<ClassicalU16<M>> : std::true_type {};
template <int KR>
struct MisOk<Montgomery<KR>> : std::true_type {};
template <int KF>
struct MisOk<Fp64<KF>> : std::true_type {};
template <bool SM, bool ALL>
struct MisOk<Zech<SM, ALL>> : std::true_type {};
template <>
struct MisOk<ClassicalS<uint64_t, uint32_t, S_HYBRID>> : std::true_type {};
template <>
struct MisOk<ClassicalS<uint64_t, uint32_t, S_CARRY>> : std::true_type {};
// the host side of MisOk: policies whose launch can take bshift != 0
static bool mis_ok(int pol) {
    return (pol >= P_CL32_ALL && pol <= P_ZL_THREAD) || pol == cs_policy(true, true, GFP_STRAT_HYBRID) ||
           pol == cs_policy(true, true, GFP_STRAT_CARRY);
}

template <class R, int NT, int U, bool PIPE>
static cudaError_t launch_dot_t(const DotPlan &P, const KParams &K, const void *a, const void *b, int64_t n,
                                Workspace ws, OutSpec O, cudaStream_t s) {
    auto kern = dot_kernel<R, NT, U, PIPE, true>;
    if constexpr (MisOk<R>::value)
        if (P.bshift != 0) kern = dot_kernel<R, NT, U, PIPE, false>;
    occupancy(kern, NT, P.smem);  // sets the smem attribute once
    cudaError_t e = launch_pdl(kern, dim3(P.grid), dim3(NT), P.smem, s, (const typename R::elem *)a,
                               (const typename R::elem *)b, n, P.head, P.bshift, K, ws, O);
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

// Explicit strategy (gfp_options) -> policy and block length; GFP_OK or the reason it is not admissible.
gfp_status resolve_strategy(const gfp_info &I, int64_t n, const gfp_options *opt, int *pol, uint64_t *kblk,
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
    // head: the elements before a's first 16-byte boundary; bshift: how far b's matching element sits past a
    // 16-byte boundary (0 = co-aligned).  The pure-Zech kernel keeps the scalar path for non-co-aligned inputs.
    const uintptr_t pa = (uintptr_t)a, pb = (uintptr_t)b;
    int64_t head = std::min<int64_t>(n, (int64_t)(((16 - pa % 16) % 16) / es));
    int bshift = (int)((pb + (uintptr_t)head * es) % 16);
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
    // operands not co-aligned: the built-in policies have a realigning kernel instance (MisOk); the other
    // explicit strategies and the pure-Zech kernel take the scalar path over the whole input
    if (bshift != 0 && !mis_ok(pol)) {
        head = n;
        bshift = 0;
    }
    P->policy = pol;
    P->grid = (int)grid;
    P->block = NT;
    P->smem = smem;
    P->head = head;
    P->bshift = bshift;
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

}  // namespace gfp
