// kernels_batch.cu -- batched dots and the GF(p) matrix-vector product: batch_cl16_kernel
// (C5: classical u16, x byte-split in shared memory, two DP2A per pair), batch_zech_kernel (Zech codes: one
// antilog lookup decodes each code of A), the generic batch_kernel (any policy, 1 / 8 / 32 lanes per row), and
// their launcher (launch_batch).
#include "kernels_common.cuh"

namespace gfp {

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

// ------------------------------------------------------------------------------ batch: Zech matrix-vector, split exponent
// Zech codes (sec. 2.4): a nonzero code c in [1, qbar] is g^c.  Write e = c - 1 = 256 h + l (16 bits):
// g^c = H[h] L[l] with L[l] = g^(l + 1) and H[h] = g^(256 h), two lookups into 256-entry tables instead of one
// into a q-entry table.  The small tables are REPLICATED per bank: row r of the table region is 256 bytes,
// words [0, 32) hold L[r] 32 times and words [32, 64) H[r] 32 times, so lane i reads word i (+ 32) of its row
// and a warp-wide lookup touches 32 distinct banks -- ONE shared-memory wavefront, where a random lookup into
// the q-entry table costs ~3.4 (the most distinct words one bank is asked for).  Two conflict-free
// lookups per term (2 wavefronts per 32 terms) against 3.37 move the L1TEX data-pipe floor of the matrix-vector
// product from ~116 us to ~75 us at 65536 x 4096, about the HBM floor (~72 us at the read ceiling).
// Addresses are built by byte permutes: the table region sits at the absolute shared address 0x10000 (64 KB
// aligned), so a row address is the byte pattern [lane*4 (+128), row, 0x01, 0] -- one PRMT from e and a base
// register per lookup.  The zero code:
//   FLAG = false (p <= 65281, so e <= qbar - 1 < 0xFF00): e = c - 1 per 16-bit half (one VIADD.16x2 per pair of
//     codes) sends code 0 to e = 0xFFFF, whose row h = 255 no nonzero code uses: H[255] = 0.
//   FLAG = true (any p): t = c + 0xFFFF in 32 bits holds e in bytes 0-1 and [c != 0] in byte 2; the H address
//     takes byte 2 of t as its 64 KB page, so code 0 reads the zero words at absolute 0xFF80 + 4 lane instead.
// Products: v = L H < p^2 < 2^32 (one IMAD), v x_j < 2^48 added into a u64 per row and lane (one IMAD.WIDE);
// the row total n (p - 1)^3 < 2^64 is host-checked.  x is decoded once per CTA and staged as u16 (one LDS.128 per
// 8 columns serves the RP rows of a warp), rows end with one mod p and the log-table encoding.
constexpr uint32_t kZsTab = 0x10000u;  // absolute shared address of the split table (256 rows x 256 bytes)
constexpr int64_t kZsXBytes = 0xFF80 - 0x1000;  // staged x below the zero words, allowing 4 KB of reserved base
template <int NT, int U, int RP, bool FLAG>
__global__ void __launch_bounds__(NT, 1) batch_zsplit_kernel(const uint16_t *__restrict__ A, int64_t lda,
                                                              const uint16_t *__restrict__ x, int64_t rows, int64_t n,
                                                              KParams K, OutSpec O) {
    extern __shared__ __align__(16) uint16_t s_x[];  // decoded x (u16), below the table; smem = 128 KB
    const uint32_t sx = (uint32_t)__cvta_generic_to_shared(s_x);
    const uint32_t qbar = K.qbar;
    // the split table (library-owned values): staged before the PDL wait
    for (uint32_t i = threadIdx.x; i < 4096; i += NT) {  // 16-byte pieces: row i / 16, piece i % 16
        const uint32_t r = i >> 4;
        const bool hi = (i & 15) >= 8;
        const uint32_t ex = hi ? 256 * r : r + 1, t = ex % qbar;  // exponent in [1, qbar] (g^qbar = g^0)
        uint32_t v = K.antilog[t == 0 ? qbar : t];
        if (!FLAG && hi && r == 255) v = 0;  // the zero code's row (e = 0xFFFF)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(kZsTab + 16 * i), "r"(v) : "memory");
    }
    if (FLAG && threadIdx.x < 8)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(kZsTab - 128 + 16 * threadIdx.x), "r"(0u) : "memory");
    batch_pdl_enter<U, 32, NT>(A, lda, rows, n / 8, true);
    // x decoded (0 for the zero code, g^c else) in the vector layout: vector slots [0, 32 vpl) of which those at
    // or past nvec hold zeros (a lane without a vector there re-reads a valid one: its products vanish), then
    // the < 8 tail elements
    const int64_t nvec = n / 8;
    const int vpl = (int)max((nvec + 31) / 32, (int64_t)1);  // 16-byte vectors per row, per lane
    const int64_t xtail = 256 * (int64_t)vpl, nxs = xtail + 8;
    if (sx + 2 * (uint64_t)nxs > kZsTab - 128) __trap();  // host-checked: x fits below the table
    for (int64_t j = threadIdx.x; j < nxs; j += NT) {
        const int64_t src = j < xtail ? (j < nvec * 8 ? j : n) : nvec * 8 + (j - xtail);
        const uint32_t c = src < n ? min((uint32_t)x[src], qbar) : 0u;
        s_x[j] = c == 0 ? (uint16_t)0 : K.antilog[c];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t bL = kZsTab | (4u * lane), bH = (FLAG ? 0u : kZsTab) | (4u * lane + 128u);
    auto lds = [](uint32_t a) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
        return v;
    };
    // two codes of one 32-bit word against their decoded x values
    auto pair = [&](uint32_t w, uint32_t xa, uint32_t xb, uint64_t &acc) {
        uint32_t la, ha, lb, hb;
        if constexpr (FLAG) {
            const uint32_t ta = (w & 0xFFFFu) + 0xFFFFu, tb = (w >> 16) + 0xFFFFu;
            la = lds(__byte_perm(ta, bL, 0x7604));
            ha = lds(__byte_perm(ta, bH, 0x7214));
            lb = lds(__byte_perm(tb, bL, 0x7604));
            hb = lds(__byte_perm(tb, bH, 0x7214));
        } else {
            uint32_t t;
            asm("add.u16x2 %0, %1, %2;" : "=r"(t) : "r"(w), "r"(0xFFFFFFFFu));  // e = c - 1 per half
            la = lds(__byte_perm(t, bL, 0x7604));
            ha = lds(__byte_perm(t, bH, 0x7614));
            lb = lds(__byte_perm(t, bL, 0x7624));
            hb = lds(__byte_perm(t, bH, 0x7634));
        }
        acc += (uint64_t)(la * ha) * xa;
        acc += (uint64_t)(lb * hb) * xb;
    };
    auto vec8 = [&](const uint4 a, const uint4 xw, uint64_t &acc) {
        pair(a.x, xw.x & 0xFFFFu, xw.x >> 16, acc);
        pair(a.y, xw.y & 0xFFFFu, xw.y >> 16, acc);
        pair(a.z, xw.z & 0xFFFFu, xw.z >> 16, acc);
        pair(a.w, xw.w & 0xFFFFu, xw.w >> 16, acc);
    };
    const uint4 *xv = reinterpret_cast<const uint4 *>(s_x);
    // row indices in 32 bits (the launcher checks rows < 2^30: row + 2 x gstride cannot wrap)
    const int nrows = (int)rows;
    const int warp0 = (int)blockIdx.x * (NT / 32) + (int)(threadIdx.x >> 5);
    const int gstride = (int)gridDim.x * (NT / 32) * RP;  // rows between a warp's row groups
    // A warp walks a stream of elements (row group of RP rows, vector k < vpl of each row); a ring of U elements
    // per lane: the slot just consumed is refilled at once with the element U ahead (the same row group or, in a
    // group's last turn, the next one), so loads stay in flight while the lane computes across row groups.  (ptxas
    // waits for the ring's loads as one scoreboard, so the effective prefetch distance is about one element; 64
    // registers per thread at 1024 threads leave no room for a deeper ring: profiles/r02_zsplit_ab.txt.)
    // Loads are never predicated off: a row past the matrix re-reads the last row (its sum is never written),
    // a vector slot past the row re-reads a valid vector (its staged x is 0).
    const uint4 *A4 = reinterpret_cast<const uint4 *>(A);
    const int64_t lda8 = lda / 8;  // row stride in 16-byte vectors (the launcher checks lda * 2 % 16 == 0)
    const int vmax = (int)max(nvec, (int64_t)1) - 1;
    int lrow = warp0 * RP;  // row group being loaded
    const uint4 *lp;        // its first row (clamped into the matrix)
    int loff[RP];           // offsets of its rows in vectors (a row past the matrix: the last row's)
    auto set_group = [&]() {
        const int r0 = lrow < nrows ? lrow : nrows - 1;
        lp = A4 + (int64_t)r0 * lda8;
#pragma unroll
        for (int r = 1; r < RP; ++r) loff[r] = (r0 + r < nrows ? r : nrows - 1 - r0) * (int)lda8;
    };
    // element k of a lane: vector lane + 32 k of each row of the group
    auto load = [&](uint4 (&e)[RP], int k) {
        const int v = min(lane + 32 * k, vmax);
#pragma unroll
        for (int r = 0; r < RP; ++r) e[r] = ld_stream(lp + (r == 0 ? v : loff[r] + v));
    };
    set_group();
    uint4 ring[U][RP];
#pragma unroll
    for (int u = 0; u < U; ++u) load(ring[u], u);
    uint64_t acc[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[r] = 0;
    // U divides vpl (launcher): each row group is vpl / U unrolled ring turns, then its completion
    for (int urow = warp0 * RP; urow < nrows; urow += gstride) {
#pragma unroll 2  // two turns per iteration: the ring is renamed instead of copied (B200: 108.3 -> 101.8 us)
        for (int uk = 0; uk < vpl; uk += U) {
            int lk = uk + U;  // elements loaded in this turn: k = lk + u of the load group
            if (lk == vpl) {
                lk = 0;
                lrow += gstride;
                set_group();
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                uint4 cur[RP];
#pragma unroll
                for (int r = 0; r < RP; ++r) cur[r] = ring[u][r];
                load(ring[u], lk + u);
                const uint4 xw = xv[lane + 32 * (uk + u)];
#pragma unroll
                for (int r = 0; r < RP; ++r) vec8(cur[r], xw, acc[r]);
            }
        }
        for (int64_t j = nvec * 8 + lane; j < n; j += 32) {  // scalar tail: code and x in the low halves
#pragma unroll
            for (int r = 0; r < RP; ++r)
                if (urow + r < nrows) pair((uint32_t)A[(int64_t)(urow + r) * lda + j], s_x[xtail + j - nvec * 8], 0u, acc[r]);
        }
#pragma unroll
        for (int r = 0; r < RP; ++r) {
            const uint64_t t = warp_sum(acc[r]);  // row total < n (p-1)^3 < 2^64 (host-checked)
            if (lane == 0 && urow + r < nrows) write_result(mod_p(t, K.p, K.mu), O, K, urow + r);
            acc[r] = 0;
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
        // split-exponent kernel (batch_zsplit_kernel): two conflict-free lookups per term; the row total
        // n (p-1)^3 must fit the u64 and x must fit below the table (absolute shared 0xFF80, less the reserved base)
        const int64_t zvpl = std::max<int64_t>((n / 8 + 31) / 32, 1);
        // (row indices and the in-group row offsets r * lda / 8, r < GFP_ZS_RP, are 32-bit in the kernel)
        const bool idx32 = rows < (int64_t(1) << 30) && lda / 8 * GFP_ZS_RP < (int64_t(1) << 31);
        if (GFP_ZSPLIT && vec && lanes == 0 && n >= 8 && idx32 && (u128)n * q2 * pm1 <= max64 &&
            2 * (256 * zvpl + 8) <= kZsXBytes) {
            constexpr int ZNT = GFP_ZS_NT, ZU = GFP_ZS_U, ZRP = GFP_ZS_RP;
            const bool flag = I.p > 65281;  // the zero code needs the flag page (no free H row)
            // ring depth: the largest of {ZU, 2, 1} dividing the vectors per lane and row
            const int64_t vpl = zvpl;
            auto kern = flag ? batch_zsplit_kernel<ZNT, 1, ZRP, true> : batch_zsplit_kernel<ZNT, 1, ZRP, false>;
            if (vpl % ZU == 0)
                kern = flag ? batch_zsplit_kernel<ZNT, ZU, ZRP, true> : batch_zsplit_kernel<ZNT, ZU, ZRP, false>;
            else if (vpl % 2 == 0)
                kern = flag ? batch_zsplit_kernel<ZNT, 2, ZRP, true> : batch_zsplit_kernel<ZNT, 2, ZRP, false>;
            const size_t smem = 2 * (size_t)kZsTab;  // the table ends at absolute 0x20000
            const int bps = occupancy(kern, ZNT, smem);
            const int64_t rpb = ZNT / 32 * GFP_ZS_RP;
            const int64_t grid = std::min<int64_t>((rows + rpb - 1) / rpb, (int64_t)num_sms(dev) * bps);
            cudaError_t le = launch_pdl(kern, dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(ZNT), smem, s,
                                        (const uint16_t *)A, lda, (const uint16_t *)x, rows, n, K, O);
            count_launch();
            *err = le != cudaSuccess ? le : cudaGetLastError();
            break;
        }
        const uint32_t zentries = (uint32_t)((I.p + 7) & ~7ull);  // codes [0, qbar] = p entries
        const size_t zsmem = (size_t)zentries * 2 + (size_t)(((n + 1) / 2 + 3) & ~int64_t(3)) * 4;
        if (GFP_ZBATCH_DECODE && vec && lanes == 0 && (u128)n * q2 <= max64 && zsmem <= kBatchSmemX) {
            const uint32_t entries = zentries;
            const size_t smem = zsmem;
            // one 1024-thread CTA per SM (64 registers: U = 4 vectors per row and lane for RP = 2 rows in flight);
            // B200 A/B (scripts/ab_zbatch.py, GF(32749) / GF(65521)): three 512-thread CTAs at 40 registers
            // (U = 2) 152.7 / - us, RP = 1 137.8 / 138.1, RP = 4 (U = 1) 148.7 / 149.1, this 130.7 (65521);
            // a register ping-pong pipeline over (row, chunk) spilled and ran 173-190 us
            constexpr int ZNT = GFP_ZDEC_NT;
            auto kern = batch_zech_kernel<ZNT, GFP_ZDEC_U, 1, GFP_ZDEC_RP>;
            const int bps = occupancy(kern, ZNT, smem);
            const int64_t rpb = ZNT / 32 * GFP_ZDEC_RP;  // rows per CTA per sweep (a warp per RP rows)
            const int64_t grid = std::min<int64_t>((rows + rpb - 1) / rpb, (int64_t)num_sms(dev) * bps);
            cudaError_t le = launch_pdl(kern, dim3((unsigned)std::max<int64_t>(grid, 1)), dim3(ZNT), smem, s,
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

}  // namespace gfp
