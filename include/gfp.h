/*
 * gfp.h -- C ABI of libgfp: the exact dot product of two vectors over a
 * word-size prime field GF(p) on NVIDIA B200 (sm_100a).
 *
 * Paper: J.-G. Dumas, "Efficient dot product over word-size finite fields",
 * arXiv cs/0404008.  Citations "P:n" are lines of its text with the
 * section; "G<k>" are the readings of ambiguous passages listed in DESIGN.md.
 *
 * What is computed (sec. 3).  For two length-n vectors whose
 * entries are canonical elements of GF(p) in one of the paper's
 * representations, the dot product r = sum_i a_i b_i in GF(p), returned in
 * the SAME representation ("the dot products are of course
 * performed with their representations", reading G10).  The method is the
 * paper's delayed modulus (sec. 3.1 Eq. (1); sec. 3.2 blocks,
 * P:352-377; sec. 3.3 overflow correction): products are summed in
 * a wide register and reduced mod p only when the bound on the register
 * would otherwise be crossed.  The result is exact; it is bit-identical to
 * the plain definition (sum a_i b_i) mod p.
 *
 * Representations (sec. 2) and admissible (rep, dtype, p):
 *   GFP_REP_CLASSICAL  residues in [0, p-1]           (sec. 2.1)
 *       GFP_U16: p <= 65521          GFP_U32: p <= 4294967291
 *   GFP_REP_MONTGOMERY a stored as a*B mod p, B=2^32  (sec. 2.2)
 *       GFP_U32: odd p <= 2654435761
 *   GFP_REP_FP64       exact integers in [0, p-1] held in binary64,
 *                      reduced by T -= floor(T*invP)*P and one +-P fix-up
 *                      (sec. 2.3, NTL listing P:112-117)
 *       GFP_F64: p <= 94906249 (largest prime with p(p-1) < 2^53; Eq. (1)
 *                at m = 53, P:338-339 reading G9)
 *   GFP_REP_ZECH       discrete-log codes: 0 -> 0, 1 -> q-1, g^i -> i
 *                      (sec. 2.4), g = smallest primitive root
 *       GFP_U16: p <= 65521 (the antilog table must fit shared memory; the
 *                paper's index bound 1073741789, is looser)
 *   GFP_REP_CENTERED   residues stored between -(p-1)/2 and (p-1)/2, signed (sec. 3.2.2);
 *                      blocks of lambda_c products with lambda_c ((p-1)/2)^2 + (p-1)/2 < 2^(m-1)
 *                      (int64 accumulators) or < 2^53 (binary64)
 *       GFP_U16 storage holds int16: odd p <= 65521     GFP_U32 storage holds int32: odd p <= 4294967291
 *       GFP_F64: exact integers, odd p <= 189812507 (largest prime with h(h+1) < 2^53, h = (p-1)/2)
 *   p must be prime (GFP_E_NOT_PRIME) and within the bound (GFP_E_BOUND);
 *   any other (rep, dtype) pair is GFP_E_UNSUPPORTED.
 *
 * Pointers.  Unless a function says "host", every array pointer is a CUDA
 * device pointer on the current device, owned by the caller.  Element
 * pointers must be aligned to their element size (GFP_E_INVAL otherwise);
 * Any alignment is accepted: elements before a's first 16-byte boundary
 * are a scalar head; b at a different 16-byte phase than a is read as
 * aligned vectors and realigned in registers by the built-in plans, the
 * sec. 3.4 hybrid and the sec. 3.3 carry word (other explicit strategies
 * and GFP_STRAT_ZECH_ADD then take a slower scalar path).
 *
 * Streams.  `stream` is a cudaStream_t passed as void* (NULL = the legacy
 * default stream).  Device-pointer calls are asynchronous: they enqueue work
 * on `stream` and return; results are ready in stream order.  They never
 * allocate on the hot path after the first call for a (device, p, rep,
 * stream) and are safe to capture in a CUDA graph after that first call.
 * Each (device, stream) owns a small self-resetting combine workspace, so
 * calls are ordered by their stream; a captured graph keeps using the
 * capturing stream's workspace -- do not replay it concurrently with other
 * library calls on that stream's workspace (e.g. two replays on two streams).
 * Kernels are launched with programmatic stream serialization (PDL): the next
 * launch is staged while the previous kernel drains.  Before waiting on the
 * stream's earlier work a kernel touches only library-owned tables and issues
 * L2 prefetches (which cannot observe stale data); every load of caller memory
 * comes after the wait, so results are exactly those of plain stream order.
 *
 * Preconditions.  Entries must be canonical elements of the representation
 * (P:49-50).  This is not checked on the hot path: non-canonical entries give
 * an unspecified result but never an out-of-bounds access (Zech indices are
 * clamped into the table).
 *
 * Errors.  Argument errors are returned synchronously with nothing enqueued
 * and nothing written.  Launch failures return GFP_E_CUDA with text from
 * gfp_last_error().  Asynchronous device faults surface at the caller's next
 * synchronisation.  All functions are thread-safe.
 */
#ifndef GFP_H
#define GFP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GFP_OK = 0,
    GFP_E_INVAL = 1,       /* bad argument: n < 0, NULL with n > 0, misaligned, unknown enum */
    GFP_E_NOT_PRIME = 2,   /* p is not prime */
    GFP_E_BOUND = 3,       /* p outside the representation's bound (table above) */
    GFP_E_UNSUPPORTED = 4, /* (rep, dtype) combination not offered */
    GFP_E_CUDA = 5,        /* CUDA runtime error (see gfp_last_error) */
    GFP_E_NOMEM = 6        /* device or pinned allocation failed */
} gfp_status;

typedef enum {
    GFP_REP_CLASSICAL = 0,
    GFP_REP_MONTGOMERY = 1,
    GFP_REP_FP64 = 2,
    GFP_REP_ZECH = 3,
    GFP_REP_CENTERED = 4
} gfp_rep;

typedef enum { GFP_U16 = 0, GFP_U32 = 1, GFP_F64 = 2 } gfp_dtype;

/* Accumulation strategy the kernels use for a (p, rep, dtype), chosen on the
 * host from the bounds of sec. 3. */
typedef enum {
    GFP_ACC_DELAYED = 0,   /* Eq. (1): n products never overflow -> one final reduction */
    GFP_ACC_BLOCKED = 1,   /* sec. 3.2: reduce every k products (Montgomery sec. 3.2.1) */
    GFP_ACC_OVERFLOW = 2   /* sec. 3.3: let the u64 wrap, add CORR = 2^64 mod p on wrap */
} gfp_acc;

/* The paper's accumulation algorithms (sec. 3), selectable per call through gfp_options. */
typedef enum {
    GFP_STRAT_AUTO = 0,     /* the library's choice (the fastest exact plan; gfp_plan reports it) */
    GFP_STRAT_DELAYED = 1,  /* sec. 3.1 Eq. (1): no reduction before the end; needs n(p-1)^2 < 2^m */
    GFP_STRAT_BLOCKED = 2,  /* sec. 3.2: reduce every k = floor((2^m-1-(p-1))/(p-1)^2) products (G7) */
    GFP_STRAT_OVERFLOW = 3, /* sec. 3.3: wrap test + CORR = 2^m mod p on every product */
    GFP_STRAT_HYBRID = 4,   /* sec. 3.4 Eq. (2): one wrap test per block of lambda, lambda p(p-1) < 2^m */
    GFP_STRAT_ZECH_ADD = 5, /* Zech only: pure discrete-log accumulation -- every product is an index
                               addition and every sum a Zech addition through the t_plus1 table
                               (sec. 2.4, Table 1); partial sums never leave the
                               representation.  Same unique result as the default (integer) plan. */
    GFP_STRAT_CARRY = 6     /* classical and Montgomery: the division-on-demand idea of sec. 3.3
                               with the correction deferred -- the carry flag of each m-bit add (add-with-
                               carry instructions, no compare) is counted in a second word and carry *
                               (2^m mod p) applied once at the end instead of adding CORR at every wrap
                               (SURVEY 8(f) F2 "carry-word"); the built-in plan for classical u32 storage
                               when lambda of Eq. (2) is below 4 (p > ~2^31.5) */
} gfp_strategy;

/* Per-call options.  acc_bits: the accumulator width m of Eq. (1): 0 = default (64; 53 for fp64),
 * 32 or 64 for classical storage (m = 32 needs p(p-1) < 2^32, i.e. p <= 65521).  Admissible
 * combinations: classical x {AUTO..HYBRID, CARRY} x {32, 64}; Montgomery x {AUTO, BLOCKED (REDC every
 * k_R products, sec. 3.2.1), OVERFLOW (overflow-Montgomery, sec. 3.3), CARRY}; fp64 x {AUTO,
 * DELAYED, BLOCKED}; Zech x {AUTO, ZECH_ADD}; centered x {AUTO, DELAYED, BLOCKED} (the signed overflow trick,
 * P:441-457, and hybrid centered, are not offered: the paper finds the first too costly and
 * shows the second cannot work).  Anything else: GFP_E_UNSUPPORTED; a strategy whose bound the
 * (p, n) pair violates: GFP_E_BOUND.
 * lanes_per_row (gfp_dot_batch_ex only; 0 for dots): how many threads share one row's accumulation --
 * 0 = the library's choice (32 for rows of >= 256 16-byte vectors or table representations, else 8), or
 * 1, 8, 32.  1 is the paper's own loop: ONE accumulator walks the whole row, so a row of
 * DIM terms reaches the block bound k of Eq. (1) exactly where the paper's scalar loop does (the DIM = 512,
 * m = 32 step after p = 2897); with L lanes each accumulator sees about DIM / L terms and the
 * step moves to the prime where (DIM / L)(p-1)^2 crosses 2^m.  1 is offered for integer storage only
 * (classical, Montgomery, centered int16 / int32); anything else is GFP_E_INVAL / GFP_E_UNSUPPORTED. */
typedef struct {
    int32_t strategy;  /* gfp_strategy */
    int32_t acc_bits;
    int32_t lanes_per_row;
} gfp_options;

/* What a call would run (gfp_plan): kernel, grid, the strategy and its block length, and per-thread
 * bounds on terms and on reductions / wrap tests. */
typedef struct {
    int32_t strategy, acc_bits;
    uint64_t block;              /* products per reduction or per wrap test; 0 = none before the end */
    int32_t grid, threads_per_block;
    int64_t terms_per_thread;    /* upper bound */
    int64_t reductions_per_thread; /* upper bound: remainders, REDCs or wrap tests */
    char kernel[64];
} gfp_plan_info;

/* Host-side description of a field/representation (gfp_query). */
typedef struct {
    uint64_t p;
    int32_t rep, dtype;
    uint64_t bound;        /* largest admissible p for (rep, dtype) */
    int32_t acc_bits;      /* m of Eq. (1): 64 (integer accumulators) or 53 (binary64) */
    int32_t mont_kr;       /* Montgomery: products per REDC allowed by the two G6 bounds, capped at 10^6; else 0 */
    uint64_t k;            /* Eq. (1) with a carried residue (reading G7):
                              largest k with k(p-1)^2 + (p-1) <= 2^m - 1 (binary64: < 2^53);
                              centered: largest k with k h^2 + h <= 2^63 - 1 (binary64: < 2^53),
                              h = (p-1)/2 */
    uint64_t corr;         /* CORR = 2^64 mod p (sec. 3.3) */
    uint32_t n_im;         /* Montgomery: -p^{-1} mod 2^32; else 0 */
    uint32_t pad0;
    uint64_t r2;           /* Montgomery: B^2 mod p, to_mont(a) = REDC(a * R2) */
    uint64_t b_mod_p;      /* 2^32 mod p */
    double inv_p;          /* binary64 RN(1/p) (reading G8) */
    uint64_t g;            /* Zech: generator (smallest primitive root, reading G12); else 0 */
    uint64_t qbar;         /* Zech: q-1; else 0 */
    uint64_t table_bytes;  /* Zech: bytes of the shared-memory antilog table; else 0 */
} gfp_info;

/* host: validate (p, rep, dtype) and fill *info.  No device work. */
gfp_status gfp_query(uint64_t p, gfp_rep rep, gfp_dtype dt, gfp_info *info);

/* r = a . b in GF(p), written to out[0] (device, one element of dtype `dt`).
 * a, b: device arrays of n elements of dtype `dt` in representation `rep`.
 * n == 0 writes the representation's zero (0, 0, +0.0, code 0).
 * One kernel launch: streaming delayed-modulus accumulation, warp-shuffle and
 * CTA-tree combination, last-CTA-done final reduction and encoding. */
gfp_status gfp_dot(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                   void *out, void *stream);

/* Batched: out[r] = A[r*lda .. r*lda+n) . x for r in [0, rows) -- many
 * independent dots / a GF(p) matrix-vector product (sec. 1).
 * A: device, row-major with leading dimension lda >= n (elements);
 * x: device, n elements; out: device, `rows` elements of dtype `dt`.
 * Supported reps: classical (u16, u32), Montgomery (u32), fp64, Zech (u16), centered.
 * Zech rows (16-byte aligned A, x and lda): each code c of A is decoded as g^c = H[(c-1) >> 8] * L[(c-1) & 255]
 * from two 256-entry tables replicated per shared-memory bank (readings G25/G26 in DESIGN.md; n (p-1)^3 < 2^64,
 * else one antilog lookup per code) and multiplied by the decoded x (x decoded once per CTA); the row value is
 * encoded back into a code; unaligned rows take the index-add kernel.  One kernel launch. */
gfp_status gfp_dot_batch(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *A, int64_t lda,
                         const void *x, int64_t rows, int64_t n, void *out, void *stream);

/* Representation conversion (sec. 2.2 a -> aB mod p; sec. 2.4 the
 * discrete-log encoding P:126-131; fp64: exact casts).  Timed separately from
 * the dot.
 *   gfp_to_rep  : `in` holds canonical classical residues (in_dt U16/U32);
 *                 `out` receives the representation in out_dt (the rep's dtype).
 *   gfp_from_rep: the inverse; in_dt is the rep's dtype, out_dt U16/U32.
 * In-place (in == out) is allowed when in_dt == out_dt. */
gfp_status gfp_to_rep(uint64_t p, gfp_rep rep, gfp_dtype in_dt, const void *in, gfp_dtype out_dt,
                      void *out, int64_t n, void *stream);
gfp_status gfp_from_rep(uint64_t p, gfp_rep rep, gfp_dtype in_dt, const void *in, gfp_dtype out_dt,
                        void *out, int64_t n, void *stream);

/* Multi-GPU bracket.  gfp_dot_partial writes to
 * partial[0] (device uint64) this shard's contribution: a residue in [0, p)
 * in the representation's additive form (classical value; Montgomery form;
 * the integer value for fp64; the classical value for Zech).  The caller sums
 * partials across ranks (e.g. an NCCL all_reduce SUM over int64; at most 2^31
 * ranks) and calls gfp_finalize(summed) -> out[0] in the representation. */
gfp_status gfp_dot_partial(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b,
                           int64_t n, uint64_t *partial, void *stream);
gfp_status gfp_finalize(uint64_t p, gfp_rep rep, gfp_dtype dt, const uint64_t *summed, void *out,
                        void *stream);

/* ---- Fused multi-GPU dot (SURVEY 8(e) "fused variant"): ONE kernel per rank
 * computes the rank's shard, and its last CTA exchanges the shard's partial with every peer over peer
 * memory (NVLink / NVSwitch stores) and finalizes -- no NCCL launch on the data path.
 *
 * Setup, once per process group: each rank creates an exchange buffer (gfp_xchg_create: device memory of
 * gfp_xchg_bytes() bytes, zeroed, owned by the library, plus its 64-byte CUDA IPC handle); the caller
 * passes the handles to every rank over any host channel (e.g. torch.distributed.all_gather_object);
 * each rank maps its peers' buffers with gfp_xchg_open (its own buffer is used directly) and fills a
 * gfp_xchg {rank, world, peers[r] = rank r's buffer as mapped in this process}.
 *
 * Protocol (all ranks call gfp_dot_allreduce in the same order -- the usual collective contract; the
 * state lives in device memory, so calls may be captured in CUDA graphs): the calling rank's epoch e is
 * its buffer's counter + 1; the last CTA stores ONE tagged 64-bit word ((e mod 2^32) << 32 | its partial
 * residue, additive form as gfp_dot_partial, < 2^32) into slot [e mod 2][rank] of every peer's buffer --
 * data and flag in one single-copy-atomic store, so no system-scope fence is needed -- then polls its own
 * slots [e mod 2][r] until every one carries the tag of epoch e, sums their residues, reduces mod p,
 * encodes out[0] and stores e.  Two slot sets suffice: a rank can only write epoch e + 2's slot after
 * every rank published epoch e + 1, i.e. after every rank has read epoch e's.  A peer that never arrives makes the kernel trap after about 30 s (the error surfaces
 * at the next synchronisation) instead of hanging.  Every rank receives the same out[0]. */
#define GFP_XCHG_MAX_WORLD 16
typedef struct {
    int32_t rank, world;              /* 1 <= world <= GFP_XCHG_MAX_WORLD, 0 <= rank < world */
    void *peers[GFP_XCHG_MAX_WORLD];  /* peers[r]: rank r's exchange buffer (device pointer valid here) */
} gfp_xchg;

uint64_t gfp_xchg_bytes(void);
/* host: allocate + zero this rank's exchange buffer on the current device; *buf = device pointer,
 * ipc_handle (64 bytes, caller-provided) receives its CUDA IPC handle. */
gfp_status gfp_xchg_create(void **buf, void *ipc_handle);
/* host: map a peer's buffer from its 64-byte handle (GFP_E_CUDA if the devices cannot peer). */
gfp_status gfp_xchg_open(const void *ipc_handle, void **peer_buf);
gfp_status gfp_xchg_close(void *peer_buf);  /* unmap a gfp_xchg_open mapping */
gfp_status gfp_xchg_destroy(void *buf);     /* free a gfp_xchg_create buffer (after every peer closed it) */
/* host, synchronous (connectivity checks before relying on the group): arm a SOFT timeout of `ns` nanoseconds
 * on this rank's own buffer -- a peer missing that long makes gfp_dot_allreduce record the timeout and encode 0
 * instead of trapping (0 restores the default trap after ~30 s); gfp_xchg_timed_out reads the record (1 if a
 * soft timeout expired since the last gfp_xchg_soft_timeout).  Never arm it for production calls: a timed-out
 * call's result is not the dot. */
gfp_status gfp_xchg_soft_timeout(void *own_buf, uint64_t ns);
gfp_status gfp_xchg_timed_out(void *own_buf, int32_t *timed_out);
/* The whole-group dot: a, b are this rank's shards (n may differ across ranks, may be 0); out[0] (device,
 * one element of dt) receives sum over all ranks' shards of a_i b_i in GF(p), in the representation.  One
 * launch; the default (AUTO) accumulation plan. */
gfp_status gfp_dot_allreduce(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                             const gfp_xchg *x, void *out, void *stream);

/* ---- The fused multi-GPU dot through an NVLink SHARP (NVLS) multicast buffer (SURVEY 8(e) "fused variant":
 * multimem.red into a multicast buffer, then a counter barrier, then finalize -- one launch per rank, no NCCL;
 * the reduction happens in the NVSwitch).  Same result and calling contract as gfp_dot_allreduce.
 *
 * Setup, once per process group (every call on the rank's current device):
 *   rank 0:      gfp_mc_create(world, &mc, &fd, &bytes) -- a multicast object for `world` devices and a POSIX
 *                file descriptor for it (owned by mc); the caller passes fd (e.g. SCM_RIGHTS over a Unix
 *                socket) and bytes to every other rank;
 *   other ranks: gfp_mc_import(fd_received, bytes, world, &mc);
 *   every rank:  gfp_mc_add_device(mc); then, after EVERY rank has added its device (a group barrier),
 *                gfp_mc_bind(mc) -- backs the object with this device's memory, maps it twice (multicast and
 *                unicast) and zeroes this rank's copy; then a group barrier before the first dot.
 *   teardown:    gfp_mc_destroy(mc) on every rank after the last dot (unbinds, unmaps, releases, closes fd).
 * GFP_E_UNSUPPORTED where the device or driver has no multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED).
 *
 * Protocol (the kernel's last CTA, one thread): epoch e = this rank's counter + 1, parity e mod 2; add the
 * partial residue (additive form, < 2^32) to the parity's running sum on every rank's copy (multimem.red.add),
 * then, with release semantics, one arrival to the parity's counter; poll this rank's copy of the counter
 * (acquire) until it reaches world x (uses of the parity so far); the group sum is the running total minus its
 * value at the parity's previous use (u64 wrap-around arithmetic, exact); reduce mod p and encode.  A missing
 * peer traps after ~30 s instead of hanging. */
typedef struct gfp_mc gfp_mc;  /* opaque: a multicast object, this rank's backing memory and its two mappings */
gfp_status gfp_mc_create(int32_t world, gfp_mc **mc, int32_t *fd, uint64_t *bytes);  /* fd, bytes may be NULL */
gfp_status gfp_mc_import(int32_t fd, uint64_t bytes, int32_t world, gfp_mc **mc);
gfp_status gfp_mc_add_device(gfp_mc *mc);
gfp_status gfp_mc_bind(gfp_mc *mc);
gfp_status gfp_mc_destroy(gfp_mc *mc);
gfp_status gfp_dot_allreduce_mc(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                                gfp_mc *mc, void *out, void *stream);

/* gfp_dot / gfp_dot_batch with explicit options (NULL = defaults): the paper's strategies side by
 * side, exact in every admissible combination.  Same pointers, streams and errors as gfp_dot. */
gfp_status gfp_dot_ex(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                      const gfp_options *opt, void *out, void *stream);
gfp_status gfp_dot_batch_ex(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *A, int64_t lda, const void *x,
                            int64_t rows, int64_t n, const gfp_options *opt, void *out, void *stream);

/* host: the plan gfp_dot_ex would use for n terms with 16-byte aligned operands on the current
 * device (no device work besides querying its SM count and kernel occupancy). */
gfp_status gfp_plan(uint64_t p, gfp_rep rep, gfp_dtype dt, int64_t n, const gfp_options *opt,
                    gfp_plan_info *info);

/* End-to-end convenience: a, b, out are HOST pointers (pinned memory gives
 * overlapped copies; pageable works but copies synchronously).  Streams the
 * operands to the device in chunks through library-owned staging buffers,
 * overlapping each chunk's host->device copy with the previous chunk's
 * kernel, then copies the result back.  Synchronous: returns when out[0] is
 * written. */
gfp_status gfp_dot_host(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                        void *out, void *stream);
/* The same from HOST buffers, but *partial (HOST, 8-byte aligned uint64) receives this shard's partial
 * residue in the representation's additive form, exactly as gfp_dot_partial writes it (classical value,
 * Montgomery form, fp64 integer, the classical value of a Zech sum -- never a code): the multi-GPU
 * end-to-end path sums these across ranks and calls gfp_finalize, as for device shards. */
gfp_status gfp_dot_host_partial(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                                uint64_t *partial, void *stream);

/* ---- Install-time tuning (the paper's conclusion: an optimal dot "should
 * switch from block methods to a floating point representation according to the vector and prime size
 * and to the architecture ... the idea is to use an Automated Empirical Optimization of Software in
 * order to produce a library which would determine and choose the best switching thresholds at
 * install time").
 *
 * gfp_tune runs, on the current device and `stream`, every admissible accumulation of sec. 3 for each
 * case (classical: the built-in plan and DELAYED / BLOCKED / OVERFLOW / HYBRID with m = 32 and 64;
 * Montgomery: built-in and overflow-Montgomery; fp64: built-in, DELAYED, BLOCKED; Zech: built-in and
 * ZECH_ADD) on synthetic canonical inputs generated on the device, checks that every candidate returns
 * the same field element(s) (GFP_E_CUDA with a message otherwise: an exactness failure), and records
 * the fastest in the library's tuning table (one entry per case; a re-tuned case replaces its entry).
 * Each candidate is timed with CUDA events over about ms_per_candidate milliseconds of replays of a CUDA
 * graph that holds 8-64 calls (after 2 warm-up calls; device time per call, as the bench measures, not the
 * host's launch rate), rotating through enough input sets that >= 3x the L2 is streamed between two uses
 * of a set (at most 64 sets / 1 GiB).  The calls run on a private stream after `stream` has drained.
 * Device memory is allocated and freed inside the call.
 *
 * GFP_STRAT_AUTO (gfp_dot, gfp_dot_batch, gfp_dot_partial, gfp_dot_ex / _batch_ex / gfp_plan with a NULL
 * or all-zero gfp_options) then follows the table: among the entries with the call's (rep, dtype, kind)
 * it takes the one nearest in (log2 p, log2 n), and log2 rows for batches (L1 distance; first entry on
 * ties) and uses its strategy
 * if that strategy is admissible for the call's (p, n); otherwise -- or with an empty table -- the
 * built-in analytic plan.  On the first AUTO call of a process the library loads a table (gfp_tune_save
 * format) from the file the environment variable GFP_TUNE_FILE names ("" = none), or, when it is unset,
 * from gfp_tune.txt in the directory of libgfp.so (written at install time by
 * `python -m paper_cs_0404008_b200.autotune --out <that directory>/gfp_tune.txt`); a missing or invalid
 * file leaves the table empty.  gfp_tune / _set / _load / _clear take precedence over that load. */
typedef struct {
    int32_t rep, dtype;
    int32_t kind;  /* 0: single dot of n terms; 1: batch of rows x n (gfp_dot_batch) */
    int32_t pad0;
    uint64_t p;
    int64_t n, rows;
} gfp_tune_case;

typedef struct {
    int32_t rep, dtype, kind;
    int32_t strategy, acc_bits; /* the winner; strategy GFP_STRAT_AUTO = the built-in plan won */
    int32_t pad0;
    uint64_t p;
    int64_t n, rows;
    double us_best, us_builtin; /* measured microseconds per call: the winner, the built-in plan */
} gfp_tune_entry;

gfp_status gfp_tune(const gfp_tune_case *cases, int32_t ncases, double ms_per_candidate, void *stream);
/* host: copy up to cap entries of the table to out (out may be NULL with cap 0); returns the count. */
int32_t gfp_tune_entries(gfp_tune_entry *out, int32_t cap);
/* host: replace the table by `count` entries (validated: known rep/dtype/kind/strategy, p > 1, n >= 0). */
gfp_status gfp_tune_set(const gfp_tune_entry *entries, int32_t count);
/* host: text file, a "# gfp-tune v1" line then one entry per line:
 * rep dtype kind p n rows strategy acc_bits us_best us_builtin */
gfp_status gfp_tune_save(const char *path);
gfp_status gfp_tune_load(const char *path);
void gfp_tune_clear(void);

/* Number of kernels the library launched on this host thread since the
 * last reset (evidence for the bench's gpu_launches claim). */
uint64_t gfp_launch_count(int reset);

const char *gfp_status_str(gfp_status s);
const char *gfp_last_error(void);    /* thread-local text of the last error */
void gfp_release_caches(void);      /* free device tables, workspaces and staging buffers */
const char *gfp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GFP_H */
