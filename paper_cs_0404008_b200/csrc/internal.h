// internal.h -- interface between the C ABI (api.cpp) and the kernel launchers (kernels_*.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "params.h"
#include "gfp.h"

namespace gfp {

// Per-(device, stream) scratch for the single-launch combine, self-resetting (no memset per call):
// dot_kernel packs the CTA residues and their arrival count into partials[0]; the pure-Zech kernel keeps
// one Zech value per CTA in partials[1 ..] and counts arrivals in `counter`.
struct Workspace {
    uint64_t *partials;
    unsigned int *counter;
};

// Where the final residue goes.  OUT_XCHG: exchange with the group's peers first (fused multi-GPU
// combine over peer stores, gfp_dot_allreduce), then encode like OUT_ENCODE.  OUT_MC: the same through an
// NVLink SHARP (NVLS) multicast buffer (multimem reductions in the switch, gfp_dot_allreduce_mc).
enum OutMode { OUT_ENCODE = 0, OUT_PARTIAL = 1, OUT_ACCUMULATE = 2, OUT_XCHG = 3, OUT_MC = 4 };
struct OutSpec {
    void *out;          // OUT_ENCODE / OUT_XCHG / OUT_MC: element of (rep, dtype); else uint64_t*
    int rep, dtype, mode;
    uint64_t *xchg;     // OUT_XCHG: this rank's exchange buffer (rank, world, peer table); OUT_MC: this rank's
                        // unicast mapping of the multicast buffer
    int prefetch;       // set by the launcher: prefetch the first chunk into L2 before griddepcontrol.wait
    uint64_t *mc;       // OUT_MC: the multicast mapping of the same buffer (multimem.red targets)
};
// Multicast-buffer layout (u64 words; gfp_dot_allreduce_mc).  Private to each rank (unicast, never a multimem
// target): [0] epoch, [1] world, [2 + par] uses of each slot parity, [4 + par] the slot's total at its last
// use.  Reduced by every rank through the multicast mapping, in their own 128-byte lines: the partial sums
// [kMcSum + par] and the arrival counts [kMcCnt + par].
constexpr int kMcSum = 32, kMcCnt = 48, kMcWords = 64;
// Packed combine: the CTA residues (< p < 2^32) are summed in bits [0, kPackShift), the CTA arrival
// count in bits [kPackShift, 64): exact for grids below 2^(64 - kPackShift) CTAs.
constexpr int kPackShift = 48;
// Exchange-buffer layout (u64 words): [0] this rank's epoch, [1] rank, [2] world; [kXFlags, kXSlots) unused
// (a separate-flag protocol, replaced by tagged slots); tagged partial slots (epoch << 32 | residue) at
// kXSlots + parity * MAXW + r; the peer table (every rank's buffer as mapped in this process) at
// kXPeers + r.  Kernel parameters stay small: one pointer.
constexpr int kXFlags = 8, kXSlots = 8 + 2 * GFP_XCHG_MAX_WORLD, kXPeers = 8 + 4 * GFP_XCHG_MAX_WORLD,
              kXWords = 8 + 5 * GFP_XCHG_MAX_WORLD;
// [kXSoft]: a soft timeout in ns (0: trap after ~30 s); [kXTimedOut]: set when a soft timeout expired
constexpr int kXSoft = 3, kXTimedOut = 4;

constexpr int kMaxGrid = 4096;

// Kernel variant selected on the host from the bounds.
struct DotPlan {
    int policy;     // enumerated in kernels_common.cuh
    int grid, block;
    size_t smem;
    int64_t head;   // scalar elements before a's first 16-byte boundary (== n: the whole input scalar)
    int bshift;     // bytes b's element `head` sits past a 16-byte boundary (0: co-aligned)
    int acc;        // gfp_acc reported for the plan
    int strategy;   // gfp_strategy actually used
    int acc_bits;   // m of the accumulator
    uint64_t kblk;  // products per reduction / per wrap test (0: none before the end)
    int64_t per_thread, reductions;  // bounds per thread
    const char *name;
};

// Build a plan: chooses grid, the accumulation policy and its mode for n elements.
gfp_status plan_dot(const gfp_info &info, const dev::KParams &K, const void *a, const void *b, int64_t n,
                    const gfp_options *opt, DotPlan *plan);
cudaError_t launch_dot(const DotPlan &plan, const dev::KParams &K, const void *a, const void *b, int64_t n,
                       Workspace ws, OutSpec out, cudaStream_t s);
cudaError_t launch_finalize(const dev::KParams &K, const uint64_t *summed, int count, OutSpec out,
                            cudaStream_t s);
gfp_status launch_batch(const gfp_info &info, const dev::KParams &K, const void *A, int64_t lda, const void *x,
                        int64_t rows, int64_t n, const gfp_options *opt, OutSpec out, cudaStream_t s,
                        cudaError_t *err);
// dir: 0 = to_rep, 1 = from_rep
gfp_status launch_convert(const gfp_info &info, const dev::KParams &K, int dir, gfp_dtype in_dt, const void *in,
                          gfp_dtype out_dt, void *out, int64_t n, cudaStream_t s, cudaError_t *err);

int num_sms(int device);
// Write rank, world and the peer table into an exchange buffer (one thread, stream-ordered).
cudaError_t launch_xchg_setup(uint64_t *own, int rank, int world, uint64_t *const *peers, cudaStream_t s);
// Set the thread-local text returned by gfp_last_error (api.cpp).
void set_last_error(const char *msg);

// Synthetic canonical elements on the device (tuner inputs): floor(hash(seed, i) p / 2^64).
cudaError_t launch_fill(void *out, int dtype, uint64_t p, uint64_t seed, int64_t n, cudaStream_t s);

// Install-time tuning table (tune.cpp): the tuned explicit options for an AUTO call of `kind` (0 dot,
// 1 batch) with n terms (per row), or false (empty table, the built-in plan won, or tuning bypassed).
bool tuned_options(const gfp_info &info, int kind, int64_t n, int64_t rows, gfp_options *out);
void count_launch();

}  // namespace gfp
