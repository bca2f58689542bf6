// api.cpp -- the C ABI of include/gfp.h: argument validation, per-(device, p, rep) constant and
// table caches, per-(device, stream) workspaces, and the host-buffer pipeline of gfp_dot_host.
#include <cuda.h>  // driver-API types only (multicast / VMM calls go through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "gfp.h"
#include "internal.h"
#include "numtheory.h"

namespace gfp {
uint64_t launches(int reset);
}

using namespace gfp;

namespace {

thread_local std::string t_err;

gfp_status fail(gfp_status s, const std::string &msg) {
    t_err = msg;
    return s;
}

gfp_status cuda_fail(cudaError_t e, const char *where) {
    t_err = std::string(where) + ": " + cudaGetErrorString(e);
    return GFP_E_CUDA;
}

size_t dtype_size(int dt) { return dt == GFP_U16 ? 2 : (dt == GFP_U32 ? 4 : 8); }

struct Ctx {
    gfp_info info;
    dev::KParams K;
    uint16_t *d_antilog = nullptr, *d_log = nullptr, *d_zplus1 = nullptr, *d_zplus1s = nullptr;
};

std::mutex g_mu;
std::map<std::tuple<int, uint64_t, int, int>, Ctx *> g_ctx;
std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;

struct Staging {
    size_t chunk_bytes = 0;
    void *buf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    uint64_t *d_partial = nullptr;
    void *d_out = nullptr;
    cudaStream_t copy = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
};
std::map<int, Staging *> g_stage;
std::mutex g_stage_mu;

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

gfp_status get_ctx(uint64_t p, gfp_rep rep, gfp_dtype dt, Ctx **out) {
    const int dev = current_device();
    auto key = std::make_tuple(dev, p, (int)rep, (int)dt);
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_ctx.find(key);
    if (it != g_ctx.end()) {
        *out = it->second;
        return GFP_OK;
    }
    Ctx *c = new Ctx();
    gfp_status st = describe(p, rep, dt, &c->info);
    if (st != GFP_OK) {
        delete c;
        switch (st) {
        case GFP_E_NOT_PRIME: return fail(st, "p = " + std::to_string(p) + " is not prime");
        case GFP_E_BOUND:
            return fail(st, "p = " + std::to_string(p) + " exceeds the bound " +
                                std::to_string(rep_bound(rep, dt)) + " of this representation/dtype");
        case GFP_E_UNSUPPORTED: return fail(st, "unsupported (representation, dtype) combination");
        default: return fail(st, "invalid representation or dtype");
        }
    }
    dev::KParams &K = c->K;
    memset(&K, 0, sizeof(K));
    K.p = p;
    K.mu = UINT64_MAX / p;
    K.corr = c->info.corr;
    K.pd = (double)p;
    K.inv_p = c->info.inv_p;
    K.r2 = c->info.r2;
    K.n_im = c->info.n_im;
    K.qbar = (uint32_t)c->info.qbar;
    K.corr32 = (uint32_t)((((u128)1) << 32) % p);
    K.mu32 = (uint32_t)(0xFFFFFFFFull / p);
    K.half = (int64_t)((p - 1) / 2);
    K.hd = (double)K.half;
    K.c63 = (uint64_t)((((u128)1) << 63) % p);
    if (rep == GFP_REP_ZECH) {
        std::vector<uint16_t> logt, anti, delta;
        zech_tables(p, c->info.g, logt, anti);
        zech_plus1_delta(p, logt, delta);
        logt.resize((logt.size() + 7) & ~size_t(7), 0);
        anti.resize((anti.size() + 7) & ~size_t(7), 0);
        delta.resize((delta.size() + 7) & ~size_t(7), 0);
        // byte-scaled, doubled copy for the fast S = 2 kernel (small fields): index e in [0, 2 qbar] holds
        // 2 delta[e mod qbar], index 2 qbar + 1 the "add nothing" 0
        const bool scaled = zech_small_layout(p);
        const uint64_t qbar = p - 1;
        // padded to 2^16 entries: any byte offset 2 L - s (L a 16-bit lane, s even) stays inside
        std::vector<uint16_t> delta2(scaled ? 65536 : 0, 0);
        for (uint64_t e = 0; scaled && e <= 2 * qbar; ++e) {
            const uint16_t v = delta[e % qbar];
            delta2[e] = v == kZechDeltaZero ? v : (uint16_t)(2 * v);
        }
        cudaError_t e = cudaMalloc(&c->d_log, logt.size() * 2);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_antilog, anti.size() * 2);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_zplus1, delta.size() * 2);
        if (e == cudaSuccess && scaled) e = cudaMalloc(&c->d_zplus1s, delta2.size() * 2);
        if (e == cudaSuccess && scaled)
            e = cudaMemcpy(c->d_zplus1s, delta2.data(), delta2.size() * 2, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->d_log, logt.data(), logt.size() * 2, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->d_antilog, anti.data(), anti.size() * 2, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->d_zplus1, delta.data(), delta.size() * 2, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(c->d_log);
            cudaFree(c->d_antilog);
            cudaFree(c->d_zplus1);
            cudaFree(c->d_zplus1s);
            delete c;
            return cuda_fail(e, "Zech table upload");
        }
        K.antilog = c->d_antilog;
        K.logt = c->d_log;
        K.antilog_entries = (uint32_t)anti.size();
        K.zplus1 = c->d_zplus1;
        K.zplus1s = c->d_zplus1s;
        K.zplus1s_entries = (uint32_t)delta2.size();
        K.zplus1_entries = (uint32_t)delta.size();
    }
    g_ctx[key] = c;
    *out = c;
    return GFP_OK;
}

gfp_status get_ws(cudaStream_t s, Workspace *ws) {
    const int dev = current_device();
    std::lock_guard<std::mutex> g(g_mu);
    auto key = std::make_pair(dev, s);
    auto it = g_ws.find(key);
    if (it != g_ws.end()) {
        *ws = it->second;
        return GFP_OK;
    }
    void *mem = nullptr;
    const size_t bytes = kMaxGrid * sizeof(uint64_t) + 64;
    cudaError_t e = cudaMalloc(&mem, bytes);
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? fail(GFP_E_NOMEM, "workspace") : cuda_fail(e, "workspace");
    e = cudaMemset(mem, 0, bytes);
    if (e != cudaSuccess) {
        cudaFree(mem);
        return cuda_fail(e, "workspace memset");
    }
    Workspace w;
    w.partials = (uint64_t *)mem;
    w.counter = (unsigned int *)((char *)mem + kMaxGrid * sizeof(uint64_t));
    g_ws[key] = w;
    *ws = w;
    return GFP_OK;
}

bool aligned(const void *p, size_t a) { return ((uintptr_t)p % a) == 0; }

gfp_status check_dot_args(gfp_dtype dt, const void *a, const void *b, int64_t n, const void *out, size_t out_align) {
    if ((int)dt < 0 || (int)dt > 2) return fail(GFP_E_INVAL, "unknown dtype");
    if (n < 0) return fail(GFP_E_INVAL, "n < 0");  // (centered storage reuses the widths: int16 / int32 / f64)
    if (out == nullptr) return fail(GFP_E_INVAL, "out is NULL");
    if (n > 0 && (a == nullptr || b == nullptr)) return fail(GFP_E_INVAL, "NULL operand with n > 0");
    const size_t es = dtype_size(dt);
    if (!aligned(a, es) || !aligned(b, es)) return fail(GFP_E_INVAL, "operand not aligned to its element size");
    if (!aligned(out, out_align)) return fail(GFP_E_INVAL, "output not aligned");
    return GFP_OK;
}

gfp_status plan_fail(gfp_status st) {
    switch (st) {
    case GFP_E_BOUND: return fail(st, "(p, n) violates the bound of the requested strategy / accumulator width");
    case GFP_E_UNSUPPORTED: return fail(st, "strategy or accumulator width not offered for this representation");
    default: return fail(st, "invalid options");
    }
}

gfp_status dot_common(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n, void *out,
                      int mode, cudaStream_t s, const gfp_options *opt = nullptr, uint64_t *xchg = nullptr,
                      uint64_t *mc = nullptr) {
    gfp_status st = check_dot_args(dt, a, b, n, out,
                                   (mode == OUT_ENCODE || mode == OUT_XCHG || mode == OUT_MC) ? dtype_size(dt) : 8);
    if (st != GFP_OK) return st;
    Ctx *c;
    if ((st = get_ctx(p, rep, dt, &c)) != GFP_OK) return st;
    Workspace ws;
    if ((st = get_ws(s, &ws)) != GFP_OK) return st;
    DotPlan plan;
    if ((st = plan_dot(c->info, c->K, a, b, n, opt, &plan)) != GFP_OK) return plan_fail(st);
    OutSpec o{out, (int)rep, (int)dt, mode, xchg, 0, mc};
    cudaError_t e = launch_dot(plan, c->K, a, b, n, ws, o, s);
    return e == cudaSuccess ? GFP_OK : cuda_fail(e, "dot launch");
}

}  // namespace

namespace gfp {
void set_last_error(const char *msg) { t_err = msg; }
}  // namespace gfp

extern "C" {

gfp_status gfp_query(uint64_t p, gfp_rep rep, gfp_dtype dt, gfp_info *info) {
    if (info == nullptr) return fail(GFP_E_INVAL, "info is NULL");
    gfp_status st = describe(p, rep, dt, info);
    if (st == GFP_E_NOT_PRIME) return fail(st, "p is not prime");
    if (st == GFP_E_BOUND) return fail(st, "p exceeds the representation bound");
    if (st == GFP_E_UNSUPPORTED) return fail(st, "unsupported (representation, dtype) combination");
    if (st != GFP_OK) return fail(st, "invalid representation or dtype");
    return GFP_OK;
}

gfp_status gfp_dot(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n, void *out,
                   void *stream) {
    return dot_common(p, rep, dt, a, b, n, out, OUT_ENCODE, (cudaStream_t)stream);
}

gfp_status gfp_dot_partial(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                           uint64_t *partial, void *stream) {
    return dot_common(p, rep, dt, a, b, n, partial, OUT_PARTIAL, (cudaStream_t)stream);
}

uint64_t gfp_xchg_bytes(void) { return (uint64_t)kXWords * sizeof(uint64_t); }

}  // extern "C"
namespace {
std::mutex g_xmu;
std::map<uint64_t *, std::vector<uint64_t>> g_xdesc;  // group description last written into each own buffer
void forget_xchg(void *buf) {
    std::lock_guard<std::mutex> g(g_xmu);
    g_xdesc.erase((uint64_t *)buf);
}
}  // namespace
extern "C" {

gfp_status gfp_xchg_create(void **buf, void *ipc_handle) {
    if (buf == nullptr || ipc_handle == nullptr) return fail(GFP_E_INVAL, "gfp_xchg_create: NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
    void *d = nullptr;
    cudaError_t e = cudaMalloc(&d, gfp_xchg_bytes());
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? fail(GFP_E_NOMEM, "exchange buffer") : cuda_fail(e, "exchange buffer");
    cudaIpcMemHandle_t h;
    if ((e = cudaMemset(d, 0, gfp_xchg_bytes())) != cudaSuccess || (e = cudaIpcGetMemHandle(&h, d)) != cudaSuccess) {
        cudaFree(d);
        return cuda_fail(e, "gfp_xchg_create");
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
        cudaFree(d);
        return cuda_fail(e, "gfp_xchg_create");
    }
    memcpy(ipc_handle, &h, sizeof h);
    forget_xchg(d);  // a recycled address carries no description
    *buf = d;
    return GFP_OK;
}

gfp_status gfp_xchg_open(const void *ipc_handle, void **peer_buf) {
    if (ipc_handle == nullptr || peer_buf == nullptr) return fail(GFP_E_INVAL, "gfp_xchg_open: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof h);
    void *d = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "gfp_xchg_open (peer access over NVLink / PCIe required)");
    *peer_buf = d;
    return GFP_OK;
}

gfp_status gfp_xchg_close(void *peer_buf) {
    if (peer_buf == nullptr) return fail(GFP_E_INVAL, "gfp_xchg_close: NULL");
    cudaError_t e = cudaIpcCloseMemHandle(peer_buf);
    return e == cudaSuccess ? GFP_OK : cuda_fail(e, "gfp_xchg_close");
}

gfp_status gfp_xchg_destroy(void *buf) {
    if (buf == nullptr) return fail(GFP_E_INVAL, "gfp_xchg_destroy: NULL");
    forget_xchg(buf);
    cudaError_t e = cudaFree(buf);
    return e == cudaSuccess ? GFP_OK : cuda_fail(e, "gfp_xchg_destroy");
}

gfp_status gfp_xchg_soft_timeout(void *own_buf, uint64_t ns) {
    if (own_buf == nullptr || !aligned(own_buf, 8)) return fail(GFP_E_INVAL, "gfp_xchg_soft_timeout: bad buffer");
    const uint64_t w[2] = {ns, 0};  // [kXSoft], and clear [kXTimedOut]
    cudaError_t e = cudaMemcpy((uint64_t *)own_buf + kXSoft, w, sizeof w, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? GFP_OK : cuda_fail(e, "gfp_xchg_soft_timeout");
}

gfp_status gfp_xchg_timed_out(void *own_buf, int32_t *timed_out) {
    if (own_buf == nullptr || timed_out == nullptr || !aligned(own_buf, 8))
        return fail(GFP_E_INVAL, "gfp_xchg_timed_out: bad arguments");
    uint64_t v = 0;
    cudaError_t e = cudaMemcpy(&v, (uint64_t *)own_buf + kXTimedOut, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "gfp_xchg_timed_out");
    *timed_out = v != 0;
    return GFP_OK;
}

gfp_status gfp_dot_allreduce(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                             const gfp_xchg *x, void *out, void *stream) {
    if (x == nullptr) return fail(GFP_E_INVAL, "gfp_dot_allreduce: x is NULL");
    if (x->world < 1 || x->world > GFP_XCHG_MAX_WORLD || x->rank < 0 || x->rank >= x->world)
        return fail(GFP_E_INVAL, "gfp_dot_allreduce: need 1 <= world <= 16 and 0 <= rank < world");
    for (int r = 0; r < x->world; ++r)
        if (x->peers[r] == nullptr || !aligned(x->peers[r], 8))
            return fail(GFP_E_INVAL, "gfp_dot_allreduce: peers[r] must be an 8-byte aligned exchange buffer");
    // rank, world and the peer table live in this rank's own buffer (one kernel pointer parameter); a tiny
    // kernel writes them, stream-ordered before the dot, whenever this buffer's group description changes
    uint64_t *own = (uint64_t *)x->peers[x->rank];
    std::vector<uint64_t> desc(2 + GFP_XCHG_MAX_WORLD, 0);
    desc[0] = (uint64_t)x->rank;
    desc[1] = (uint64_t)x->world;
    for (int r = 0; r < x->world; ++r) desc[2 + r] = (uint64_t)(uintptr_t)x->peers[r];
    {
        std::lock_guard<std::mutex> g(g_xmu);
        auto it = g_xdesc.find(own);
        if (it == g_xdesc.end() || it->second != desc) {
            cudaError_t e = launch_xchg_setup(own, x->rank, x->world, (uint64_t *const *)x->peers, (cudaStream_t)stream);
            if (e != cudaSuccess) return cuda_fail(e, "gfp_dot_allreduce: group description");
            g_xdesc[own] = desc;
        }
    }
    return dot_common(p, rep, dt, a, b, n, out, OUT_XCHG, (cudaStream_t)stream, nullptr, own);
}


}  // extern "C"

// ------------------------------------------------------------------------------ NVLS multicast exchange
// Driver-API calls (multicast objects, virtual memory management) through cudaGetDriverEntryPoint: libgfp.so does
// not link libcuda, so it still loads on hosts without a GPU driver (the CPU tests).
namespace {
struct McApi {
    CUresult (*mcGetGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags) = nullptr;
    CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *) = nullptr;
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long) = nullptr;
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long) = nullptr;
    CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
    CUresult (*exportHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
    CUresult (*importHandle)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType) = nullptr;
    CUresult (*deviceGet)(CUdevice *, int) = nullptr;
    CUresult (*deviceGetAttribute)(int *, CUdevice_attribute, CUdevice) = nullptr;
    bool ok = false;
};

const McApi *mc_api(std::string *why) {
    static McApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        bool all = true;
        auto get = [&](const char *name, auto &fn) {
            void *f = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
                f == nullptr)
                all = false;
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(f);
        };
        get("cuMulticastGetGranularity", api.mcGetGranularity);
        get("cuMulticastCreate", api.mcCreate);
        get("cuMulticastAddDevice", api.mcAddDevice);
        get("cuMulticastBindMem", api.mcBindMem);
        get("cuMulticastUnbind", api.mcUnbind);
        get("cuMemCreate", api.memCreate);
        get("cuMemRelease", api.memRelease);
        get("cuMemAddressReserve", api.addrReserve);
        get("cuMemAddressFree", api.addrFree);
        get("cuMemMap", api.memMap);
        get("cuMemUnmap", api.memUnmap);
        get("cuMemSetAccess", api.memSetAccess);
        get("cuMemExportToShareableHandle", api.exportHandle);
        get("cuMemImportFromShareableHandle", api.importHandle);
        get("cuDeviceGet", api.deviceGet);
        get("cuDeviceGetAttribute", api.deviceGetAttribute);
        api.ok = all;
    });
    if (!api.ok && why) *why = "the CUDA driver does not provide the multicast / VMM entry points";
    return api.ok ? &api : nullptr;
}

gfp_status cu_fail(CUresult r, const char *where) {
    t_err = std::string(where) + ": CUDA driver error " + std::to_string((int)r);
    return GFP_E_CUDA;
}
}  // namespace

struct gfp_mc {
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    CUdeviceptr mc_va = 0, uc_va = 0;
    size_t size = 0;
    int world = 0, fd = -1, dev = -1;
    bool added = false, bound = false, mc_mapped = false, uc_mapped = false, ready = false;
};

extern "C" {

gfp_status gfp_mc_create(int32_t world, gfp_mc **mc, int32_t *fd, uint64_t *bytes) {
    if (mc == nullptr || world < 1 || world > GFP_XCHG_MAX_WORLD)
        return fail(GFP_E_INVAL, "gfp_mc_create: need mc and 1 <= world <= 16");
    std::string why;
    const McApi *A = mc_api(&why);
    if (!A) return fail(GFP_E_UNSUPPORTED, why);
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce != cudaSuccess) return cuda_fail(ce, "gfp_mc_create");
    CUdevice cd;
    CUresult r = A->deviceGet(&cd, dev);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuDeviceGet");
    int supported = 0;
    r = A->deviceGetAttribute(&supported, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd);
    if (r != CUDA_SUCCESS || !supported) return fail(GFP_E_UNSUPPORTED, "gfp_mc_create: multicast (NVLS) not supported here");
    CUmulticastObjectProp prop;
    memset(&prop, 0, sizeof prop);
    prop.numDevices = (unsigned)world;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = kMcWords * sizeof(uint64_t);
    size_t gran = 0;
    if ((r = A->mcGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED)) != CUDA_SUCCESS)
        return cu_fail(r, "cuMulticastGetGranularity");
    prop.size = (prop.size + gran - 1) / gran * gran;
    gfp_mc *m = new gfp_mc();
    m->size = prop.size;
    m->world = world;
    if ((r = A->mcCreate(&m->mc, &prop)) != CUDA_SUCCESS) {
        delete m;
        // the properties are valid by construction (size a multiple of the granularity): a refusal means this
        // platform (driver, fabric manager, visible devices) offers no multicast team
        if (r == CUDA_ERROR_INVALID_VALUE || r == CUDA_ERROR_NOT_SUPPORTED || r == CUDA_ERROR_NOT_PERMITTED)
            return fail(GFP_E_UNSUPPORTED, "gfp_mc_create: the driver refused a multicast object (CUDA driver error " +
                                               std::to_string((int)r) + "): no NVLS multicast team on this platform");
        return cu_fail(r, "cuMulticastCreate");
    }
    if (fd != nullptr) {
        int h = -1;
        if ((r = A->exportHandle(&h, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS) {
            A->memRelease(m->mc);
            delete m;
            return cu_fail(r, "cuMemExportToShareableHandle");
        }
        *fd = h;
        m->fd = h;
    }
    if (bytes) *bytes = m->size;
    *mc = m;
    return GFP_OK;
}

gfp_status gfp_mc_import(int32_t fd, uint64_t bytes, int32_t world, gfp_mc **mc) {
    if (mc == nullptr || fd < 0 || bytes == 0 || world < 1 || world > GFP_XCHG_MAX_WORLD)
        return fail(GFP_E_INVAL, "gfp_mc_import: need mc, fd >= 0, bytes > 0, 1 <= world <= 16");
    std::string why;
    const McApi *A = mc_api(&why);
    if (!A) return fail(GFP_E_UNSUPPORTED, why);
    gfp_mc *m = new gfp_mc();
    m->size = bytes;
    m->world = world;
    CUresult r = A->importHandle(&m->mc, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) {
        delete m;
        return cu_fail(r, "cuMemImportFromShareableHandle");
    }
    *mc = m;
    return GFP_OK;
}

gfp_status gfp_mc_add_device(gfp_mc *m) {
    if (m == nullptr || m->added) return fail(GFP_E_INVAL, "gfp_mc_add_device: NULL or already added");
    const McApi *A = mc_api(nullptr);
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce != cudaSuccess) return cuda_fail(ce, "gfp_mc_add_device");
    CUdevice cd;
    CUresult r = A->deviceGet(&cd, dev);
    if (r == CUDA_SUCCESS) r = A->mcAddDevice(m->mc, cd);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMulticastAddDevice");
    m->dev = dev;
    m->added = true;
    return GFP_OK;
}

gfp_status gfp_mc_bind(gfp_mc *m) {
    if (m == nullptr || !m->added || m->bound) return fail(GFP_E_INVAL, "gfp_mc_bind: NULL, not added, or bound");
    if (m->mem) return fail(GFP_E_INVAL, "gfp_mc_bind: a previous bind failed part-way: destroy and recreate");
    const McApi *A = mc_api(nullptr);
    CUdevice cd;
    CUresult r = A->deviceGet(&cd, m->dev);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuDeviceGet");
    CUmemAllocationProp prop;
    memset(&prop, 0, sizeof prop);
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = m->dev;
    CUmemAccessDesc acc;
    memset(&acc, 0, sizeof acc);
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    // every step records what it set up, so that gfp_mc_destroy undoes exactly that after a partial failure
    if ((r = A->memCreate(&m->mem, m->size, &prop, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemCreate");
    if ((r = A->mcBindMem(m->mc, 0, m->mem, 0, m->size, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMulticastBindMem");
    m->bound = true;
    if ((r = A->addrReserve(&m->mc_va, m->size, m->size, 0, 0)) != CUDA_SUCCESS) return cu_fail(r, "multicast reserve");
    if ((r = A->memMap(m->mc_va, m->size, 0, m->mc, 0)) != CUDA_SUCCESS) return cu_fail(r, "multicast map");
    m->mc_mapped = true;
    if ((r = A->memSetAccess(m->mc_va, m->size, &acc, 1)) != CUDA_SUCCESS) return cu_fail(r, "multicast access");
    if ((r = A->addrReserve(&m->uc_va, m->size, m->size, 0, 0)) != CUDA_SUCCESS) return cu_fail(r, "unicast reserve");
    if ((r = A->memMap(m->uc_va, m->size, 0, m->mem, 0)) != CUDA_SUCCESS) return cu_fail(r, "unicast map");
    m->uc_mapped = true;
    if ((r = A->memSetAccess(m->uc_va, m->size, &acc, 1)) != CUDA_SUCCESS) return cu_fail(r, "unicast access");
    // zero this rank's copy, then record the group size in its private words (the caller synchronises the
    // group -- e.g. a barrier -- before any rank's first gfp_dot_allreduce_mc)
    std::vector<uint64_t> init(kMcWords, 0);
    init[1] = (uint64_t)m->world;
    cudaError_t ce = cudaMemset((void *)m->uc_va, 0, m->size);
    if (ce == cudaSuccess) ce = cudaMemcpy((void *)m->uc_va, init.data(), init.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) return cuda_fail(ce, "gfp_mc_bind: init");
    m->ready = true;
    return GFP_OK;
}

gfp_status gfp_mc_destroy(gfp_mc *m) {
    if (m == nullptr) return fail(GFP_E_INVAL, "gfp_mc_destroy: NULL");
    const McApi *A = mc_api(nullptr);
    cudaDeviceSynchronize();
    if (m->mc_mapped) A->memUnmap(m->mc_va, m->size);
    if (m->mc_va) A->addrFree(m->mc_va, m->size);
    if (m->uc_mapped) A->memUnmap(m->uc_va, m->size);
    if (m->uc_va) A->addrFree(m->uc_va, m->size);
    if (m->bound) {
        CUdevice cd;
        if (A->deviceGet(&cd, m->dev) == CUDA_SUCCESS) A->mcUnbind(m->mc, cd, 0, m->size);
    }
    if (m->mem) A->memRelease(m->mem);
    if (m->mc) A->memRelease(m->mc);
    if (m->fd >= 0) close(m->fd);
    delete m;
    return GFP_OK;
}

gfp_status gfp_dot_allreduce_mc(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                                gfp_mc *m, void *out, void *stream) {
    if (m == nullptr || !m->ready) return fail(GFP_E_INVAL, "gfp_dot_allreduce_mc: multicast buffer not bound");
    return dot_common(p, rep, dt, a, b, n, out, OUT_MC, (cudaStream_t)stream, nullptr, (uint64_t *)m->uc_va,
                      (uint64_t *)m->mc_va);
}

gfp_status gfp_finalize(uint64_t p, gfp_rep rep, gfp_dtype dt, const uint64_t *summed, void *out, void *stream) {
    if (summed == nullptr || out == nullptr) return fail(GFP_E_INVAL, "NULL pointer");
    if (!aligned(summed, 8) || ((int)dt >= 0 && (int)dt <= 2 && !aligned(out, dtype_size(dt))))
        return fail(GFP_E_INVAL, "misaligned pointer");
    Ctx *c;
    gfp_status st = get_ctx(p, rep, dt, &c);
    if (st != GFP_OK) return st;
    OutSpec o{out, (int)rep, (int)dt, OUT_ENCODE};
    cudaError_t e = launch_finalize(c->K, summed, 1, o, (cudaStream_t)stream);
    return e == cudaSuccess ? GFP_OK : cuda_fail(e, "finalize launch");
}

static gfp_status batch_common(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *A, int64_t lda, const void *x,
                               int64_t rows, int64_t n, const gfp_options *opt, void *out, void *stream) {
    if ((int)dt < 0 || (int)dt > 2) return fail(GFP_E_INVAL, "unknown dtype");
    if (rows < 0 || n < 0 || lda < n) return fail(GFP_E_INVAL, "need rows >= 0, n >= 0, lda >= n");
    if (rows == 0) return GFP_OK;
    if (out == nullptr || (n > 0 && (A == nullptr || x == nullptr))) return fail(GFP_E_INVAL, "NULL pointer");
    const size_t es = dtype_size(dt);
    if (!aligned(A, es) || !aligned(x, es) || !aligned(out, es)) return fail(GFP_E_INVAL, "misaligned pointer");
    Ctx *c;
    gfp_status st = get_ctx(p, rep, dt, &c);
    if (st != GFP_OK) return st;
    OutSpec o{out, (int)rep, (int)dt, OUT_ENCODE};
    cudaError_t e = cudaSuccess;
    st = launch_batch(c->info, c->K, A, lda, x, rows, n, opt, o, (cudaStream_t)stream, &e);
    if (st == GFP_E_CUDA) return cuda_fail(e, "batch launch");
    if (st != GFP_OK) return plan_fail(st);
    return GFP_OK;
}

gfp_status gfp_dot_batch(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *A, int64_t lda, const void *x,
                         int64_t rows, int64_t n, void *out, void *stream) {
    return batch_common(p, rep, dt, A, lda, x, rows, n, nullptr, out, stream);
}

gfp_status gfp_dot_batch_ex(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *A, int64_t lda, const void *x,
                            int64_t rows, int64_t n, const gfp_options *opt, void *out, void *stream) {
    return batch_common(p, rep, dt, A, lda, x, rows, n, opt, out, stream);
}

gfp_status gfp_dot_ex(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                      const gfp_options *opt, void *out, void *stream) {
    return dot_common(p, rep, dt, a, b, n, out, OUT_ENCODE, (cudaStream_t)stream, opt);
}

gfp_status gfp_plan(uint64_t p, gfp_rep rep, gfp_dtype dt, int64_t n, const gfp_options *opt, gfp_plan_info *info) {
    if (info == nullptr || n < 0) return fail(GFP_E_INVAL, "info is NULL or n < 0");
    gfp_info I;
    gfp_status st = gfp_query(p, rep, dt, &I);
    if (st != GFP_OK) return st;
    dev::KParams K;  // planning needs only the table size (no device tables are built here)
    memset(&K, 0, sizeof(K));
    K.p = p;
    K.antilog_entries = (uint32_t)((I.table_bytes / 2 + 7) & ~uint64_t(7));
    K.zplus1_entries = (uint32_t)((p + 1 + 7) & ~uint64_t(7));  // qbar + 2 = p + 1 entries
    K.zplus1s_entries = 65536;  // the fast pure-Zech table, padded (see zech context setup)
    DotPlan plan;
    const void *aligned_ptr = (const void *)(uintptr_t)4096;
    if ((st = plan_dot(I, K, aligned_ptr, aligned_ptr, n, opt, &plan)) != GFP_OK) return plan_fail(st);
    memset(info, 0, sizeof(*info));
    info->strategy = plan.strategy;
    info->acc_bits = plan.acc_bits;
    info->block = plan.kblk;
    info->grid = plan.grid;
    info->threads_per_block = plan.block;
    info->terms_per_thread = plan.per_thread;
    info->reductions_per_thread = plan.reductions;
    snprintf(info->kernel, sizeof(info->kernel), "%s", plan.name);
    return GFP_OK;
}

static gfp_status convert(uint64_t p, gfp_rep rep, int dir, gfp_dtype in_dt, const void *in, gfp_dtype out_dt,
                          void *out, int64_t n, void *stream) {
    if ((int)in_dt < 0 || (int)in_dt > 2 || (int)out_dt < 0 || (int)out_dt > 2)
        return fail(GFP_E_INVAL, "unknown dtype");
    if (n < 0) return fail(GFP_E_INVAL, "n < 0");
    if (n > 0 && (in == nullptr || out == nullptr)) return fail(GFP_E_INVAL, "NULL pointer");
    if (!aligned(in, dtype_size(in_dt)) || !aligned(out, dtype_size(out_dt)))
        return fail(GFP_E_INVAL, "misaligned pointer");
    if (in == out && in_dt != out_dt) return fail(GFP_E_INVAL, "in-place conversion needs in_dt == out_dt");
    const gfp_dtype rep_dt = dir == 0 ? out_dt : in_dt;
    Ctx *c;
    gfp_status st = get_ctx(p, rep, rep_dt, &c);
    if (st != GFP_OK) return st;
    if (n == 0) return GFP_OK;
    cudaError_t e = cudaSuccess;
    st = launch_convert(c->info, c->K, dir, in_dt, in, out_dt, out, n, (cudaStream_t)stream, &e);
    if (st == GFP_E_CUDA) return cuda_fail(e, "convert launch");
    if (st != GFP_OK) return fail(st, "unsupported conversion dtypes for this representation");
    return GFP_OK;
}

gfp_status gfp_to_rep(uint64_t p, gfp_rep rep, gfp_dtype in_dt, const void *in, gfp_dtype out_dt, void *out,
                      int64_t n, void *stream) {
    return convert(p, rep, 0, in_dt, in, out_dt, out, n, stream);
}

gfp_status gfp_from_rep(uint64_t p, gfp_rep rep, gfp_dtype in_dt, const void *in, gfp_dtype out_dt, void *out,
                        int64_t n, void *stream) {
    return convert(p, rep, 1, in_dt, in, out_dt, out, n, stream);
}

// gfp_dot_host / gfp_dot_host_partial: partial_only writes the additive-form residue (u64) instead of the
// encoded element.
static gfp_status dot_host_common(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                                  void *out, void *stream, bool partial_only) {
    gfp_status st = check_dot_args(dt, a, b, n, out, 1);
    if (st != GFP_OK) return st;
    Ctx *c;
    if ((st = get_ctx(p, rep, dt, &c)) != GFP_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace ws;
    if ((st = get_ws(s, &ws)) != GFP_OK) return st;
    const int dev = current_device();
    const size_t es = dtype_size(dt);
    Staging *S;
    {
        std::lock_guard<std::mutex> g(g_stage_mu);
        auto it = g_stage.find(dev);
        if (it == g_stage.end()) {
            S = new Staging();
            S->chunk_bytes = 64ull << 20;  // per operand per slot
            cudaError_t e = cudaSuccess;
            for (int i = 0; i < 2 && e == cudaSuccess; ++i)
                for (int j = 0; j < 2 && e == cudaSuccess; ++j) e = cudaMalloc(&S->buf[i][j], S->chunk_bytes);
            if (e == cudaSuccess) e = cudaMalloc(&S->d_partial, 64);
            if (e == cudaSuccess) e = cudaMalloc(&S->d_out, 64);
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&S->copy, cudaStreamNonBlocking);
            for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
                e = cudaEventCreateWithFlags(&S->copied[i], cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&S->consumed[i], cudaEventDisableTiming);
            }
            if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
            g_stage[dev] = S;
        } else {
            S = it->second;
        }
    }
    std::lock_guard<std::mutex> g(g_stage_mu);  // one host pipeline per device at a time
    const int64_t chunk = (int64_t)(S->chunk_bytes / es) & ~int64_t(7);
    const int64_t nchunks = n == 0 ? 1 : (n + chunk - 1) / chunk;
    cudaError_t e = cudaSuccess;
    for (int64_t ci = 0; ci < nchunks && e == cudaSuccess; ++ci) {
        const int slot = (int)(ci & 1);
        const int64_t off = ci * chunk, len = std::min<int64_t>(chunk, n - off);
        if (ci >= 2) e = cudaStreamWaitEvent(S->copy, S->consumed[slot], 0);  // slot free again
        if (len > 0 && e == cudaSuccess)
            e = cudaMemcpyAsync(S->buf[slot][0], (const char *)a + off * es, len * es, cudaMemcpyHostToDevice, S->copy);
        if (len > 0 && e == cudaSuccess)
            e = cudaMemcpyAsync(S->buf[slot][1], (const char *)b + off * es, len * es, cudaMemcpyHostToDevice, S->copy);
        if (e == cudaSuccess) e = cudaEventRecord(S->copied[slot], S->copy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, S->copied[slot], 0);
        if (e != cudaSuccess) break;
        DotPlan plan;
        if ((st = plan_dot(c->info, c->K, S->buf[slot][0], S->buf[slot][1], std::max<int64_t>(len, 0), nullptr,
                           &plan)) != GFP_OK)
            return plan_fail(st);
        OutSpec o{S->d_partial, (int)rep, (int)dt, ci == 0 ? OUT_PARTIAL : OUT_ACCUMULATE};
        e = launch_dot(plan, c->K, S->buf[slot][0], S->buf[slot][1], std::max<int64_t>(len, 0), ws, o, s);
        if (e == cudaSuccess) e = cudaEventRecord(S->consumed[slot], s);
    }
    if (e == cudaSuccess && !partial_only) {
        OutSpec o{S->d_out, (int)rep, (int)dt, OUT_ENCODE};
        e = launch_finalize(c->K, S->d_partial, 1, o, s);
    }
    // the chunks' partials are residues < p summed over at most n / chunk + 1 chunks: no wrap
    if (e == cudaSuccess)
        e = partial_only ? cudaMemcpyAsync(out, S->d_partial, 8, cudaMemcpyDeviceToHost, s)
                         : cudaMemcpyAsync(out, S->d_out, es, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    // the chunks' residues were summed on the device: one remainder makes the partial a residue in [0, p)
    if (e == cudaSuccess && partial_only) *(uint64_t *)out %= p;
    return e == cudaSuccess ? GFP_OK : cuda_fail(e, "gfp_dot_host");
}

gfp_status gfp_dot_host(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n, void *out,
                        void *stream) {
    return dot_host_common(p, rep, dt, a, b, n, out, stream, false);
}

gfp_status gfp_dot_host_partial(uint64_t p, gfp_rep rep, gfp_dtype dt, const void *a, const void *b, int64_t n,
                                uint64_t *partial, void *stream) {
    if (partial != nullptr && !aligned(partial, 8)) return fail(GFP_E_INVAL, "partial not 8-byte aligned");
    return dot_host_common(p, rep, dt, a, b, n, partial, stream, true);
}

uint64_t gfp_launch_count(int reset) { return launches(reset); }

const char *gfp_status_str(gfp_status s) {
    switch (s) {
    case GFP_OK: return "GFP_OK";
    case GFP_E_INVAL: return "GFP_E_INVAL: invalid argument";
    case GFP_E_NOT_PRIME: return "GFP_E_NOT_PRIME: modulus is not prime";
    case GFP_E_BOUND: return "GFP_E_BOUND: modulus outside the representation bound";
    case GFP_E_UNSUPPORTED: return "GFP_E_UNSUPPORTED: representation/dtype not supported";
    case GFP_E_CUDA: return "GFP_E_CUDA: CUDA error";
    case GFP_E_NOMEM: return "GFP_E_NOMEM: allocation failed";
    }
    return "unknown gfp_status";
}

const char *gfp_last_error(void) { return t_err.c_str(); }

void gfp_release_caches(void) {
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> g(g_mu);
    for (auto &kv : g_ctx) {
        cudaFree(kv.second->d_antilog);
        cudaFree(kv.second->d_log);
        cudaFree(kv.second->d_zplus1);
        cudaFree(kv.second->d_zplus1s);
        delete kv.second;
    }
    g_ctx.clear();
    for (auto &kv : g_ws) cudaFree(kv.second.partials);
    g_ws.clear();
    std::lock_guard<std::mutex> g2(g_stage_mu);
    for (auto &kv : g_stage) {
        Staging *S = kv.second;
        for (auto &row : S->buf)
            for (void *q : row) cudaFree(q);
        cudaFree(S->d_partial);
        cudaFree(S->d_out);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(S->copied[i]);
            cudaEventDestroy(S->consumed[i]);
        }
        cudaStreamDestroy(S->copy);
        delete S;
    }
    g_stage.clear();
}

const char *gfp_version(void) { return "gfp-b200 0.1.0 (sm_100a)"; }

}  // extern "C"
