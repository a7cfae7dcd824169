// =====================================================================================
// Host side of the C ABI (include/rtm.h): validation, CFL check, device buffers, streams,
// CUDA graphs, source tables, z-slab decomposition with in-process peer copies or NCCL
// send/recv halo exchange.  All arithmetic of the step runs in
// the kernels of rtm_kernels.cu; nothing here computes field values.
// =====================================================================================
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rtm_internal.h"

using namespace rtm;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(RTM_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                             \
    } while (0)

#define NK(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(RTM_ENCCL, "%s failed: %s (%s:%d)", #call, ncclGetErrorString(r_), \
                        __FILE__, __LINE__);                                                  \
    } while (0)

#define RET(call)             \
    do {                      \
        int rc_ = (call);     \
        if (rc_ != RTM_OK) return rc_; \
    } while (0)

struct DeviceGuard {  // restore the caller's current device
    int saved = -1;
    DeviceGuard() { cudaGetDevice(&saved); }
    ~DeviceGuard() {
        if (saved >= 0) cudaSetDevice(saved);
    }
};

struct HostSource {
    int x, y, z;  // global
    int shot;
    std::vector<float> samples;
};

constexpr int GRAPH_PAIRS = 8;  // a captured graph advances 2*GRAPH_PAIRS steps

struct Slab {
    int dev = 0;
    int z0 = 0, nzl = 0;
    int nshots = 1;                      // batched independent wavefields sharing C
    int share = 1;                       // slabs of this context on the same device
    bool lo_nb = false, hi_nb = false;
    float* buf[2] = {nullptr, nullptr};  // nshots*(nzl+10) planes each
    size_t buf_planes() const { return (size_t)nshots * (nzl + 10); }
    float* C = nullptr;                  // nzl planes
    int* d_step = nullptr;               // [2]
    unsigned int* d_stats = nullptr;     // [2] velocity check (also the deferred async verdict)
    unsigned int* d_fstats = nullptr;    // [2] field check (rtm_field_stats): its own buffer, so a
                                         // scan never overwrites a pending velocity verdict
    int tb_nbands = -1;                  // band count of the last two-step plan (flags reset on change)
    float* d_samples = nullptr;
    std::vector<DevSource> srcs;
    std::vector<float> h_samples;
    cudaStream_t s_own = nullptr, s_comm = nullptr, s_user = nullptr;
    bool has_user = false;
    cudaEvent_t ev_bnd = nullptr, ev_comm = nullptr, ev_done = nullptr;
    CUtensorMap tm_u[2];   // u with the halo box, one per time-level buffer
    CUtensorMap tm_in[2];  // TX x TY box over each buffer (u_prev read of k_stream)
    CUtensorMap tm_c;      // TX x TY box over C
    int tm_variant = -1;
    int occupancy = 0;     // resident CTAs per SM of tm_variant
    cudaGraphExec_t graph = nullptr;
    cudaGraph_t graph_def = nullptr;
    int graph_variant = -1;
    int graph_bank = 0;
    bool graph_valid = false;
    // two-step passes (kind 4): the second bank they write, then the banks swap
    float* alt[2] = {nullptr, nullptr};
    int bank = 0;                              // toggled at every bank swap
    unsigned long long* d_flags = nullptr;     // stage-A progress per CTA of a band
    unsigned long long* d_epoch = nullptr;     // pass epoch (never reset)
    unsigned* d_bar = nullptr;                 // k_resident grid barrier [2]
    cudaGraphExec_t tb_graph[4] = {nullptr, nullptr, nullptr, nullptr};  // key bank*2 + parity
    unsigned long long* d_msflags = nullptr;   // multi-step launches: progress flag per work unit
    long long ms_units = 0;                    // capacity of d_msflags
    unsigned long long ms_epoch = 0;           // per-launch tag (upper 32 bits of the flags)
    int tb_graph_variant[4] = {-1, -1, -1, -1};
    // fused halo push with the flag protocol (halo mode 2): the neighbours' time-level buffers
    // and flag words — direct pointers in-process, CUDA-IPC mappings across processes
    unsigned long long* d_sig = nullptr;       // [4]: steps completed by the lo / hi neighbour
                                               // ([0] / [1], mode 2), boundary of step n ready
                                               // at the lo / hi neighbour ([2] / [3], mode 3)
    float* nb_lo[2] = {nullptr, nullptr};
    float* nb_hi[2] = {nullptr, nullptr};
    int nb_lo_nzl = 0;
    unsigned long long* nb_lo_sig = nullptr;   // the lo neighbour's d_sig (we write its [1] / [3])
    unsigned long long* nb_hi_sig = nullptr;   // the hi neighbour's d_sig (we write its [0] / [2])
    std::vector<void*> ipc_open;               // mappings to cudaIpcCloseMemHandle
    cudaStream_t stream() const { return has_user ? s_user : s_own; }
};

}  // namespace

struct rtm_ctx {
    int mode = 0;  // 0 single, 1 multi (in-process slabs), 2 dist (NCCL), 3 peer (CUDA IPC, no NCCL)
    int nx = 0, ny = 0, nz = 0;  // nz = global planes
    int px = 0;                  // device row pitch in floats: nx rounded up to a multiple of 4
    float dx = 0, dt = 0;
    float coeffs[6] = {};
    double nu_crit = 0;
    std::vector<Slab> slabs;
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    long long step = 0;
    bool vel_set = false;
    int tile = -1;
    int zchunk = 0;  // 0 = auto
    int cache_mode = 0x45;  // u box TMA evict_last (+0.8 % on C4, profiles/sweep_cache_r01h.log); D=0 variants: L2 prefetch of u_prev/C 4 planes ahead, evict_last
    int shot_order = 0;     // 0 auto, 1 shot-major, 2 shot-fastest
    int halo_mode = 0;      // slabs: 0 boundary first + copies / NCCL, 1 fused push (events,
                            // in-process), 2 fused push + flag protocol (in-process or IPC),
                            // 3 copy-engine pull + flag protocol (in-process or IPC)
    bool host_ordered = false;       // RTM_OPT_HOST_ORDERED: rank barrier before flag waits
    bool ipc_imported = false;       // peer / dist contexts: neighbours' records opened
    rtm_barrier_fn barrier_fn = nullptr;  // peer contexts: the caller's rank barrier
    void* barrier_user = nullptr;
    double enqueue_ms = 0;           // host enqueue time of the last rtm_step
    bool slab_graphs_broken = false; // capture of the slab step failed once: direct launches
    unsigned long long sig_gen = 0;  // flag generation (bumped at every synchronising reset)
    bool sig_fresh = true;           // first step of a generation: no flag waits
    unsigned sig_flush = 0;          // CU_STREAM_WAIT_VALUE_FLUSH when the devices support it
    int check_every = 0;    // NaN/Inf scan every k steps (0 = off)
    int tb_ctas = 0;        // two-step passes: max CTAs per band (0 = #SMs)
    bool pdl = false;       // programmatic dependent launch of consecutive k_stream steps
    bool share_sms = false; // RTM_OPT_SLAB_SHARE: slabs sharing a device split its SMs
    int zdir = 2;           // RTM_OPT_ZDIR bits: 1 = k_stream sweeps z downward on odd-parity
                            // steps, 2 = on every other unit (wave) of a CTA
    int l2_bytes = 0;
    bool graphs = true;
    std::vector<HostSource> sources;
    bool profiling = false;
    std::vector<cudaEvent_t> prof_ev;
    std::vector<int> prof_weight;       // stencil launches between each event pair (graph: 16)
    long long prof_launches = 0;        // event pairs recorded in the current rtm_step
    long long prof_total_launches = 0;  // since rtm_set_profiling / last rtm_kernel_stats
    double prof_ms = 0;
    long long launches = 0;
    float last_ms = 0;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    int num_sms = 148;
    // asynchronous host-buffer pipeline (single-slab contexts; rtm_*_async, rtm_sync)
    cudaStream_t s_copy = nullptr;  // D2H of results
    cudaStream_t s_h2d = nullptr;   // H2D of velocities (separate: it must not queue behind a D2H)
    cudaEvent_t ev_h2d = nullptr, ev_conv = nullptr, ev_snap = nullptr, ev_d2h = nullptr;
    float* v_stage = nullptr;   // H2D staging of the next velocity (nx*ny*nz floats)
    float* snap = nullptr;      // device snapshot of u^n for the D2H (nshots*nx*ny*nz floats)
    bool vcheck_pending = false;  // deferred CFL / validity verdict of async velocities
};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

typedef CUresult (*PFN_devattr)(int*, CUdevice_attribute, CUdevice);
template <class F>
F driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<F>(p);
    return nullptr;
}

bool finite_coeffs(const float c[6]) {
    for (int k = 0; k < 6; ++k)
        if (!std::isfinite(c[k])) return false;
    return true;
}

// S_max = max_theta -(c0 + 2 sum_m c_m cos m theta), sampled on [0, pi] and refined.
double smax_of(const float c[6]) {
    auto S = [&](double th) {
        double s = c[0];
        for (int m = 1; m <= 5; ++m) s += 2.0 * c[m] * std::cos(m * th);
        return -s;
    };
    const int N = 8192;
    double best = -1e300, bt = 0;
    for (int i = 0; i <= N; ++i) {
        const double th = M_PI * i / N;
        const double v = S(th);
        if (v > best) best = v, bt = th;
    }
    double lo = std::max(0.0, bt - M_PI / N), hi = std::min(M_PI, bt + M_PI / N);
    for (int it = 0; it < 100; ++it) {  // golden-section refinement
        const double a = lo + (hi - lo) * 0.381966, b = lo + (hi - lo) * 0.618034;
        if (S(a) < S(b)) lo = a; else hi = b;
    }
    return std::max(best, S(0.5 * (lo + hi)));
}

int validate_grid(int nx, int ny, int nz, float dx, float dt, const float* coeffs) {
    if (nx < 1 || ny < 1 || nz < 1)
        return fail(RTM_EINVAL, "grid extents must be >= 1 (nx=%d ny=%d nz=%d)", nx, ny, nz);
    if ((long long)nx * ny > (1LL << 31))
        return fail(RTM_EINVAL, "nx*ny=%lld exceeds 2^31", (long long)nx * ny);
    if (!(std::isfinite(dx) && dx > 0)) return fail(RTM_EINVAL, "dx must be finite and > 0");
    if (!(std::isfinite(dt) && dt > 0)) return fail(RTM_EINVAL, "dt must be finite and > 0");
    if (!coeffs) return fail(RTM_EINVAL, "coeffs is NULL");
    if (!finite_coeffs(coeffs)) return fail(RTM_EINVAL, "coeffs must be finite");
    if (!(smax_of(coeffs) > 0))
        return fail(RTM_EINVAL, "coeffs do not define a negative-definite 2nd difference (S_max <= 0)");
    return RTM_OK;
}

// Device planes are pitched (c->px floats per row); host arrays are unpadded (nx per row).
size_t dplane(const rtm_ctx* c) { return (size_t)c->px * c->ny; }
size_t hplane(const rtm_ctx* c) { return (size_t)c->nx * c->ny; }

int alloc_slab(rtm_ctx* c, Slab& s) {
    CK(cudaSetDevice(s.dev));
    const size_t plane = dplane(c);
    const size_t nbuf = plane * s.buf_planes();
    for (int b = 0; b < 2; ++b) {
        if (cudaMalloc(&s.buf[b], nbuf * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            return fail(RTM_ENOMEM, "cudaMalloc of %zu bytes (field %d) failed", nbuf * 4, b);
        }
    }
    if (cudaMalloc(&s.C, plane * s.nzl * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        return fail(RTM_ENOMEM, "cudaMalloc of %zu bytes (C) failed", plane * s.nzl * 4);
    }
    CK(cudaMalloc(&s.d_step, 2 * sizeof(int)));
    CK(cudaMalloc(&s.d_stats, 2 * sizeof(unsigned int)));
    CK(cudaMalloc(&s.d_fstats, 2 * sizeof(unsigned int)));
    CK(cudaStreamCreateWithFlags(&s.s_own, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s.s_comm, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&s.ev_bnd, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s.ev_comm, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) CK(cudaMemsetAsync(s.buf[b], 0, nbuf * sizeof(float), s.s_own));
    CK(cudaMemsetAsync(s.C, 0, plane * s.nzl * sizeof(float), s.s_own));
    CK(cudaMemsetAsync(s.d_step, 0, 2 * sizeof(int), s.s_own));
    CK(cudaStreamSynchronize(s.s_own));
    return RTM_OK;
}

void free_slab(Slab& s) {
    cudaSetDevice(s.dev);
    if (s.graph) cudaGraphExecDestroy(s.graph);
    if (s.graph_def) cudaGraphDestroy(s.graph_def);
    for (auto& g : s.tb_graph)
        if (g) cudaGraphExecDestroy(g);
    for (int b = 0; b < 2; ++b) {
        if (s.buf[b]) cudaFree(s.buf[b]);
        if (s.alt[b]) cudaFree(s.alt[b]);
    }
    if (s.d_flags) cudaFree(s.d_flags);
    if (s.d_msflags) cudaFree(s.d_msflags);
    if (s.d_bar) cudaFree(s.d_bar);
    if (s.d_epoch) cudaFree(s.d_epoch);
    for (void* q : s.ipc_open) cudaIpcCloseMemHandle(q);
    if (s.d_sig) cudaFree(s.d_sig);
    if (s.C) cudaFree(s.C);
    if (s.d_step) cudaFree(s.d_step);
    if (s.d_stats) cudaFree(s.d_stats);
    if (s.d_fstats) cudaFree(s.d_fstats);
    if (s.d_samples) cudaFree(s.d_samples);
    if (s.ev_bnd) cudaEventDestroy(s.ev_bnd);
    if (s.ev_comm) cudaEventDestroy(s.ev_comm);
    if (s.ev_done) cudaEventDestroy(s.ev_done);
    if (s.s_own) cudaStreamDestroy(s.s_own);
    if (s.s_comm) cudaStreamDestroy(s.s_comm);
    s = Slab();
}

void destroy_ctx(rtm_ctx* c) {
    if (!c) return;
    DeviceGuard g;
    for (auto& s : c->slabs) {
        if (s.s_own) {
            cudaSetDevice(s.dev);
            cudaStreamSynchronize(s.s_own);
            cudaStreamSynchronize(s.s_comm);
        }
    }
    if (c->comm) ncclCommDestroy(c->comm);
    if (!c->slabs.empty()) cudaSetDevice(c->slabs[0].dev);
    for (auto e : c->prof_ev) cudaEventDestroy(e);
    if (c->t0) cudaEventDestroy(c->t0);
    if (c->t1) cudaEventDestroy(c->t1);
    for (cudaStream_t q : {c->s_copy, c->s_h2d})
        if (q) {
            cudaStreamSynchronize(q);
            cudaStreamDestroy(q);
        }
    for (cudaEvent_t e : {c->ev_h2d, c->ev_conv, c->ev_snap, c->ev_d2h})
        if (e) cudaEventDestroy(e);
    if (c->v_stage) cudaFree(c->v_stage);
    if (c->snap) cudaFree(c->snap);
    for (auto& s : c->slabs) free_slab(s);
    delete c;
}

rtm_ctx* new_ctx(int nx, int ny, int nz, float dx, float dt, const float* coeffs) {
    if (validate_grid(nx, ny, nz, dx, dt, coeffs) != RTM_OK) return nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        fail(RTM_ECUDA, "no CUDA device available (the library has no CPU fallback)");
        return nullptr;
    }
    rtm_ctx* c = new rtm_ctx();
    c->nx = nx;
    c->px = (nx + 3) / 4 * 4;
    c->ny = ny;
    c->nz = nz;
    c->dx = dx;
    c->dt = dt;
    std::memcpy(c->coeffs, coeffs, sizeof c->coeffs);
    c->nu_crit = 2.0 / std::sqrt(3.0 * smax_of(coeffs));
    return c;
}

int finish_ctx(rtm_ctx* c) {
    CK(cudaSetDevice(c->slabs[0].dev));
    CK(cudaEventCreate(&c->t0));
    CK(cudaEventCreate(&c->t1));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->slabs[0].dev));
    CK(cudaDeviceGetAttribute(&c->l2_bytes, cudaDevAttrL2CacheSize, c->slabs[0].dev));
    for (auto& s : c->slabs) RET(alloc_slab(c, s));
    return RTM_OK;
}

int resolve_tile(const rtm_ctx* c) {
    if (c->tile >= 0) return c->tile;
    return 35;  // stream64x30k10d6u4: best on C4 (profiles/sweep_c4_s6.log); bench autotunes
}

// The variant that runs single time steps: a two-step variant (kind 4) runs its paired
// k_stream variant for odd remainders and for contexts it does not cover (slabs, shots).
int single_variant(const rtm_ctx* c) {
    const int v = resolve_tile(c);
    const int k = variant(v).kind;
    return (k >= 3 && k != 7) ? variant(v).pair : v;
}

// 3D tensor map over a pitched device field: logical x extent nx (TMA zero-fills x >= nx, so
// the padding columns are never read through it), row stride px floats.
int encode_3d(CUtensorMap* tm, void* base, const rtm_ctx* c, int nplanes, int bx, int by,
              int promo = 3) {
    auto enc = encode_fn();
    if (!enc) return fail(RTM_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t dims[3] = {(cuuint64_t)c->nx, (cuuint64_t)c->ny, (cuuint64_t)nplanes};
    cuuint64_t strides[2] = {(cuuint64_t)c->px * 4, (cuuint64_t)c->px * c->ny * 4};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                     : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                     : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                  : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(RTM_ECUDA, "cuTensorMapEncodeTiled(box %dx%d) failed (%d)", bx, by, (int)r);
    return RTM_OK;
}

int ensure_tmaps(rtm_ctx* c, Slab& s, int var) {
    // promotion of the halo'd u box: cache_mode bits 8-9 hold 3 - promo (0 = 256B default)
    const int promo = 3 - ((c->cache_mode >> 8) & 3);
    const int key = var * 4 + promo;
    if (var == 0 || s.tm_variant == key) return RTM_OK;
    const TileVariant& tv = variant(var);
    for (int b = 0; b < 2; ++b) {
        RET(encode_3d(&s.tm_u[b], s.buf[b], c, (int)s.buf_planes(), tv.TX + 16,
                      tv.TY + 10, promo));
        RET(encode_3d(&s.tm_in[b], s.buf[b], c, (int)s.buf_planes(), tv.TX, tv.TY));
    }
    RET(encode_3d(&s.tm_c, s.C, c, s.nzl, tv.TX, tv.TY));
    int tpb = 0;
    s.occupancy = variant_occupancy(var, &tpb);
    if (s.occupancy < 1)
        return fail(RTM_ECUDA, "variant %s cannot be resident on this device", tv.name);
    s.tm_variant = key;
    return RTM_OK;
}

// z-chunks for a range of len planes: minimise (wave quantisation) x (chunk-halo re-read).
int choose_chunks(const rtm_ctx* c, int occ, int ntiles, int len, int share = 1) {
    if (c->zchunk > 0) return std::max(1, (len + c->zchunk - 1) / c->zchunk);
    if (occ < 1) occ = 1;
    const double S = std::max(1.0, (double)c->num_sms * occ / share);
    int best = 1;
    double bestc = 1e300;
    const int maxc = std::max(1, len / 8);
    for (int nc = 1; nc <= maxc; ++nc) {
        const double units = (double)ntiles * nc;
        const double waves = units / S;
        const double eff = std::ceil(waves - 1e-9) / waves;
        const double zc = (double)len / nc;
        const double cost = eff * (1.0 + 2.5 / zc);
        if (cost < bestc - 1e-12) bestc = cost, best = nc;
    }
    return best;
}

void fill_params(const rtm_ctx* c, const Slab& s, int parity, StencilParams& p) {
    std::memset(&p, 0, sizeof p);
    p.nx = c->nx;
    p.ny = c->ny;
    p.nzl = s.nzl;
    p.pitch = c->px;
    p.nshots = s.nshots;
    p.plane = (long long)dplane(c);
    p.coef[0] = 3.0f * c->coeffs[0];
    for (int k = 1; k < 6; ++k) p.coef[k] = c->coeffs[k];
    p.u = s.buf[parity];
    p.next = s.buf[parity ^ 1];
    p.C = s.C;
    p.d_step = s.d_step;
    p.parity = parity;
    p.nsrc = (int)s.srcs.size();
    for (int k = 0; k < p.nsrc; ++k) p.src[k] = s.srcs[k];
    p.samples = s.d_samples;
    p.cache_mode = c->cache_mode;
    p.zalt = c->zdir;
    // auto: shot-major when one C field fits comfortably in L2 (it is then re-read from L2 by
    // every shot and the shots keep the full co-running tile set for halo reuse); otherwise
    // shot-fastest so co-running CTAs share each C tile
    const double c_bytes = 4.0 * c->nx * c->ny * s.nzl;
    p.shot_major = c->shot_order == 1 ? 1 : c->shot_order == 2 ? 0 : (c_bytes <= 0.4 * c->l2_bytes ? 1 : 0);
}

// Launch the stencil on planes [b0,b0+l0) (+ [b1,b1+l1) if l1 > 0) of slab s.
int launch_stencil(rtm_ctx* c, Slab& s, int parity, int b0, int l0, int b1, int l1,
                   int write_next, cudaStream_t st, float* push_lo = nullptr,
                   float* push_hi = nullptr) {
    const int var = single_variant(c);
    StencilParams p;
    fill_params(c, s, parity, p);
    p.push_lo = push_lo;
    p.push_hi = push_hi;
    p.write_next = write_next;
    p.nranges = l1 > 0 ? 2 : 1;
    p.r_begin[0] = b0;
    p.r_len[0] = l0;
    p.r_begin[1] = b1;
    p.r_len[1] = l1 > 0 ? l1 : 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) {
        const size_t k = 2 * (size_t)c->prof_launches;
        while (c->prof_ev.size() < k + 2) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            c->prof_ev.push_back(e);
        }
        e0 = c->prof_ev[k];
        e1 = c->prof_ev[k + 1];
        CK(cudaEventRecord(e0, st));
    }
    if (var == 0) {
        CK(launch_naive(p, st));
    } else {
        RET(ensure_tmaps(c, s, var));
        const TileVariant& tv = variant(var);
        p.tiles_x = (c->nx + tv.TX - 1) / tv.TX;
        p.tiles_y = (c->ny + tv.TY - 1) / tv.TY;
        const int nt = p.tiles_x * p.tiles_y;
        // slabs that share a device (one-GPU decomposition runs) may split its SMs so that all of
        // them run concurrently (RTM_OPT_SLAB_SHARE); otherwise every launch gets all SMs
        const int share = c->share_sms ? s.share : 1;
        p.r_chunks[0] = choose_chunks(c, s.occupancy, nt * s.nshots, l0, share);  // units = tiles x chunks x shots
        p.r_chunks[1] = l1 > 0 ? choose_chunks(c, s.occupancy, nt * s.nshots, l1, share) : 0;
        CK(launch_variant(var, &s.tm_u[parity], &s.tm_in[parity ^ 1], &s.tm_c, p,
                          std::max(1, c->num_sms * s.occupancy / share), st,
                          c->pdl && (variant(var).kind == 2 || variant(var).kind == 7)));
    }
    if (c->profiling) {
        CK(cudaEventRecord(e1, st));
        if (c->prof_weight.size() <= (size_t)c->prof_launches) c->prof_weight.resize(c->prof_launches + 1);
        c->prof_weight[c->prof_launches] = 1;
        ++c->prof_launches;
    }
    ++c->launches;
    return RTM_OK;
}

int collect_profile(rtm_ctx* c) {
    if (!c->profiling) return RTM_OK;
    for (long long k = 0; k < c->prof_launches; ++k) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->prof_ev[2 * k], c->prof_ev[2 * k + 1]));
        c->prof_ms += ms;
        c->prof_total_launches += c->prof_weight[k];
    }
    return RTM_OK;
}

int build_graph(rtm_ctx* c, Slab& s) {
    const int var = single_variant(c);
    if (s.graph_valid && s.graph_variant == var && s.graph_bank == s.bank) return RTM_OK;
    if (s.graph) cudaGraphExecDestroy(s.graph), s.graph = nullptr;
    if (s.graph_def) cudaGraphDestroy(s.graph_def), s.graph_def = nullptr;
    RET(ensure_tmaps(c, s, var));
    CK(cudaStreamBeginCapture(s.s_own, cudaStreamCaptureModeThreadLocal));
    const long long saved = c->launches;
    const bool prof = c->profiling;  // per-launch events stay outside the capture
    c->profiling = false;
    int rc = RTM_OK;
    for (int k = 0; k < 2 * GRAPH_PAIRS && rc == RTM_OK; ++k)
        rc = launch_stencil(c, s, k & 1, 0, s.nzl, 0, 0, 1, s.s_own);
    c->profiling = prof;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s.s_own, &g);
    c->launches = saved;
    if (rc != RTM_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return fail(RTM_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    s.graph_def = g;
    CK(cudaGraphInstantiate(&s.graph, g, 0));
    s.graph_valid = true;
    s.graph_variant = var;
    s.graph_bank = s.bank;
    return RTM_OK;
}

void invalidate_graphs(rtm_ctx* c) {
    for (auto& s : c->slabs) {
        s.graph_valid = false;
        for (int k = 0; k < 4; ++k) s.tb_graph_variant[k] = -1;
    }
}

// ---- two-step passes (kind 4, k_tb2s in rtm_tb.cu) ----------------------
// CUDA events around a launch when profiling (rtm_set_profiling)
int prof_begin(rtm_ctx* c, cudaStream_t st) {
    if (!c->profiling) return RTM_OK;
    const size_t k = 2 * (size_t)c->prof_launches;
    while (c->prof_ev.size() < k + 2) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->prof_ev.push_back(e);
    }
    CK(cudaEventRecord(c->prof_ev[k], st));
    return RTM_OK;
}
int prof_end(rtm_ctx* c, cudaStream_t st, int weight = 1) {
    if (!c->profiling) return RTM_OK;
    CK(cudaEventRecord(c->prof_ev[2 * (size_t)c->prof_launches + 1], st));
    if (c->prof_weight.size() <= (size_t)c->prof_launches) c->prof_weight.resize(c->prof_launches + 1);
    c->prof_weight[c->prof_launches] = weight;
    ++c->prof_launches;
    return RTM_OK;
}
struct TBBand {
    int ya_lo, ya_hi, yb_lo, yb_hi, tiles_y;
};

// y-bands of a single-slab single-shot grid for variant tv: each band's A region (its rows
// + 5 each side, clipped to the grid) must fit the CTA grid tiles_x x tiles_y <= #SMs (one
// resident CTA per SM).  Rows are split evenly over the fewest bands that fit.
bool tb_plan(const rtm_ctx* c, const TileVariant& tv, int* tiles_x, std::vector<TBBand>* bands) {
    if (c->mode != 0 || c->slabs.size() != 1 || c->slabs[0].nshots != 1) return false;
    const int tx = (c->nx + tv.TX - 1) / tv.TX;
    const int ctas = c->tb_ctas > 0 ? std::min(c->tb_ctas, c->num_sms) : c->num_sms;
    const int cap = ctas / tx;  // tile rows per band
    if (cap < 1) return false;
    const int R = cap * tv.TY;
    int nb = 1;
    if (R < c->ny) {
        if (R <= 10) return false;
        nb = (c->ny + (R - 10) - 1) / (R - 10);
    }
    bands->clear();
    for (int b = 0; b < nb; ++b) {
        TBBand t;
        t.yb_lo = (int)((long long)b * c->ny / nb);
        t.yb_hi = (int)((long long)(b + 1) * c->ny / nb);
        t.ya_lo = std::max(0, t.yb_lo - 5);
        t.ya_hi = std::min(c->ny, t.yb_hi + 5);
        t.tiles_y = (t.ya_hi - t.ya_lo + tv.TY - 1) / tv.TY;
        if (t.tiles_y > cap || t.yb_hi <= t.yb_lo) return false;
        bands->push_back(t);
    }
    *tiles_x = tx;
    return true;
}

bool tb_active(const rtm_ctx* c) {
    const int v = resolve_tile(c);
    if (variant(v).kind != 4) return false;
    int tx;
    std::vector<TBBand> b;
    return tb_plan(c, variant(v), &tx, &b);
}

int tb_alloc(rtm_ctx* c, Slab& s) {
    if (s.alt[0]) return RTM_OK;
    CK(cudaSetDevice(s.dev));
    const size_t nbuf = dplane(c) * s.buf_planes();
    for (int b = 0; b < 2; ++b) {
        if (cudaMalloc(&s.alt[b], nbuf * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            if (s.alt[0]) cudaFree(s.alt[0]), s.alt[0] = nullptr;
            return fail(RTM_ENOMEM, "cudaMalloc of %zu bytes (two-step bank %d) failed", nbuf * 4, b);
        }
        CK(cudaMemsetAsync(s.alt[b], 0, nbuf * sizeof(float), s.stream()));  // z-halo planes stay 0
    }
    CK(cudaMalloc(&s.d_flags, 2 * (size_t)c->num_sms * sizeof(unsigned long long)));
    CK(cudaMalloc(&s.d_epoch, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(s.d_flags, 0, 2 * (size_t)c->num_sms * sizeof(unsigned long long), s.stream()));
    CK(cudaMemsetAsync(s.d_epoch, 0, sizeof(unsigned long long), s.stream()));
    CK(cudaStreamSynchronize(s.stream()));
    return RTM_OK;
}

// One pass n -> n+2 (parity = n & 1): stage A reads u^n = buf[parity], u^{n-1} = buf[parity^1]
// and writes u^{n+1} to alt[parity^1]; stage B writes u^{n+2} to alt[parity]; then the banks
// swap so that u^{n+2} is buf[parity] again (u^m always lives in buf[m & 1]).
int tb_pass(rtm_ctx* c, Slab& s, int parity, cudaStream_t st) {
    const int var = resolve_tile(c);
    const TileVariant& tv = variant(var);
    int tiles_x;
    std::vector<TBBand> bands;
    if (!tb_plan(c, tv, &tiles_x, &bands)) return fail(RTM_EINVAL, "two-step plan does not fit");
    RET(tb_alloc(c, s));
    CUtensorMap tm[6];
    const int np = (int)s.buf_planes();
    RET(encode_3d(&tm[0], s.buf[parity], c, np, tv.TX + 16, tv.TY + 10));  // u^n box
    RET(encode_3d(&tm[1], s.buf[parity ^ 1], c, np, tv.TX, tv.TY));        // u^{n-1}
    RET(encode_3d(&tm[2], s.C, c, s.nzl, tv.TX, tv.TY));                   // C
    RET(encode_3d(&tm[3], s.alt[parity ^ 1], c, np, tv.TX + 16, tv.TY + 10));  // u^{n+1} box
    RET(encode_3d(&tm[4], s.buf[parity], c, np, tv.TX, tv.TY));            // u^n tile
    RET(encode_3d(&tm[5], s.alt[parity ^ 1], c, np, tv.TX, tv.TY));        // u^{n+1} store
    TB2SParams q;
    std::memset(&q, 0, sizeof q);
    q.nx = c->nx;
    q.ny = c->ny;
    q.nzl = s.nzl;
    q.pitch = c->px;
    q.plane = (long long)dplane(c);
    q.coef[0] = 3.0f * c->coeffs[0];
    for (int k = 1; k < 6; ++k) q.coef[k] = c->coeffs[k];
    q.outB = s.alt[parity];
    q.d_step = s.d_step;
    q.parity = parity;
    q.flagsA = s.d_flags;
    q.flagsB = s.d_flags + c->num_sms;
    q.d_epoch = s.d_epoch;
    q.nbands = (int)bands.size();
    if (s.tb_nbands != q.nbands) {
        // the flag epoch E = (epoch * nbands + band + 1) << 32 only grows while nbands is fixed:
        // a new plan (RTM_OPT_TB_CTAS, tile) starts from cleared flags so no stale value can
        // satisfy a >= wait of the new numbering
        CK(cudaMemsetAsync(s.d_flags, 0, 2 * (size_t)c->num_sms * sizeof(unsigned long long), st));
        s.tb_nbands = q.nbands;
    }
    q.tiles_x = tiles_x;
    q.nsrc = (int)s.srcs.size();
    for (int k = 0; k < q.nsrc; ++k) q.src[k] = s.srcs[k];
    q.samples = s.d_samples;
    for (size_t b = 0; b < bands.size(); ++b) {
        q.band = (int)b;
        q.tiles_y = bands[b].tiles_y;
        q.ntiles = tiles_x * bands[b].tiles_y;
        q.ya_lo = bands[b].ya_lo;
        q.ya_hi = bands[b].ya_hi;
        q.yb_lo = bands[b].yb_lo;
        q.yb_hi = bands[b].yb_hi;
        RET(prof_begin(c, st));
        CK(launch_tb2s(var, tm, q, st));
        RET(prof_end(c, st));
        ++c->launches;
    }
    CK(launch_tb_advance(s.d_step, parity, s.d_epoch, st));
    ++c->launches;
    std::swap(s.buf[0], s.alt[0]);
    std::swap(s.buf[1], s.alt[1]);
    s.bank ^= 1;
    s.tm_variant = -1;  // k_stream tensor maps follow the buffers
    return RTM_OK;
}

// A graph of 2*GRAPH_PAIRS passes (4*GRAPH_PAIRS steps): an even number of bank swaps, so it
// starts and ends on the same bank; one graph per (bank, parity) it starts from.
int tb_graph_launch(rtm_ctx* c, Slab& s, int parity, cudaStream_t st) {
    const int var = resolve_tile(c);
    const int key = s.bank * 2 + parity;
    if (s.tb_graph_variant[key] != var) {
        if (s.tb_graph[key]) cudaGraphExecDestroy(s.tb_graph[key]), s.tb_graph[key] = nullptr;
        RET(tb_alloc(c, s));
        CK(cudaStreamBeginCapture(s.s_own, cudaStreamCaptureModeThreadLocal));
        const long long saved = c->launches;
        int rc = RTM_OK;
        for (int k = 0; k < 2 * GRAPH_PAIRS && rc == RTM_OK; ++k) rc = tb_pass(c, s, parity, s.s_own);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(s.s_own, &g);
        c->launches = saved;
        if (rc != RTM_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return fail(RTM_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
        cudaError_t ei = cudaGraphInstantiate(&s.tb_graph[key], g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) return fail(RTM_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ei));
        s.tb_graph_variant[key] = var;
    }
    CK(cudaGraphLaunch(s.tb_graph[key], st));
    return RTM_OK;
}

int upload_sources(rtm_ctx* c, Slab& s) {
    CK(cudaSetDevice(s.dev));
    if (s.d_samples) {
        CK(cudaStreamSynchronize(s.stream()));
        CK(cudaFree(s.d_samples));
        s.d_samples = nullptr;
    }
    if (!s.h_samples.empty()) {
        CK(cudaMalloc(&s.d_samples, s.h_samples.size() * sizeof(float)));
        CK(cudaMemcpy(s.d_samples, s.h_samples.data(), s.h_samples.size() * sizeof(float),
                      cudaMemcpyHostToDevice));
    }
    invalidate_graphs(c);
    return RTM_OK;
}

// Resident multi-step launches (kind 5): the whole run in cooperative launches of up to 4096
// steps, one grid barrier per step inside.
int step_resident(rtm_ctx* c, int nsteps) {
    Slab& s = c->slabs[0];
    cudaStream_t st = s.stream();
    const TileVariant& tv = variant(resolve_tile(c));
    int occ = variant_occupancy(resolve_tile(c), nullptr);
    if (occ < 1) return fail(RTM_ECUDA, "variant %s cannot be resident", tv.name);
    const int ctas = c->num_sms * std::min(occ, tv.MINB);
    if (!s.d_bar) CK(cudaMalloc(&s.d_bar, 2 * sizeof(unsigned)));
    ResParams p;
    std::memset(&p, 0, sizeof p);
    p.nx = c->nx;
    p.ny = c->ny;
    p.nzl = s.nzl;
    p.pitch = c->px;
    p.nshots = s.nshots;
    p.plane = (long long)dplane(c);
    p.coef[0] = 3.0f * c->coeffs[0];
    for (int k = 1; k < 6; ++k) p.coef[k] = c->coeffs[k];
    p.buf0 = s.buf[0];
    p.buf1 = s.buf[1];
    p.C = s.C;
    p.d_step = s.d_step;
    p.bar = s.d_bar;
    p.nsrc = (int)s.srcs.size();
    for (int k = 0; k < p.nsrc; ++k) p.src[k] = s.srcs[k];
    p.samples = s.d_samples;
    for (int k = 0; k < nsteps;) {
        p.parity0 = (int)(c->step & 1);
        p.nsteps = std::min(nsteps - k, 4096);
        RET(prof_begin(c, st));
        CK(launch_resident(p, ctas, tv.TX, st));
        RET(prof_end(c, st));
        ++c->launches;
        c->step += p.nsteps;
        k += p.nsteps;
    }
    return RTM_OK;
}

// Multi-step launches (kind 6): up to kMaxMsSteps time steps per cooperative launch of
// k_stream<..., MS = true>; work units start a step once they and their face-neighbour units
// have published the previous one (flags), instead of at a launch boundary.
constexpr int kMaxMsSteps = 1 << 20;
int step_mstep(rtm_ctx* c, int nsteps) {
    Slab& s = c->slabs[0];
    cudaStream_t st = s.stream();
    const int var = resolve_tile(c);
    const TileVariant& tv = variant(var);
    RET(ensure_tmaps(c, s, var));
    for (int k = 0; k < nsteps;) {
        const int parity = (int)(c->step & 1);
        StencilParams p;
        fill_params(c, s, parity, p);
        p.nranges = 1;
        p.r_begin[0] = 0;
        p.r_len[0] = s.nzl;
        p.tiles_x = (c->nx + tv.TX - 1) / tv.TX;
        p.tiles_y = (c->ny + tv.TY - 1) / tv.TY;
        p.r_chunks[0] = choose_chunks(c, s.occupancy, p.tiles_x * p.tiles_y * s.nshots, s.nzl);
        const long long units = (long long)p.tiles_x * p.tiles_y * p.r_chunks[0] * s.nshots;
        if (units > s.ms_units) {
            if (s.d_msflags) {
                CK(cudaStreamSynchronize(st));
                CK(cudaFree(s.d_msflags));
                s.d_msflags = nullptr;
            }
            CK(cudaMalloc(&s.d_msflags, units * sizeof(unsigned long long)));
            CK(cudaMemsetAsync(s.d_msflags, 0, units * sizeof(unsigned long long), st));
            s.ms_units = units;
        }
        p.flags = s.d_msflags;
        p.epoch = (++s.ms_epoch) << 32;  // flags of earlier launches are always smaller
        p.nsteps = std::min(nsteps - k, kMaxMsSteps);
        p.step0 = (int)c->step;
        RET(prof_begin(c, st));
        CK(launch_mstep(var, &s.tm_u[parity], &s.tm_in[parity ^ 1], &s.tm_u[parity ^ 1], &s.tm_in[parity],
                        &s.tm_c, p, c->num_sms * s.occupancy, st));
        RET(prof_end(c, st));
        ++c->launches;
        c->step += p.nsteps;
        k += p.nsteps;
    }
    return RTM_OK;
}

int step_single(rtm_ctx* c, int nsteps) {
    Slab& s = c->slabs[0];
    cudaStream_t st = s.stream();
    if (variant(resolve_tile(c)).kind == 5) return step_resident(c, nsteps);
    if (variant(resolve_tile(c)).kind == 6) return step_mstep(c, nsteps);
    int k = 0;
    int tb_bands = 0;
    if (variant(resolve_tile(c)).kind == 4) {
        int tx;
        std::vector<TBBand> b;
        if (tb_plan(c, variant(resolve_tile(c)), &tx, &b)) tb_bands = (int)b.size();
    }
    const bool tb = tb_bands > 0;
    while (k < nsteps) {
        const int parity = (int)(c->step & 1);
        if (tb && nsteps - k >= 2) {  // two time steps per pass
            const int passes = c->graphs && !c->profiling && nsteps - k >= 4 * GRAPH_PAIRS ? 2 * GRAPH_PAIRS : 1;
            if (passes > 1) {
                RET(tb_graph_launch(c, s, parity, st));
                c->launches += (long long)passes * (tb_bands + 1);  // + d_step/epoch advance
            } else {
                RET(tb_pass(c, s, parity, st));
            }
            c->step += 2 * passes;
            k += 2 * passes;
            continue;
        }
        if (c->graphs && parity == 0 && nsteps - k >= 2 * GRAPH_PAIRS) {
            // profiling: one event pair around the replay (16 launches, back to back on the
            // device), so short launches are timed without breaking the graph
            RET(build_graph(c, s));
            RET(prof_begin(c, st));
            CK(cudaGraphLaunch(s.graph, st));
            RET(prof_end(c, st, 2 * GRAPH_PAIRS));
            c->step += 2 * GRAPH_PAIRS;
            c->launches += 2 * GRAPH_PAIRS;
            k += 2 * GRAPH_PAIRS;
            continue;
        }
        RET(launch_stencil(c, s, parity, 0, s.nzl, 0, 0, 1, st));
        ++c->step;
        ++k;
    }
    return RTM_OK;
}

int exchange_local(rtm_ctx* c, int parity_next) {
    const int G = (int)c->slabs.size();
    const size_t plane = dplane(c);
    const size_t bytes = 5 * plane * sizeof(float);
    for (int r = 0; r < G; ++r) {
        Slab& s = c->slabs[r];
        CK(cudaSetDevice(s.dev));
        for (int d = -1; d <= 1; ++d)
            if (r + d >= 0 && r + d < G) CK(cudaStreamWaitEvent(s.s_comm, c->slabs[r + d].ev_bnd, 0));
        float* dst = s.buf[parity_next];
        if (s.lo_nb) {
            const Slab& n = c->slabs[r - 1];
            CK(cudaMemcpyAsync(dst, n.buf[parity_next] + (size_t)n.nzl * plane, bytes,
                               cudaMemcpyDefault, s.s_comm));  // peer copy through UVA (capturable)
        }
        if (s.hi_nb) {
            const Slab& n = c->slabs[r + 1];
            CK(cudaMemcpyAsync(dst + (size_t)(s.nzl + 5) * plane, n.buf[parity_next] + 5 * plane,
                               bytes, cudaMemcpyDefault, s.s_comm));
        }
        CK(cudaEventRecord(s.ev_comm, s.s_comm));
    }
    return RTM_OK;
}

int exchange_nccl(rtm_ctx* c, int parity_next) {
    Slab& s = c->slabs[0];
    const size_t plane = dplane(c);
    const size_t cnt = 5 * plane;
    CK(cudaStreamWaitEvent(s.s_comm, s.ev_bnd, 0));
    float* b = s.buf[parity_next];
    NK(ncclGroupStart());
    if (s.lo_nb) {
        NK(ncclSend(b + 5 * plane, cnt, ncclFloat32, c->rank - 1, c->comm, s.s_comm));
        NK(ncclRecv(b, cnt, ncclFloat32, c->rank - 1, c->comm, s.s_comm));
    }
    if (s.hi_nb) {
        NK(ncclSend(b + (size_t)s.nzl * plane, cnt, ncclFloat32, c->rank + 1, c->comm, s.s_comm));
        NK(ncclRecv(b + (size_t)(s.nzl + 5) * plane, cnt, ncclFloat32, c->rank + 1, c->comm,
                    s.s_comm));
    }
    NK(ncclGroupEnd());
    CK(cudaEventRecord(s.ev_comm, s.s_comm));
    return RTM_OK;
}

// ---- rank synchronisation -------------------------------------------------------------
// Barrier across the ranks of a distributed context: the NCCL communicator (all-reduce of one
// value, then a stream synchronisation) or, for a peer context, the caller's host barrier.
// In-process and single contexts have nothing to wait for.  On return every rank reached it.
int ranks_barrier(rtm_ctx* c) {
    if (c->comm) {
        Slab& s = c->slabs[0];
        CK(cudaSetDevice(s.dev));
        double* d = nullptr;
        CK(cudaMalloc(&d, sizeof(double)));
        const ncclResult_t nr = ncclAllReduce(d, d, 1, ncclFloat64, ncclSum, c->comm, s.stream());
        const cudaError_t e = cudaStreamSynchronize(s.stream());
        cudaFree(d);
        if (nr != ncclSuccess || e != cudaSuccess) return fail(RTM_ENCCL, "rank barrier failed");
        return RTM_OK;
    }
    if (c->mode == 3 && c->world > 1) {
        if (!c->barrier_fn)
            return fail(RTM_ESTATE, "peer context: this call is collective and needs rtm_set_host_barrier");
        if (c->barrier_fn(c->barrier_user) != 0) return fail(RTM_ESTATE, "the host barrier callback failed");
    }
    return RTM_OK;
}

// ---- CUDA-IPC records (peer contexts; NCCL-distributed contexts in halo modes 2-3) -------
// Every rank exports IPC handles of its two time-level buffers and its flag words; a
// neighbour opens them (cudaIpcMemLazyEnablePeerAccess: NVLink peer mappings between GPUs,
// plain mappings when the ranks share a device).
constexpr unsigned kIpcMagic = 0x52544d31u;  // "RTM1"
struct IpcRecord {
    unsigned magic;
    int version;
    int rank, world;
    int nx, ny, nz, nzl;
    int device;
    int pad0[7];
    cudaIpcMemHandle_t buf[2];
    cudaIpcMemHandle_t sig;
    unsigned char pad1[RTM_IPC_RECORD_BYTES - 64 - 3 * sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(IpcRecord) == RTM_IPC_RECORD_BYTES, "IPC record size");

int alloc_sig(Slab& s) {
    CK(cudaSetDevice(s.dev));
    if (!s.d_sig) {
        CK(cudaMalloc(&s.d_sig, 4 * sizeof(unsigned long long)));
        CK(cudaMemset(s.d_sig, 0, 4 * sizeof(unsigned long long)));
    }
    return RTM_OK;
}

int export_record(rtm_ctx* c, IpcRecord* r) {
    Slab& s = c->slabs[0];
    RET(alloc_sig(s));
    std::memset(r, 0, sizeof *r);
    r->magic = kIpcMagic;
    r->version = 1;
    r->rank = c->rank;
    r->world = c->world;
    r->nx = c->nx;
    r->ny = c->ny;
    r->nz = c->nz;
    r->nzl = s.nzl;
    r->device = s.dev;
    for (int b = 0; b < 2; ++b) CK(cudaIpcGetMemHandle(&r->buf[b], s.buf[b]));
    CK(cudaIpcGetMemHandle(&r->sig, s.d_sig));
    return RTM_OK;
}

int import_records(rtm_ctx* c, const IpcRecord* lo, const IpcRecord* hi) {
    Slab& s = c->slabs[0];
    if (c->ipc_imported) return fail(RTM_ESTATE, "the neighbours' IPC records are already imported");
    if (s.lo_nb != (lo != nullptr) || s.hi_nb != (hi != nullptr))
        return fail(RTM_EINVAL, "rank %d of %d needs %s lo record and %s hi record", c->rank, c->world,
                    s.lo_nb ? "a" : "no", s.hi_nb ? "a" : "no");
    for (int side = 0; side < 2; ++side) {
        const IpcRecord* r = side == 0 ? lo : hi;
        if (!r) continue;
        const int want = c->rank + (side == 0 ? -1 : 1);
        int z0, nzl;
        if (r->magic != kIpcMagic || r->version != 1)
            return fail(RTM_EINVAL, "%s record: not an RTM IPC record", side ? "hi" : "lo");
        if (r->nx != c->nx || r->ny != c->ny || r->nz != c->nz || r->world != c->world || r->rank != want)
            return fail(RTM_EINVAL, "%s record belongs to rank %d of %d on a %dx%dx%d grid (want rank %d of %d, %dx%dx%d)",
                        side ? "hi" : "lo", r->rank, r->world, r->nx, r->ny, r->nz, want, c->world, c->nx, c->ny, c->nz);
        RET(rtm_slab_range(c->nz, c->world, want, &z0, &nzl));
        if (r->nzl != nzl) return fail(RTM_EINVAL, "%s record: nzl %d != %d", side ? "hi" : "lo", r->nzl, nzl);
    }
    CK(cudaSetDevice(s.dev));
    RET(alloc_sig(s));
    auto open = [&](const cudaIpcMemHandle_t& hd, void** out) -> int {
        const cudaError_t e = cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(RTM_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
        s.ipc_open.push_back(*out);
        return RTM_OK;
    };
    void* q;
    if (lo) {
        for (int b = 0; b < 2; ++b) {
            RET(open(lo->buf[b], &q));
            s.nb_lo[b] = static_cast<float*>(q);
        }
        RET(open(lo->sig, &q));
        s.nb_lo_sig = static_cast<unsigned long long*>(q);
        s.nb_lo_nzl = lo->nzl;
    }
    if (hi) {
        for (int b = 0; b < 2; ++b) {
            RET(open(hi->buf[b], &q));
            s.nb_hi[b] = static_cast<float*>(q);
        }
        RET(open(hi->sig, &q));
        s.nb_hi_sig = static_cast<unsigned long long*>(q);
    }
    // the neighbours' buffers follow the local time-level convention (u^n in buf[n & 1]): if a
    // rtm_set_step_count swapped this rank's buffers, every rank swapped alike
    c->ipc_imported = true;
    return RTM_OK;
}

// Halo modes 2-3 set-up: flag words per slab, neighbours' buffer / flag pointers.  In-process
// (mode 1) they are the other slabs' allocations; an NCCL-distributed context all-gathers the
// IPC records over its communicator (a collective call); a peer context already imported them.
// Ends with a rank barrier: no rank may signal into a neighbour's flag words before the
// neighbour has cleared them.
int setup_signal(rtm_ctx* c) {
    static PFN_devattr devattr = driver_fn<PFN_devattr>("cuDeviceGetAttribute");
    if (!devattr) return fail(RTM_ECUDA, "cuDeviceGetAttribute unavailable from the driver");
    unsigned flush = CU_STREAM_WAIT_VALUE_FLUSH;
    for (auto& s : c->slabs) {
        int mem64 = 0, fl = 0;
        devattr(&mem64, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, (CUdevice)s.dev);
        devattr(&fl, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, (CUdevice)s.dev);
        if (!mem64) return fail(RTM_EINVAL, "device %d has no 64-bit stream memory operations", s.dev);
        if (!fl) flush = 0;
        RET(alloc_sig(s));
        CK(cudaMemset(s.d_sig, 0, 4 * sizeof(unsigned long long)));
    }
    c->sig_flush = flush;
    const int G = (int)c->slabs.size();
    if (c->mode == 1) {
        for (int r = 0; r < G; ++r) {
            Slab& s = c->slabs[r];
            if (s.lo_nb) {
                const Slab& n = c->slabs[r - 1];
                s.nb_lo[0] = n.buf[0], s.nb_lo[1] = n.buf[1], s.nb_lo_nzl = n.nzl, s.nb_lo_sig = n.d_sig;
            }
            if (s.hi_nb) {
                const Slab& n = c->slabs[r + 1];
                s.nb_hi[0] = n.buf[0], s.nb_hi[1] = n.buf[1], s.nb_hi_sig = n.d_sig;
            }
        }
    } else if (c->mode == 2 && !c->ipc_imported) {
        Slab& s = c->slabs[0];
        CK(cudaSetDevice(s.dev));
        IpcRecord mine;
        RET(export_record(c, &mine));
        const int W = c->world;
        unsigned char* d = nullptr;
        CK(cudaMalloc(&d, (size_t)W * sizeof(IpcRecord)));
        std::vector<IpcRecord> all(W);
        int rc = RTM_OK;
        if (cudaMemcpy(d + (size_t)c->rank * sizeof(IpcRecord), &mine, sizeof mine,
                       cudaMemcpyHostToDevice) != cudaSuccess)
            rc = fail(RTM_ECUDA, "IPC record upload failed");
        if (rc == RTM_OK) {
            const ncclResult_t nr = ncclAllGather(d + (size_t)c->rank * sizeof(IpcRecord), d,
                                                  sizeof(IpcRecord), ncclUint8, c->comm, s.stream());
            if (nr != ncclSuccess) rc = fail(RTM_ENCCL, "ncclAllGather of IPC handles: %s", ncclGetErrorString(nr));
        }
        if (rc == RTM_OK && (cudaStreamSynchronize(s.stream()) != cudaSuccess ||
                             cudaMemcpy(all.data(), d, (size_t)W * sizeof(IpcRecord),
                                        cudaMemcpyDeviceToHost) != cudaSuccess))
            rc = fail(RTM_ECUDA, "IPC record gather failed");
        cudaFree(d);
        RET(rc);
        RET(import_records(c, s.lo_nb ? &all[c->rank - 1] : nullptr, s.hi_nb ? &all[c->rank + 1] : nullptr));
    } else if (c->mode == 3 && c->world > 1 && !c->ipc_imported) {
        return fail(RTM_ESTATE, "peer context: rtm_ipc_import the neighbours' records first");
    }
    RET(ranks_barrier(c));
    ++c->sig_gen;
    c->sig_fresh = true;
    return RTM_OK;
}

typedef CUresult (*PFN_waitv64_t)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
PFN_waitv64_t waitv64() {
    static PFN_waitv64_t f = driver_fn<PFN_waitv64_t>("cuStreamWaitValue64");
    return f;
}
// Stream-side wait (no spinning kernel) until *flag >= v.
int wait_flag(rtm_ctx* c, cudaStream_t st, unsigned long long* flag, unsigned long long v) {
    auto f = waitv64();
    if (!f) return fail(RTM_ECUDA, "cuStreamWaitValue64 unavailable from the driver");
    const CUresult r = f((CUstream)st, (CUdeviceptr)flag, v, CU_STREAM_WAIT_VALUE_GEQ | c->sig_flush);
    if (r != CUDA_SUCCESS) return fail(RTM_ECUDA, "cuStreamWaitValue64 failed (%d)", (int)r);
    return RTM_OK;
}

// RTM_OPT_HOST_ORDERED: drain this context's streams, then meet every rank at the barrier —
// after it, every flag a wait enqueued next targets has already been released.
int host_order_point(rtm_ctx* c) {
    if (!c->host_ordered) return RTM_OK;
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.stream()));
        CK(cudaStreamSynchronize(s.s_comm));
    }
    return ranks_barrier(c);
}

// G > 1 step, fused halo push + flag protocol (f1, halo mode 2; across processes through the
// IPC mappings): step n on slab r waits (stream-side cuStreamWaitValue64, no spinning kernel)
// until both neighbours have completed step n-1 — their pushes into r's halo have landed (RAW)
// and their step n-1 reads of the halo planes r now overwrites are done (WAR) — then one stencil
// launch whose epilogue also stores r's boundary planes into the neighbours' halos (peer / IPC
// stores over NVLink), then k_signal releases "steps done = n+1" into the neighbours' flags.
// Values carry a generation (bumped by every synchronising reset), so stale flags never pass.
int step_slabs_signal(rtm_ctx* c, int nsteps) {
    const size_t plane = dplane(c);
    const unsigned long long g = c->sig_gen << 40;
    for (int k = 0; k < nsteps; ++k) {
        const int parity = (int)(c->step & 1);
        const unsigned long long n = (unsigned long long)c->step;
        RET(host_order_point(c));
        for (auto& s : c->slabs) {
            CK(cudaSetDevice(s.dev));
            cudaStream_t st = s.stream();
            if (!c->sig_fresh) {
                if (s.lo_nb) RET(wait_flag(c, st, s.d_sig + 0, g | n));
                if (s.hi_nb) RET(wait_flag(c, st, s.d_sig + 1, g | n));
            }
            float* lo = s.lo_nb ? s.nb_lo[parity ^ 1] + (size_t)(s.nb_lo_nzl + 5) * plane : nullptr;
            float* hi = s.hi_nb ? s.nb_hi[parity ^ 1] : nullptr;
            RET(launch_stencil(c, s, parity, 0, s.nzl, 0, 0, 1, st, lo, hi));
            CK(launch_signal(s.lo_nb ? s.nb_lo_sig + 1 : nullptr, s.hi_nb ? s.nb_hi_sig : nullptr,
                             g | (n + 1), st));
        }
        c->sig_fresh = false;
        ++c->step;
    }
    return RTM_OK;
}

// G > 1 step, copy-engine pull + flag protocol (halo mode 3; SURVEY §8(e) "SM-free
// alternative"; in-process or across processes through the IPC mappings).  Step n on slab r:
//   stream:  boundary planes [0,5) + [nzl-5,nzl) of u^{n+1} (after r's own pulls of step n-1:
//            stream order), then k_signal B := g|(n+1) into the neighbours ("boundary of step
//            n ready");
//   comm:    after the boundary (event), wait B_lo, B_hi >= g|(n+1) [RAW], then cudaMemcpyAsync
//            the neighbours' 5 boundary planes of u^{n+1} into r's own halo planes (copy engines
//            reading the peer / IPC mapping; no SM time, no NCCL kernels);
//   stream:  interior planes [5, nzl-5) (overlapping the pulls), then wait for the pulls (event).
// Every rank writes only its own memory.  The WAR hazard — r's boundary of step n overwrites the
// u^{n-1} planes a neighbour pulled at its step n-2 — needs no flag of its own: r's boundary n
// follows r's pulls of n-1, which waited for the neighbour's boundary n-1, which followed the
// neighbour's pulls of n-2 (model-checked in tests/test_halo_protocol_model.py).
int step_slabs_pull(rtm_ctx* c, int nsteps) {
    const size_t plane = dplane(c);
    const size_t bytes = 5 * plane * sizeof(float);
    const unsigned long long g = c->sig_gen << 40;
    for (int k = 0; k < nsteps; ++k) {
        const int parity = (int)(c->step & 1);
        const unsigned long long n = (unsigned long long)c->step;
        for (auto& s : c->slabs) {
            CK(cudaSetDevice(s.dev));
            cudaStream_t st = s.stream();
            if (s.lo_nb || s.hi_nb) {
                const int b0 = s.lo_nb ? 0 : s.nzl - 5;
                const int b1 = s.nzl - 5, l1 = (s.lo_nb && s.hi_nb) ? 5 : 0;
                RET(launch_stencil(c, s, parity, b0, 5, b1, l1, 0, st));
                CK(launch_signal(s.lo_nb ? s.nb_lo_sig + 3 : nullptr, s.hi_nb ? s.nb_hi_sig + 2 : nullptr,
                                 g | (n + 1), st));
            }
            CK(cudaEventRecord(s.ev_bnd, st));
        }
        RET(host_order_point(c));
        for (auto& s : c->slabs) {
            CK(cudaSetDevice(s.dev));
            cudaStream_t st = s.stream();
            float* dst = s.buf[parity ^ 1];
            if (s.lo_nb || s.hi_nb) {
                CK(cudaStreamWaitEvent(s.s_comm, s.ev_bnd, 0));
                if (s.lo_nb) {
                    RET(wait_flag(c, s.s_comm, s.d_sig + 2, g | (n + 1)));
                    CK(cudaMemcpyAsync(dst, s.nb_lo[parity ^ 1] + (size_t)s.nb_lo_nzl * plane, bytes,
                                       cudaMemcpyDefault, s.s_comm));
                }
                if (s.hi_nb) {
                    RET(wait_flag(c, s.s_comm, s.d_sig + 3, g | (n + 1)));
                    CK(cudaMemcpyAsync(dst + (size_t)(s.nzl + 5) * plane, s.nb_hi[parity ^ 1] + 5 * plane,
                                       bytes, cudaMemcpyDefault, s.s_comm));
                }
                CK(cudaEventRecord(s.ev_comm, s.s_comm));
            }
            const int ib = s.lo_nb ? 5 : 0;
            const int ie = s.hi_nb ? s.nzl - 5 : s.nzl;
            RET(launch_stencil(c, s, parity, ib, ie - ib, 0, 0, 1, st));
            if (s.lo_nb || s.hi_nb) CK(cudaStreamWaitEvent(st, s.ev_comm, 0));
        }
        c->sig_fresh = false;
        ++c->step;
    }
    return RTM_OK;
}

// Halo fill of u^{parity} from the neighbours' owned planes through the peer / IPC mappings
// (peer contexts' rtm_reset / rtm_set_fields; synchronous, after a rank barrier).
int pull_halos_now(rtm_ctx* c, int parity) {
    const size_t plane = dplane(c);
    const size_t bytes = 5 * plane * sizeof(float);
    RET(ranks_barrier(c));  // every rank's initial data is in place
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        float* dst = s.buf[parity];
        if (s.lo_nb)
            CK(cudaMemcpyAsync(dst, s.nb_lo[parity] + (size_t)s.nb_lo_nzl * plane, bytes, cudaMemcpyDefault, s.s_comm));
        if (s.hi_nb)
            CK(cudaMemcpyAsync(dst + (size_t)(s.nzl + 5) * plane, s.nb_hi[parity] + 5 * plane, bytes,
                               cudaMemcpyDefault, s.s_comm));
        CK(cudaStreamSynchronize(s.s_comm));
    }
    return RTM_OK;
}

// One G > 1 step with boundary planes first, the exchange on the comm streams (NCCL or
// in-process copy engines), interior concurrently (halo mode 0).
int enqueue_slab_step0(rtm_ctx* c) {
    const int G = (int)c->slabs.size();
    const int parity = (int)(c->step & 1);
    for (int r = 0; r < G; ++r) {
        Slab& s = c->slabs[r];
        CK(cudaSetDevice(s.dev));
        for (int d = -1; d <= 1; ++d)  // previous exchange done (reads and writes)
            if (r + d >= 0 && r + d < G) CK(cudaStreamWaitEvent(s.stream(), c->slabs[r + d].ev_comm, 0));
        if (s.lo_nb || s.hi_nb) {
            const int b0 = s.lo_nb ? 0 : s.nzl - 5;
            const int l0 = 5;
            const int b1 = s.nzl - 5, l1 = (s.lo_nb && s.hi_nb) ? 5 : 0;
            RET(launch_stencil(c, s, parity, b0, l0, b1, l1, 0, s.stream()));
        }
        CK(cudaEventRecord(s.ev_bnd, s.stream()));
    }
    if (c->mode == 2) RET(exchange_nccl(c, parity ^ 1));
    else RET(exchange_local(c, parity ^ 1));
    for (int r = 0; r < G; ++r) {
        Slab& s = c->slabs[r];
        CK(cudaSetDevice(s.dev));
        const int ib = s.lo_nb ? 5 : 0;
        const int ie = s.hi_nb ? s.nzl - 5 : s.nzl;
        RET(launch_stencil(c, s, parity, ib, ie - ib, 0, 0, 1, s.stream()));
    }
    ++c->step;
    return RTM_OK;
}

// One G > 1 step of the event-ordered fused push (in-process halo mode 1): one launch per
// slab whose epilogue also stores the boundary planes into the neighbours' z-halo.  Step n on
// slab r waits for step n-1 of r-1, r, r+1: their pushes into r's halo (RAW) and their reads of
// the halo planes r is about to overwrite (WAR).
int enqueue_slab_step1(rtm_ctx* c) {
    const int G = (int)c->slabs.size();
    const size_t plane = dplane(c);
    const int parity = (int)(c->step & 1);
    for (int r = 0; r < G; ++r) {
        Slab& s = c->slabs[r];
        CK(cudaSetDevice(s.dev));
        for (int d = -1; d <= 1; d += 2)
            if (r + d >= 0 && r + d < G) CK(cudaStreamWaitEvent(s.stream(), c->slabs[r + d].ev_done, 0));
    }
    for (int r = 0; r < G; ++r) {
        Slab& s = c->slabs[r];
        CK(cudaSetDevice(s.dev));
        float* lo = s.lo_nb ? c->slabs[r - 1].buf[parity ^ 1] + (size_t)(c->slabs[r - 1].nzl + 5) * plane
                            : nullptr;
        float* hi = s.hi_nb ? c->slabs[r + 1].buf[parity ^ 1] : nullptr;
        RET(launch_stencil(c, s, parity, 0, s.nzl, 0, 0, 1, s.stream(), lo, hi));
        CK(cudaEventRecord(s.ev_done, s.stream()));
    }
    ++c->step;
    return RTM_OK;
}

// Join: every slab's stream waits for its neighbours' last exchange / push events, so the
// field is complete when rtm_step's final synchronisation returns.
int join_slabs(rtm_ctx* c) {
    const int G = (int)c->slabs.size();
    for (int r = 0; r < G; ++r) {
        Slab& s = c->slabs[r];
        CK(cudaSetDevice(s.dev));
        for (int d = -1; d <= 1; ++d)
            if (r + d >= 0 && r + d < G) {
                CK(cudaStreamWaitEvent(s.stream(), c->slabs[r + d].ev_comm, 0));
                CK(cudaStreamWaitEvent(s.stream(), c->slabs[r + d].ev_done, 0));
            }
    }
    return RTM_OK;
}

// CUDA graph of 2*GRAPH_PAIRS event-ordered slab steps (halo modes 0 and 1, in-process or NCCL):
// captured from slab 0's stream, the other slabs' streams (and comm streams) join the capture
// through an event and are joined back at the end, so one cudaGraphLaunch replays every
// slab's launches, copies / NCCL calls and event edges.  Starts at an even step (parity 0);
// every captured parameter (buffers, ranges, step-counter slots) repeats with period 2.
int build_slab_graph(rtm_ctx* c) {
    Slab& s0 = c->slabs[0];
    const int var = single_variant(c);
    if (s0.graph_valid && s0.graph_variant == var) return RTM_OK;
    if (s0.graph) cudaGraphExecDestroy(s0.graph), s0.graph = nullptr;
    if (s0.graph_def) cudaGraphDestroy(s0.graph_def), s0.graph_def = nullptr;
    for (auto& s : c->slabs) RET(ensure_tmaps(c, s, var));
    CK(cudaSetDevice(s0.dev));
    cudaStream_t origin = s0.stream();
    CK(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed));
    const long long saved_step = c->step, saved_launches = c->launches;
    int rc = RTM_OK;
    cudaEvent_t fork = nullptr;
    if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) rc = fail(RTM_ECUDA, "event");
    if (rc == RTM_OK && cudaEventRecord(fork, origin) != cudaSuccess) rc = fail(RTM_ECUDA, "fork record");
    for (auto& s : c->slabs) {  // every stream of the step joins the capture
        if (rc != RTM_OK) break;
        cudaSetDevice(s.dev);
        if ((&s != &s0 && cudaStreamWaitEvent(s.stream(), fork, 0) != cudaSuccess) ||
            cudaStreamWaitEvent(s.s_comm, fork, 0) != cudaSuccess)
            rc = fail(RTM_ECUDA, "capture fork failed");
        // the events of the previous step are outside the capture: re-record them inside
        if (rc == RTM_OK && (cudaEventRecord(s.ev_comm, s.s_comm) != cudaSuccess ||
                             cudaEventRecord(s.ev_done, s.stream()) != cudaSuccess))
            rc = fail(RTM_ECUDA, "capture event re-record failed");
    }
    c->step = 0;
    for (int k = 0; k < 2 * GRAPH_PAIRS && rc == RTM_OK; ++k)
        rc = c->halo_mode == 1 ? enqueue_slab_step1(c) : enqueue_slab_step0(c);
    if (rc == RTM_OK) rc = join_slabs(c);
    for (auto& s : c->slabs) {  // join every stream back into the origin
        if (rc != RTM_OK) break;
        cudaSetDevice(s.dev);
        if (cudaEventRecord(s.ev_bnd, s.s_comm) != cudaSuccess) rc = fail(RTM_ECUDA, "join record");
        cudaSetDevice(s0.dev);
        if (rc == RTM_OK && cudaStreamWaitEvent(origin, s.ev_bnd, 0) != cudaSuccess) rc = fail(RTM_ECUDA, "join");
        if (&s != &s0 && rc == RTM_OK) {
            cudaSetDevice(s.dev);
            if (cudaEventRecord(s.ev_bnd, s.stream()) != cudaSuccess) rc = fail(RTM_ECUDA, "join record");
            cudaSetDevice(s0.dev);
            if (rc == RTM_OK && cudaStreamWaitEvent(origin, s.ev_bnd, 0) != cudaSuccess) rc = fail(RTM_ECUDA, "join");
        }
    }
    cudaSetDevice(s0.dev);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(origin, &g);
    c->step = saved_step;
    c->launches = saved_launches;
    if (fork) cudaEventDestroy(fork);
    if (rc == RTM_OK && e != cudaSuccess) rc = fail(RTM_ECUDA, "slab graph capture failed: %s", cudaGetErrorString(e));
    if (rc != RTM_OK) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return rc;
    }
    s0.graph_def = g;
    if (cudaGraphInstantiate(&s0.graph, g, 0) != cudaSuccess) {
        cudaGetLastError();
        return fail(RTM_ECUDA, "slab graph instantiate failed");
    }
    s0.graph_valid = true;
    s0.graph_variant = var;
    return RTM_OK;
}

// G > 1 steps (halo modes 0-3).
int step_slabs(rtm_ctx* c, int nsteps) {
    if (c->halo_mode == 2) return step_slabs_signal(c, nsteps);
    if (c->halo_mode == 3) return step_slabs_pull(c, nsteps);
    long long launches_per_step = 0;
    for (auto& s : c->slabs) launches_per_step += (c->halo_mode == 0 && (s.lo_nb || s.hi_nb)) ? 2 : 1;
    int k = 0;
    while (k < nsteps) {
        const bool even = (c->step & 1) == 0;
        // In-process slabs only: capturing NCCL send/recv (distributed contexts) is supported by
        // NCCL but has never run on more than one GPU here, so those steps stay direct.
        if (c->graphs && c->mode == 1 && !c->profiling && !c->slab_graphs_broken && even &&
            nsteps - k >= 2 * GRAPH_PAIRS) {
            if (build_slab_graph(c) != RTM_OK) {
                // e.g. a capture the driver refuses: direct launches from now on.  Events last
                // recorded inside the aborted capture cannot be waited on: re-record them.
                if (std::getenv("RTM_DEBUG")) std::fprintf(stderr, "rtm: slab graph capture failed: %s\n", g_err.c_str());
                c->slab_graphs_broken = true;
                g_err.clear();
                cudaGetLastError();
                for (auto& s : c->slabs) {
                    CK(cudaSetDevice(s.dev));
                    CK(cudaEventRecord(s.ev_comm, s.s_comm));
                    CK(cudaEventRecord(s.ev_done, s.stream()));
                    CK(cudaEventRecord(s.ev_bnd, s.stream()));
                }
                continue;
            }
            Slab& s0 = c->slabs[0];
            // the graph runs on slab 0's stream: it starts after every stream's pending work
            // and every stream's later work starts after it
            for (auto& s : c->slabs) {
                CK(cudaSetDevice(s.dev));
                CK(cudaEventRecord(s.ev_bnd, s.s_comm));
                CK(cudaSetDevice(s0.dev));
                CK(cudaStreamWaitEvent(s0.stream(), s.ev_bnd, 0));
                if (&s != &s0) {
                    CK(cudaSetDevice(s.dev));
                    CK(cudaEventRecord(s.ev_bnd, s.stream()));
                    CK(cudaSetDevice(s0.dev));
                    CK(cudaStreamWaitEvent(s0.stream(), s.ev_bnd, 0));
                }
            }
            CK(cudaSetDevice(s0.dev));
            CK(cudaGraphLaunch(s0.graph, s0.stream()));
            CK(cudaEventRecord(s0.ev_bnd, s0.stream()));
            for (auto& s : c->slabs) {
                CK(cudaSetDevice(s.dev));
                CK(cudaStreamWaitEvent(s.s_comm, s0.ev_bnd, 0));
                if (&s != &s0) CK(cudaStreamWaitEvent(s.stream(), s0.ev_bnd, 0));
                CK(cudaEventRecord(s.ev_comm, s.s_comm));  // the neighbours' next waits see the graph
                CK(cudaEventRecord(s.ev_done, s.stream()));
            }
            c->step += 2 * GRAPH_PAIRS;
            c->launches += launches_per_step * 2 * GRAPH_PAIRS;
            k += 2 * GRAPH_PAIRS;
            continue;
        }
        RET(c->halo_mode == 1 ? enqueue_slab_step1(c) : enqueue_slab_step0(c));
        ++k;
    }
    return join_slabs(c);
}

int sync_all(rtm_ctx* c) {
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        CK(cudaStreamSynchronize(s.stream()));
        CK(cudaStreamSynchronize(s.s_comm));
    }
    if (c->comm) {
        ncclResult_t ar;
        NK(ncclCommGetAsyncError(c->comm, &ar));
        if (ar != ncclSuccess) return fail(RTM_ENCCL, "NCCL async error: %s", ncclGetErrorString(ar));
    }
    return RTM_OK;
}

// Copy host slab arrays (x fastest) into/out of the interior planes of a device buffer.
// Copy nplanes planes between an unpadded array (nx per row) and a pitched device field.
// to_dev: src unpadded -> dst pitched; otherwise src pitched -> dst unpadded.
int copy_planes(const rtm_ctx* c, void* dst, const void* src, size_t nplanes, bool to_dev,
                cudaMemcpyKind kind, cudaStream_t st) {
    const size_t rows = (size_t)c->ny * nplanes;
    if (c->px == c->nx)
        CK(cudaMemcpyAsync(dst, src, rows * c->nx * sizeof(float), kind, st));
    else
        CK(cudaMemcpy2DAsync(dst, (to_dev ? c->px : c->nx) * sizeof(float), src,
                             (to_dev ? c->nx : c->px) * sizeof(float), c->nx * sizeof(float), rows,
                             kind, st));
    return RTM_OK;
}

int h2d_planes(rtm_ctx* c, Slab& s, float* dst_base, const float* host, cudaStream_t st) {
    return copy_planes(c, dst_base, host, s.nzl, true, cudaMemcpyHostToDevice, st);
}

int async_vcheck(rtm_ctx* c);

int set_velocity_impl(rtm_ctx* c, const float* v, bool device_ptr) {
    RET(async_vcheck(c));  // verdict of earlier rtm_set_velocity_async calls (synchronising)
    c->vel_set = false;
    const size_t plane = hplane(c);  // offsets into the caller's unpadded array
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        cudaStream_t st = s.stream();
        const float* src;
        if (device_ptr && c->px == c->nx) {
            src = v + (size_t)(s.z0 - c->slabs[0].z0) * plane;
        } else {
            // stage v in C (pitched) and convert in place
            const float* h = v + (device_ptr ? (size_t)(s.z0 - c->slabs[0].z0) * plane
                                             : (c->mode == 1 ? (size_t)s.z0 * plane : 0));
            RET(copy_planes(c, s.C, h, s.nzl, true,
                            device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
            src = s.C;
        }
        CK(cudaMemsetAsync(s.d_stats, 0, 2 * sizeof(unsigned int), st));
        CK(launch_velocity(src, s.C, (long long)(dplane(c) * s.nzl), c->nx, c->px, (double)c->dt,
                           (double)c->dx, s.d_stats, st));
    }
    float vmax = 0.0f;
    unsigned long long bad = 0;
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        unsigned int h[2];
        CK(cudaMemcpyAsync(h, s.d_stats, sizeof h, cudaMemcpyDeviceToHost, s.stream()));
        CK(cudaStreamSynchronize(s.stream()));
        float m;
        std::memcpy(&m, &h[0], 4);
        vmax = std::max(vmax, m);
        bad += h[1];
    }
    if (bad) return fail(RTM_EINVAL, "velocity has %llu non-finite or non-positive values", bad);
    const double nu = (double)vmax * (double)c->dt / (double)c->dx;
    if (nu > c->nu_crit)
        return fail(RTM_ECFL, "CFL violated: max(v)*dt/dx = %.6f > nu_crit = %.6f (max v = %g m/s)",
                    nu, c->nu_crit, (double)vmax);
    c->vel_set = true;
    return RTM_OK;
}

int reset_impl(rtm_ctx* c, const float* u, const float* up) {
    const size_t plane = hplane(c), dpl = dplane(c);
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        cudaStream_t st = s.stream();
        CK(cudaStreamSynchronize(s.s_comm));
        const size_t nbuf = dpl * s.buf_planes();
        for (int b = 0; b < 2; ++b) CK(cudaMemsetAsync(s.buf[b], 0, nbuf * sizeof(float), st));
        const size_t off = c->mode == 1 ? (size_t)s.z0 * plane : 0;
        for (int k = 0; k < s.nshots; ++k) {  // host arrays: (nshots, nz, ny, nx)
            const size_t hoff = off + (size_t)k * plane * s.nzl;
            const size_t doff = ((size_t)k * (s.nzl + 10) + 5) * dpl;
            if (u) RET(h2d_planes(c, s, s.buf[0] + doff, u + hoff, st));
            if (up) RET(h2d_planes(c, s, s.buf[1] + doff, up + hoff, st));
        }
        CK(cudaMemsetAsync(s.d_step, 0, 2 * sizeof(int), st));
    }
    c->step = 0;
    ++c->sig_gen;  // synchronising (halo exchange + sync below): flags restart
    c->sig_fresh = true;
    // G > 1: fill the halo planes of u^0 from the neighbours' initial data.  Only u^0: the
    // stencil reads u^{-1} at owned points only, so the halo planes of buf[1] are never read
    // before step 0 overwrites them (its exchange or fused push).  Not exchanging them also
    // keeps the first (wait-free) fused-push step of a generation race-free across ranks: the
    // only remote write into this slab's buf[1] halo planes is then the neighbour's push, and
    // the neighbour can only push after this exchange, i.e. after this rank's reset memsets
    // (stream order on the sending side of the exchange).
    if (c->mode == 3) {  // peer context: pull through the IPC mappings after a barrier
        RET(sync_all(c));
        if (c->world > 1) RET(pull_halos_now(c, 0));
        return RTM_OK;
    }
    if (c->slabs.size() > 1 || c->mode == 2) {
        for (auto& s : c->slabs) {
            CK(cudaSetDevice(s.dev));
            CK(cudaEventRecord(s.ev_bnd, s.stream()));
        }
        if (c->mode == 2) RET(exchange_nccl(c, 0));
        else RET(exchange_local(c, 0));
    }
    return sync_all(c);
}

int read_impl(rtm_ctx* c, float* out, int which /*0 = u^n, 1 = u^{n-1}*/) {
    const size_t plane = hplane(c), dpl = dplane(c);
    const int par = (int)((c->step + which) & 1);
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        const size_t off = c->mode == 1 ? (size_t)s.z0 * plane : 0;
        for (int k = 0; k < s.nshots; ++k)
            RET(copy_planes(c, out + off + (size_t)k * plane * s.nzl,
                            s.buf[par] + ((size_t)k * (s.nzl + 10) + 5) * dpl, s.nzl, false,
                            cudaMemcpyDeviceToHost, s.stream()));
    }
    return sync_all(c);
}

// The asynchronous pipeline's copy stream, events and staging buffers (lazily, single slab).
int async_setup(rtm_ctx* c, bool need_stage, bool need_snap) {
    if (c->slabs.size() != 1) return fail(RTM_EINVAL, "the asynchronous calls need a single-slab context");
    Slab& s = c->slabs[0];
    CK(cudaSetDevice(s.dev));
    if (!c->s_copy) {
        CK(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&c->ev_h2d, &c->ev_conv, &c->ev_snap, &c->ev_d2h})
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    const size_t n = hplane(c) * s.nzl;  // the snapshot is unpadded (host layout)
    const size_t nst = dplane(c) * s.nzl;  // the velocity staging is pitched (device layout)
    if (need_stage && !c->v_stage && cudaMalloc(&c->v_stage, nst * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        return fail(RTM_ENOMEM, "velocity staging buffer (%zu bytes)", nst * 4);
    }
    if (need_snap && !c->snap && cudaMalloc(&c->snap, n * s.nshots * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        return fail(RTM_ENOMEM, "readback snapshot buffer (%zu bytes)", n * s.nshots * 4);
    }
    return RTM_OK;
}

// Deferred verdict of the velocities given to rtm_set_velocity_async since the last check
// (d_stats accumulates max v and the invalid count over all of them).  Host-synchronising.
int async_vcheck(rtm_ctx* c) {
    if (!c->vcheck_pending) return RTM_OK;
    c->vcheck_pending = false;
    Slab& s = c->slabs[0];
    unsigned int hs[2];
    CK(cudaMemcpyAsync(hs, s.d_stats, sizeof hs, cudaMemcpyDeviceToHost, s.stream()));
    CK(cudaStreamSynchronize(s.stream()));
    float m;
    std::memcpy(&m, &hs[0], 4);
    if (hs[1]) {
        c->vel_set = false;
        return fail(RTM_EINVAL, "an asynchronous velocity had %u non-finite or non-positive values", hs[1]);
    }
    const double nu = (double)m * (double)c->dt / (double)c->dx;
    if (nu > c->nu_crit) {
        c->vel_set = false;
        return fail(RTM_ECFL, "an asynchronous velocity violated CFL: max(v)*dt/dx = %.6f > %.6f", nu, c->nu_crit);
    }
    return RTM_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

const char* rtm_last_error(void) { return g_err.c_str(); }

double rtm_nu_crit(const float coeffs[6]) {
    if (!coeffs || !finite_coeffs(coeffs)) return -1.0;
    const double s = smax_of(coeffs);
    return s > 0 ? 2.0 / std::sqrt(3.0 * s) : -1.0;
}

int rtm_slab_range(int nz_global, int world, int rank, int* z0, int* nzl) {
    if (world < 1 || rank < 0 || rank >= world || nz_global < 1 || !z0 || !nzl)
        return fail(RTM_EINVAL, "invalid slab request (nz=%d world=%d rank=%d)", nz_global, world, rank);
    const long long a = (long long)rank * nz_global / world;
    const long long b = (long long)(rank + 1) * nz_global / world;
    if (world > 1 && (long long)nz_global / world < 10)
        return fail(RTM_EINVAL, "nz/world = %d/%d < 10 planes per slab", nz_global, world);
    *z0 = (int)a;
    *nzl = (int)(b - a);
    return RTM_OK;
}

int rtm_halo_plan(int nx, int ny, int nzl, int rank, int world, long long offsets[4],
                  long long* count) {
    if (nx < 1 || ny < 1 || nzl < 1 || world < 1 || rank < 0 || rank >= world || !offsets || !count)
        return fail(RTM_EINVAL, "invalid halo plan request");
    if (world > 1 && nzl < 10) return fail(RTM_EINVAL, "nzl=%d < 10", nzl);
    const long long plane = (long long)nx * ny;
    const bool lo = rank > 0, hi = rank < world - 1;
    offsets[0] = lo ? 5 * plane : -1;
    offsets[1] = lo ? 0 : -1;
    offsets[2] = hi ? (long long)nzl * plane : -1;
    offsets[3] = hi ? (long long)(nzl + 5) * plane : -1;
    *count = 5 * plane;
    return RTM_OK;
}

int rtm_num_tiles(void) { return num_variants(); }
const char* rtm_tile_name(int id) {
    if (id < 0 || id >= num_variants()) return nullptr;
    return variant(id).name;
}

rtm_ctx* rtm_create(int nx, int ny, int nz, float dx, float dt, const float coeffs[6]) {
    DeviceGuard g;
    rtm_ctx* c = new_ctx(nx, ny, nz, dx, dt, coeffs);
    if (!c) return nullptr;
    c->mode = 0;
    Slab s;
    cudaGetDevice(&s.dev);
    s.z0 = 0;
    s.nzl = nz;
    c->slabs.push_back(s);
    if (finish_ctx(c) != RTM_OK) {
        std::string e = g_err;
        destroy_ctx(c);
        g_err = e;
        return nullptr;
    }
    return c;
}

rtm_ctx* rtm_create_batch(int nx, int ny, int nz, float dx, float dt, const float coeffs[6],
                          int nshots) {
    DeviceGuard g;
    if (nshots < 1) {
        fail(RTM_EINVAL, "nshots must be >= 1");
        return nullptr;
    }
    if ((long long)nshots * (nz + 10) > (1LL << 31) - 1) {
        fail(RTM_EINVAL, "nshots*(nz+10) = %lld planes exceeds 2^31", (long long)nshots * (nz + 10));
        return nullptr;
    }
    rtm_ctx* c = new_ctx(nx, ny, nz, dx, dt, coeffs);
    if (!c) return nullptr;
    c->mode = 0;
    Slab s;
    cudaGetDevice(&s.dev);
    s.z0 = 0;
    s.nzl = nz;
    s.nshots = nshots;
    c->slabs.push_back(s);
    if (finish_ctx(c) != RTM_OK) {
        std::string e = g_err;
        destroy_ctx(c);
        g_err = e;
        return nullptr;
    }
    return c;
}

int rtm_num_shots(rtm_ctx* c) { return c ? c->slabs[0].nshots : -1; }

rtm_ctx* rtm_create_multi(int nx, int ny, int nz, float dx, float dt, const float coeffs[6],
                          int nslabs, const int* devices) {
    DeviceGuard g;
    if (nslabs < 1 || !devices) {
        fail(RTM_EINVAL, "nslabs must be >= 1 and devices non-NULL");
        return nullptr;
    }
    int z0, nzl;
    for (int r = 0; r < nslabs; ++r)
        if (rtm_slab_range(nz, nslabs, r, &z0, &nzl) != RTM_OK) return nullptr;
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    for (int r = 0; r < nslabs; ++r)
        if (devices[r] < 0 || devices[r] >= ndev) {
            fail(RTM_EINVAL, "devices[%d] = %d is not a CUDA device (count %d)", r, devices[r], ndev);
            return nullptr;
        }
    rtm_ctx* c = new_ctx(nx, ny, nz, dx, dt, coeffs);
    if (!c) return nullptr;
    c->mode = 1;
    for (int r = 0; r < nslabs; ++r) {
        Slab s;
        s.dev = devices[r];
        rtm_slab_range(nz, nslabs, r, &s.z0, &s.nzl);
        s.lo_nb = r > 0;
        s.hi_nb = r < nslabs - 1;
        c->slabs.push_back(s);
    }
    for (int r = 0; r < nslabs; ++r)
        for (int q = 0; q < nslabs; ++q)
            if (devices[q] == devices[r] && q != r) ++c->slabs[r].share;
    for (int r = 0; r < nslabs; ++r)  // best effort peer access (copies work either way)
        for (int q = 0; q < nslabs; ++q)
            if (devices[r] != devices[q]) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, devices[r], devices[q]);
                if (can) {
                    cudaSetDevice(devices[r]);
                    cudaDeviceEnablePeerAccess(devices[q], 0);
                    cudaGetLastError();
                }
            }
    if (finish_ctx(c) != RTM_OK) {
        std::string e = g_err;
        destroy_ctx(c);
        g_err = e;
        return nullptr;
    }
    return c;
}

int rtm_get_unique_id(unsigned char id[128]) {
    if (!id) return fail(RTM_EINVAL, "id is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    NK(ncclGetUniqueId(&u));
    std::memcpy(id, &u, 128);
    return RTM_OK;
}

rtm_ctx* rtm_create_dist(int nx, int ny, int nz_global, float dx, float dt,
                         const float coeffs[6], int rank, int world, const unsigned char id[128],
                         int device) {
    DeviceGuard g;
    int z0, nzl;
    if (rtm_slab_range(nz_global, world, rank, &z0, &nzl) != RTM_OK) return nullptr;
    if (!id) {
        fail(RTM_EINVAL, "id is NULL");
        return nullptr;
    }
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    if (device < 0 || device >= ndev) {
        fail(RTM_EINVAL, "device %d is not a CUDA device (count %d)", device, ndev);
        return nullptr;
    }
    rtm_ctx* c = new_ctx(nx, ny, nz_global, dx, dt, coeffs);
    if (!c) return nullptr;
    c->mode = 2;
    c->rank = rank;
    c->world = world;
    Slab s;
    s.dev = device;
    s.z0 = z0;
    s.nzl = nzl;
    s.lo_nb = rank > 0;
    s.hi_nb = rank < world - 1;
    c->slabs.push_back(s);
    if (finish_ctx(c) != RTM_OK) {
        std::string e = g_err;
        destroy_ctx(c);
        g_err = e;
        return nullptr;
    }
    cudaSetDevice(device);
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        destroy_ctx(c);
        fail(RTM_ENCCL, "ncclCommInitRank failed: %s", ncclGetErrorString(r));
        return nullptr;
    }
    return c;
}

rtm_ctx* rtm_create_peer(int nx, int ny, int nz_global, float dx, float dt, const float coeffs[6],
                         int rank, int world, int device) {
    DeviceGuard g;
    int z0, nzl;
    if (rtm_slab_range(nz_global, world, rank, &z0, &nzl) != RTM_OK) return nullptr;
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    if (device < 0 || device >= ndev) {
        fail(RTM_EINVAL, "device %d is not a CUDA device (count %d)", device, ndev);
        return nullptr;
    }
    rtm_ctx* c = new_ctx(nx, ny, nz_global, dx, dt, coeffs);
    if (!c) return nullptr;
    c->mode = 3;
    c->rank = rank;
    c->world = world;
    c->halo_mode = 3;
    Slab s;
    s.dev = device;
    s.z0 = z0;
    s.nzl = nzl;
    s.lo_nb = rank > 0;
    s.hi_nb = rank < world - 1;
    c->slabs.push_back(s);
    if (finish_ctx(c) != RTM_OK || alloc_sig(c->slabs[0]) != RTM_OK) {
        std::string e = g_err;
        destroy_ctx(c);
        g_err = e;
        return nullptr;
    }
    return c;
}

int rtm_ipc_export(rtm_ctx* c, unsigned char rec[RTM_IPC_RECORD_BYTES]) {
    if (!c || !rec) return fail(RTM_EINVAL, "NULL argument");
    if (c->mode != 2 && c->mode != 3) return fail(RTM_EINVAL, "IPC records belong to distributed or peer contexts");
    DeviceGuard g;
    IpcRecord r;
    RET(export_record(c, &r));
    std::memcpy(rec, &r, sizeof r);
    return RTM_OK;
}

int rtm_ipc_import(rtm_ctx* c, const unsigned char* lo, const unsigned char* hi) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (c->mode != 2 && c->mode != 3) return fail(RTM_EINVAL, "IPC records belong to distributed or peer contexts");
    DeviceGuard g;
    IpcRecord rl, rh;
    if (lo) std::memcpy(&rl, lo, sizeof rl);
    if (hi) std::memcpy(&rh, hi, sizeof rh);
    return import_records(c, lo ? &rl : nullptr, hi ? &rh : nullptr);
}

int rtm_set_host_barrier(rtm_ctx* c, rtm_barrier_fn fn, void* user) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    c->barrier_fn = fn;
    c->barrier_user = user;
    return RTM_OK;
}

double rtm_last_enqueue_ms(rtm_ctx* c) { return c ? c->enqueue_ms : -1.0; }

void rtm_destroy(rtm_ctx* ctx) { destroy_ctx(ctx); }

int rtm_set_velocity(rtm_ctx* c, const float* v) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (!v) return fail(RTM_EINVAL, "v is NULL");
    DeviceGuard g;
    return set_velocity_impl(c, v, false);
}

int rtm_set_velocity_device(rtm_ctx* c, const float* d_v) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (!d_v) return fail(RTM_EINVAL, "d_v is NULL");
    if (c->slabs.size() != 1) return fail(RTM_EINVAL, "device velocity needs a single-slab context");
    DeviceGuard g;
    return set_velocity_impl(c, d_v, true);
}

int rtm_inject_source_shot(rtm_ctx* c, int shot, int ix, int iy, int iz, const float* samples,
                           int nsamples) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (shot < 0 || shot >= c->slabs[0].nshots)
        return fail(RTM_EINVAL, "shot %d outside [0, %d)", shot, c->slabs[0].nshots);
    if (ix < 0 || ix >= c->nx || iy < 0 || iy >= c->ny || iz < 0 || iz >= c->nz)
        return fail(RTM_EINVAL, "source (%d,%d,%d) outside the %dx%dx%d interior", ix, iy, iz,
                    c->nx, c->ny, c->nz);
    if (nsamples < 0 || (nsamples > 0 && !samples))
        return fail(RTM_EINVAL, "nsamples must be >= 0 with non-NULL samples");
    for (int n = 0; n < nsamples; ++n)
        if (!std::isfinite(samples[n])) return fail(RTM_EINVAL, "samples[%d] is not finite", n);
    if ((int)c->sources.size() >= RTM_MAX_SOURCES)
        return fail(RTM_EINVAL, "at most %d sources", RTM_MAX_SOURCES);
    DeviceGuard g;
    HostSource hs{ix, iy, iz, shot, std::vector<float>(samples, samples + nsamples)};
    c->sources.push_back(hs);
    for (auto& s : c->slabs) {
        if (iz < s.z0 || iz >= s.z0 + s.nzl) continue;  // owned by another slab / rank
        DevSource d;
        d.x = ix;
        d.y = iy;
        d.z = iz - s.z0;
        d.shot = shot;
        d.nsamples = nsamples;
        d.offset = (long long)s.h_samples.size();
        s.h_samples.insert(s.h_samples.end(), samples, samples + nsamples);
        s.srcs.push_back(d);
        RET(upload_sources(c, s));
    }
    return RTM_OK;
}

int rtm_inject_source(rtm_ctx* c, int ix, int iy, int iz, const float* samples, int nsamples) {
    return rtm_inject_source_shot(c, 0, ix, iy, iz, samples, nsamples);
}

int rtm_step(rtm_ctx* c, int nsteps) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (nsteps < 0) return fail(RTM_EINVAL, "nsteps must be >= 0");
    if (!c->vel_set) return fail(RTM_ESTATE, "rtm_step before a successful rtm_set_velocity");
    DeviceGuard g;
    Slab& s0 = c->slabs[0];
    CK(cudaSetDevice(s0.dev));
    c->prof_launches = 0;
    if (c->check_every > 0) {  // failure detection: advance in blocks, scan between them
        int left = nsteps;
        while (left > 0) {
            const long long to_boundary = c->check_every - (c->step % c->check_every);
            const int k = (int)std::min<long long>(left, to_boundary);
            c->check_every = -c->check_every;  // run the block unchecked
            const int rc = rtm_step(c, k);
            c->check_every = -c->check_every;
            if (rc != RTM_OK) return rc;
            left -= k;
            if (c->step % c->check_every == 0) {
                double m;
                long long bad;
                RET(rtm_field_stats(c, &m, &bad));
                if (bad)
                    return fail(RTM_EUNSTABLE, "%lld non-finite values in u at step %lld", bad, c->step);
            }
        }
        return RTM_OK;
    }
    if (c->mode == 3 && c->world > 1 && !c->ipc_imported)
        return fail(RTM_ESTATE, "peer context: rtm_ipc_import the neighbours' records before rtm_step");
    const auto h0 = std::chrono::steady_clock::now();
    CK(cudaEventRecord(c->t0, s0.stream()));
    if (c->mode == 0) {
        RET(step_single(c, nsteps));
    } else {
        for (size_t r = 1; r < c->slabs.size(); ++r) {  // start together
            CK(cudaSetDevice(c->slabs[r].dev));
            CK(cudaStreamWaitEvent(c->slabs[r].stream(), c->t0, 0));
        }
        RET(step_slabs(c, nsteps));
        CK(cudaSetDevice(s0.dev));
        for (size_t r = 1; r < c->slabs.size(); ++r) {
            CK(cudaEventRecord(c->slabs[r].ev_bnd, c->slabs[r].stream()));
            CK(cudaStreamWaitEvent(s0.stream(), c->slabs[r].ev_bnd, 0));
        }
    }
    CK(cudaSetDevice(s0.dev));
    CK(cudaEventRecord(c->t1, s0.stream()));
    c->enqueue_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    RET(sync_all(c));
    CK(cudaEventElapsedTime(&c->last_ms, c->t0, c->t1));
    RET(collect_profile(c));
    c->prof_launches = 0;
    return async_vcheck(c);
}

int rtm_read_field(rtm_ctx* c, float* out) {
    if (!c || !out) return fail(RTM_EINVAL, "NULL argument");
    DeviceGuard g;
    return read_impl(c, out, 0);
}

int rtm_read_fields(rtm_ctx* c, float* u, float* up) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    DeviceGuard g;
    if (u) RET(read_impl(c, u, 0));
    if (up) RET(read_impl(c, up, 1));
    return RTM_OK;
}

int rtm_read_field_device(rtm_ctx* c, float* d_out) {
    if (!c || !d_out) return fail(RTM_EINVAL, "NULL argument");
    if (c->slabs.size() != 1) return fail(RTM_EINVAL, "device readback needs a single-slab context");
    DeviceGuard g;
    Slab& s = c->slabs[0];
    CK(cudaSetDevice(s.dev));
    const size_t plane = hplane(c), dpl = dplane(c);
    for (int k = 0; k < s.nshots; ++k)
        RET(copy_planes(c, d_out + (size_t)k * plane * s.nzl,
                        s.buf[c->step & 1] + ((size_t)k * (s.nzl + 10) + 5) * dpl, s.nzl, false,
                        cudaMemcpyDeviceToDevice, s.stream()));
    return RTM_OK;
}

int rtm_set_fields(rtm_ctx* c, const float* u, const float* up) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    DeviceGuard g;
    return reset_impl(c, u, up);
}

int rtm_reset(rtm_ctx* c) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    DeviceGuard g;
    if (c->mode == 0) {  // enqueue only (the bench times reset inside a step)
        Slab& s = c->slabs[0];
        CK(cudaSetDevice(s.dev));
        const size_t nbuf = dplane(c) * s.buf_planes();
        for (int b = 0; b < 2; ++b) CK(cudaMemsetAsync(s.buf[b], 0, nbuf * sizeof(float), s.stream()));
        CK(cudaMemsetAsync(s.d_step, 0, 2 * sizeof(int), s.stream()));
        c->step = 0;
        return RTM_OK;
    }
    return reset_impl(c, nullptr, nullptr);
}

long long rtm_step_count(rtm_ctx* c) { return c ? c->step : -1; }

int rtm_get_dims(rtm_ctx* c, int* nx, int* ny, int* nzl, int* nshots) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (nx) *nx = c->nx;
    if (ny) *ny = c->ny;
    if (nzl) *nzl = (c->mode == 2 || c->mode == 3) ? c->slabs[0].nzl : c->nz;
    if (nshots) *nshots = c->slabs[0].nshots;
    return RTM_OK;
}

int rtm_set_step_count(rtm_ctx* c, long long n) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (n < 0 || n > (1LL << 30)) return fail(RTM_EINVAL, "step index %lld out of range", n);
    DeviceGuard g;
    RET(sync_all(c));
    // the time levels stay where rtm_set_fields put them (u in buf[0], u_prev in buf[1]): if
    // the parity of n is odd, swap so that u^n lives in buf[n & 1]
    if ((n & 1) != (c->step & 1))
        for (auto& s : c->slabs) {
            std::swap(s.buf[0], s.buf[1]);
            std::swap(s.nb_lo[0], s.nb_lo[1]);  // every slab / rank swaps alike
            std::swap(s.nb_hi[0], s.nb_hi[1]);
            s.tm_variant = -1;  // tensor maps follow the buffers
            s.graph_valid = false;
            for (int k = 0; k < 4; ++k) s.tb_graph_variant[k] = -1;
        }
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        int h[2] = {(int)n, (int)n};
        CK(cudaMemcpy(s.d_step, h, sizeof h, cudaMemcpyHostToDevice));
    }
    c->step = n;
    if (c->halo_mode >= 2) {  // flags restart: make the call collective across ranks
        RET(ranks_barrier(c));
        ++c->sig_gen;
        c->sig_fresh = true;
    }
    return RTM_OK;
}

int rtm_field_stats(rtm_ctx* c, double* max_abs, long long* nonfinite) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    DeviceGuard g;
    const long long plane = (long long)dplane(c);  // padding columns are zero: no effect on stats
    double m = 0;
    long long bad = 0;
    for (auto& s : c->slabs) {
        CK(cudaSetDevice(s.dev));
        CK(cudaMemsetAsync(s.d_fstats, 0, 2 * sizeof(unsigned int), s.stream()));
        CK(launch_field_stats(s.buf[c->step & 1], plane, s.nzl, s.nshots, s.d_fstats, s.stream()));
        unsigned int h[2];
        CK(cudaMemcpyAsync(h, s.d_fstats, sizeof h, cudaMemcpyDeviceToHost, s.stream()));
        CK(cudaStreamSynchronize(s.stream()));
        float f;
        std::memcpy(&f, &h[0], 4);
        m = std::max(m, (double)f);
        bad += h[1];
    }
    if (max_abs) *max_abs = m;
    if (nonfinite) *nonfinite = bad;
    return RTM_OK;
}

int rtm_set_tile(rtm_ctx* c, int tile_id) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (tile_id < -1 || tile_id >= num_variants())
        return fail(RTM_EINVAL, "unknown tile id %d (valid: -1 .. %d)", tile_id, num_variants() - 1);
    c->tile = tile_id;
    invalidate_graphs(c);
    return RTM_OK;
}

int rtm_get_tile(rtm_ctx* c) { return c ? resolve_tile(c) : -1; }

int rtm_set_zchunk(rtm_ctx* c, int planes) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (planes < 0) return fail(RTM_EINVAL, "planes must be >= 0");
    c->zchunk = planes;
    invalidate_graphs(c);
    return RTM_OK;
}

int rtm_set_option(rtm_ctx* c, int key, long long value) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    switch (key) {
        case RTM_OPT_ZCHUNK:
            if (value < 0 || value > (1 << 30)) return fail(RTM_EINVAL, "zchunk %lld out of range", value);
            c->zchunk = (int)value;
            break;
        case RTM_OPT_CACHE_MODE:
            if (value < 0 || value > 0xfff) return fail(RTM_EINVAL, "cache mode %lld out of range", value);
            c->cache_mode = (int)value;
            break;
        case RTM_OPT_GRAPHS:
            c->graphs = value != 0;
            break;
        case RTM_OPT_SHOT_ORDER:
            if (value < 0 || value > 2) return fail(RTM_EINVAL, "shot order %lld not in 0..2", value);
            c->shot_order = (int)value;
            break;
        case RTM_OPT_CHECK_EVERY:
            if (value < 0 || value > (1 << 30)) return fail(RTM_EINVAL, "check interval %lld", value);
            c->check_every = (int)value;
            break;
        case RTM_OPT_TB_CTAS:
            if (value < 0 || value > (1 << 20)) return fail(RTM_EINVAL, "tb ctas %lld out of range", value);
            c->tb_ctas = (int)value;
            break;
        case RTM_OPT_PDL:
            if (value < 0 || value > 1) return fail(RTM_EINVAL, "pdl %lld not in 0..1", value);
            c->pdl = value != 0;
            break;
        case RTM_OPT_HOST_ORDERED:
            if (value < 0 || value > 1) return fail(RTM_EINVAL, "host ordered %lld not in 0..1", value);
            c->host_ordered = value != 0;
            break;
        case RTM_OPT_SLAB_SHARE:
            if (value < 0 || value > 1) return fail(RTM_EINVAL, "slab share %lld not in 0..1", value);
            c->share_sms = value != 0;
            break;
        case RTM_OPT_ZDIR:
            if (value < 0 || value > 7) return fail(RTM_EINVAL, "z direction mode %lld not in 0..7", value);
            c->zdir = (int)value;
            break;
        case RTM_OPT_HALO_MODE:
            if (value < 0 || value > 3) return fail(RTM_EINVAL, "halo mode %lld not in 0..3", value);
            if (value == 0 && c->mode == 3 && c->world > 1)
                return fail(RTM_EINVAL, "halo mode 0 (NCCL / in-process copies) is not available in a peer context (no NCCL)");
            if (value == 1 && c->mode != 1)
                return fail(RTM_EINVAL, "halo mode 1 (fused push, event ordered) needs an in-process multi-slab context");
            if (value >= 2 && c->mode == 0)
                return fail(RTM_EINVAL, "halo modes 2-3 (flag protocol) need a multi-slab, distributed or peer context");
            if (value >= 1 && c->mode == 1) {  // every slab must be able to store into its neighbours
                for (size_t r = 0; r + 1 < c->slabs.size(); ++r) {
                    const int a = c->slabs[r].dev, b = c->slabs[r + 1].dev;
                    int ab = 1, ba = 1;
                    if (a != b) {
                        cudaDeviceCanAccessPeer(&ab, a, b);
                        cudaDeviceCanAccessPeer(&ba, b, a);
                    }
                    if (!ab || !ba)
                        return fail(RTM_EINVAL, "devices %d and %d have no peer access", a, b);
                }
            }
            {  // switch cleanly: drain first (mode 2 contexts: a collective call)
                DeviceGuard g;
                RET(sync_all(c));
                if (value >= 2) RET(setup_signal(c));
                c->halo_mode = (int)value;
            }
            break;
        default:
            return fail(RTM_EINVAL, "unknown option key %d", key);
    }
    invalidate_graphs(c);
    return RTM_OK;
}

long long rtm_get_option(rtm_ctx* c, int key) {
    if (!c) return -1;
    switch (key) {
        case RTM_OPT_ZCHUNK: return c->zchunk;
        case RTM_OPT_CACHE_MODE: return c->cache_mode;
        case RTM_OPT_GRAPHS: return c->graphs ? 1 : 0;
        case RTM_OPT_SHOT_ORDER: return c->shot_order;
        case RTM_OPT_HALO_MODE: return c->halo_mode;
        case RTM_OPT_CHECK_EVERY: return c->check_every;
        case RTM_OPT_TB_CTAS: return c->tb_ctas;
        case RTM_OPT_PDL: return c->pdl ? 1 : 0;
        case RTM_OPT_HOST_ORDERED: return c->host_ordered ? 1 : 0;
        case RTM_OPT_ZDIR: return c->zdir;
        case RTM_OPT_SLAB_SHARE: return c->share_sms ? 1 : 0;
        default: return -1;
    }
}

int rtm_blocksize_lattice(int S, int P, int* out) {
    if (S < 1 || P < 2 || !out) return fail(RTM_EINVAL, "lattice needs S >= 1, P >= 2, out != NULL");
    int n = 0;
    for (int k = 0; k < P; ++k) {
        long long b = (long long)k * S / (P - 1) + 1;
        if (b > S) b = S;                               // PAPER.md:301 worked example (R17)
        if (n == 0 || out[n - 1] != (int)b) out[n++] = (int)b;
    }
    return n;
}

int rtm_select_mwmb(const double* times, int nranks, int ncand) {
    if (!times || nranks < 1 || ncand < 1) return -1;
    int best = -1;
    double bestv = 0;
    for (int cnd = 0; cnd < ncand; ++cnd) {
        double worst = -1e300;
        bool failed = false;
        for (int r = 0; r < nranks; ++r) {
            const double t = times[(size_t)r * ncand + cnd];
            if (std::isnan(t)) failed = true;  // the candidate failed somewhere
            else worst = std::max(worst, t);
        }
        if (failed) continue;
        if (best < 0 || worst < bestv) best = cnd, bestv = worst;
    }
    return best;
}

namespace {

// Time nI steps (after one warm-up step) on the context's streams; in a distributed context
// the result is the max over ranks (NCCL all-reduce).
int timed_steps(rtm_ctx* c, int nI, double* ms_out, double* d_scratch) {
    RET(rtm_step(c, 1));
    RET(rtm_step(c, nI));
    double ms = c->last_ms;
    if (c->comm) {
        Slab& s = c->slabs[0];
        CK(cudaMemcpyAsync(d_scratch, &ms, sizeof(double), cudaMemcpyHostToDevice, s.stream()));
        NK(ncclAllReduce(d_scratch, d_scratch, 1, ncclFloat64, ncclMax, c->comm, s.stream()));
        CK(cudaMemcpyAsync(&ms, d_scratch, sizeof(double), cudaMemcpyDeviceToHost, s.stream()));
        CK(cudaStreamSynchronize(s.stream()));
    }
    *ms_out = ms;
    return RTM_OK;
}

}  // namespace

int rtm_autotune(rtm_ctx* c, int nI, const int* tiles, const int* zchunks, int ncand,
                 rtm_tune_result* out, double* cand_ms) {
    if (!c || !out) return fail(RTM_EINVAL, "NULL argument");
    if (nI < 1) return fail(RTM_EINVAL, "nI must be >= 1");
    if (!c->vel_set) return fail(RTM_ESTATE, "rtm_autotune before a successful rtm_set_velocity");
    std::vector<int> ct, cz;
    if (tiles) {
        if (ncand < 1) return fail(RTM_EINVAL, "ncand must be >= 1");
        for (int k = 0; k < ncand; ++k) {
            if (tiles[k] < 0 || tiles[k] >= num_variants())
                return fail(RTM_EINVAL, "candidate %d: unknown tile %d", k, tiles[k]);
            const int z = zchunks ? zchunks[k] : 0;
            if (z < 0) return fail(RTM_EINVAL, "candidate %d: z-chunk %d < 0", k, z);
            ct.push_back(tiles[k]);
            cz.push_back(z);
        }
    } else {
        for (int t = 1; t < num_variants(); ++t) {
            ct.push_back(t);
            cz.push_back(0);
        }
    }
    DeviceGuard g;
    const int saved_tile = c->tile, saved_zc = c->zchunk;
    const long long saved_step = c->step;
    // snapshot both time levels + step counters of every slab
    std::vector<float*> snap(2 * c->slabs.size(), nullptr);
    std::vector<int> snap_step(2 * c->slabs.size());
    double* d_scratch = nullptr;
    int rc = RTM_OK;
    auto cleanup = [&]() {
        for (size_t k = 0; k < c->slabs.size(); ++k) {
            cudaSetDevice(c->slabs[k].dev);
            for (int b = 0; b < 2; ++b)
                if (snap[2 * k + b]) cudaFree(snap[2 * k + b]);
        }
        if (d_scratch) cudaFree(d_scratch);
    };
    for (size_t k = 0; k < c->slabs.size() && rc == RTM_OK; ++k) {
        Slab& s = c->slabs[k];
        cudaSetDevice(s.dev);
        const size_t bytes = dplane(c) * s.buf_planes() * sizeof(float);
        for (int b = 0; b < 2 && rc == RTM_OK; ++b) {
            if (cudaMalloc(&snap[2 * k + b], bytes) != cudaSuccess) {
                cudaGetLastError();
                rc = fail(RTM_ENOMEM, "autotune snapshot allocation (%zu bytes) failed", bytes);
                break;
            }
            if (cudaMemcpyAsync(snap[2 * k + b], s.buf[b], bytes, cudaMemcpyDeviceToDevice,
                                s.stream()) != cudaSuccess)
                rc = fail(RTM_ECUDA, "autotune snapshot copy failed");
        }
        if (rc == RTM_OK &&
            cudaMemcpyAsync(&snap_step[2 * k], s.d_step, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                            s.stream()) != cudaSuccess)
            rc = fail(RTM_ECUDA, "autotune step-counter snapshot failed");
    }
    if (rc == RTM_OK && c->comm) {
        cudaSetDevice(c->slabs[0].dev);
        if (cudaMalloc(&d_scratch, sizeof(double)) != cudaSuccess) rc = fail(RTM_ENOMEM, "scratch");
    }
    if (rc == RTM_OK) rc = sync_all(c);
    std::vector<double> times(ct.size(), std::nan(""));
    for (size_t k = 0; k < ct.size() && rc == RTM_OK; ++k) {  // selection phase
        c->tile = ct[k];
        c->zchunk = cz[k];
        invalidate_graphs(c);
        rc = timed_steps(c, nI, &times[k], d_scratch);
    }
    int best = -1;
    if (rc == RTM_OK) {
        best = rtm_select_mwmb(times.data(), 1, (int)times.size());  // times are already max over ranks
        if (best < 0) rc = fail(RTM_ECUDA, "no candidate could be timed");
    }
    double actual = 0;
    if (rc == RTM_OK) {  // verification phase
        c->tile = ct[best];
        c->zchunk = cz[best];
        invalidate_graphs(c);
        rc = timed_steps(c, nI, &actual, d_scratch);
    }
    // restore the wavefield and step counter (always, even on failure).  A peer context has
    // no all-reduce in the timed phases: meet at the barrier first, so no neighbour is still
    // stepping (pushing into / pulling from this slab) while it is restored.
    if (!c->comm && c->mode == 3 && rc == RTM_OK) rc = ranks_barrier(c);
    for (size_t k = 0; k < c->slabs.size(); ++k) {
        Slab& s = c->slabs[k];
        cudaSetDevice(s.dev);
        const size_t bytes = dplane(c) * s.buf_planes() * sizeof(float);
        for (int b = 0; b < 2; ++b)
            if (snap[2 * k + b])
                cudaMemcpyAsync(s.buf[b], snap[2 * k + b], bytes, cudaMemcpyDeviceToDevice, s.stream());
        cudaMemcpyAsync(s.d_step, &snap_step[2 * k], 2 * sizeof(int), cudaMemcpyHostToDevice, s.stream());
        cudaStreamSynchronize(s.stream());
    }
    c->step = saved_step;
    cleanup();
    if (c->halo_mode >= 2) {
        // The flag words hold g|(steps reached while tuning), beyond every later target g|n:
        // start a new generation so the waits order the slabs again.  Across ranks the restore
        // must also be complete everywhere before anyone pushes into a neighbour's halo: the
        // timed phases end in an all-reduce (all ranks' tuning steps done), and this barrier
        // orders every rank's restore before the next step of any rank.
        if (rc == RTM_OK) rc = ranks_barrier(c);
        ++c->sig_gen;
        c->sig_fresh = true;
    }
    if (rc != RTM_OK) {
        c->tile = saved_tile;
        c->zchunk = saved_zc;
        invalidate_graphs(c);
        return rc;
    }
    out->best_tile = ct[best];
    out->best_zchunk = cz[best];
    out->ncandidates = (int)ct.size();
    out->min_time_ms = times[best];
    out->actual_time_ms = actual;
    out->quality_pct = 100.0 * (actual - times[best]) / times[best];
    if (cand_ms)
        for (size_t k = 0; k < times.size(); ++k) cand_ms[k] = times[k];
    return RTM_OK;
}

int rtm_set_stream(rtm_ctx* c, void* stream) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (c->slabs.size() != 1)
        return fail(RTM_EINVAL, "rtm_set_stream needs a single-slab (single-GPU or distributed) context");
    Slab& s = c->slabs[0];
    DeviceGuard g;
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamSynchronize(s.stream()));
    s.has_user = stream != nullptr;
    s.s_user = static_cast<cudaStream_t>(stream);
    return RTM_OK;
}

float rtm_last_elapsed_ms(rtm_ctx* c) { return c ? c->last_ms : -1.0f; }

int rtm_set_profiling(rtm_ctx* c, int on) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    c->profiling = on != 0;
    c->prof_ms = 0;
    c->prof_launches = 0;
    c->prof_total_launches = 0;
    return RTM_OK;
}

int rtm_kernel_stats(rtm_ctx* c, long long* launches, double* total_ms) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (launches) *launches = c->prof_total_launches;
    if (total_ms) *total_ms = c->prof_ms;
    c->prof_total_launches = 0;
    c->prof_ms = 0;
    return RTM_OK;
}

long long rtm_launch_count(rtm_ctx* c) { return c ? c->launches : -1; }

int rtm_set_velocity_async(rtm_ctx* c, const float* v) {
    if (!c || !v) return fail(RTM_EINVAL, "NULL argument");
    DeviceGuard g;
    RET(async_setup(c, true, false));
    Slab& s = c->slabs[0];
    const size_t n = dplane(c) * s.nzl;
    cudaStream_t st = s.stream();
    if (!c->vcheck_pending) CK(cudaMemsetAsync(s.d_stats, 0, 2 * sizeof(unsigned int), st));
    CK(cudaStreamWaitEvent(c->s_h2d, c->ev_conv, 0));  // the previous conversion read v_stage
    RET(copy_planes(c, c->v_stage, v, s.nzl, true, cudaMemcpyHostToDevice, c->s_h2d));
    CK(cudaEventRecord(c->ev_h2d, c->s_h2d));
    CK(cudaStreamWaitEvent(st, c->ev_h2d, 0));  // C changes after the steps already enqueued
    CK(launch_velocity(c->v_stage, s.C, (long long)n, c->nx, c->px, (double)c->dt, (double)c->dx,
                       s.d_stats, st));
    CK(cudaEventRecord(c->ev_conv, st));
    c->vcheck_pending = true;
    c->vel_set = true;  // provisional: rtm_sync returns the verdict
    return RTM_OK;
}

int rtm_step_async(rtm_ctx* c, int nsteps) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    if (nsteps < 0) return fail(RTM_EINVAL, "nsteps must be >= 0");
    if (!c->vel_set) return fail(RTM_ESTATE, "rtm_step_async before a velocity was set");
    if (c->slabs.size() != 1) return fail(RTM_EINVAL, "the asynchronous calls need a single-slab context");
    if (c->check_every > 0 || c->profiling)
        return fail(RTM_ESTATE, "rtm_step_async with the field check or profiling on (use rtm_step)");
    DeviceGuard g;
    CK(cudaSetDevice(c->slabs[0].dev));
    c->prof_launches = 0;
    if (c->mode == 0) return step_single(c, nsteps);
    return step_slabs(c, nsteps);
}

int rtm_read_field_async(rtm_ctx* c, float* out) {
    if (!c || !out) return fail(RTM_EINVAL, "NULL argument");
    DeviceGuard g;
    RET(async_setup(c, false, true));
    Slab& s = c->slabs[0];
    const size_t n = hplane(c) * s.nzl, dpl = dplane(c);
    cudaStream_t st = s.stream();
    CK(cudaStreamWaitEvent(st, c->ev_d2h, 0));  // the previous D2H has read the snapshot
    for (int k = 0; k < s.nshots; ++k)  // unpadded snapshot of the interior
        RET(copy_planes(c, c->snap + (size_t)k * n, s.buf[c->step & 1] + ((size_t)k * (s.nzl + 10) + 5) * dpl,
                        s.nzl, false, cudaMemcpyDeviceToDevice, st));
    CK(cudaEventRecord(c->ev_snap, st));
    CK(cudaStreamWaitEvent(c->s_copy, c->ev_snap, 0));
    CK(cudaMemcpyAsync(out, c->snap, n * s.nshots * sizeof(float), cudaMemcpyDeviceToHost, c->s_copy));
    CK(cudaEventRecord(c->ev_d2h, c->s_copy));
    return RTM_OK;
}

int rtm_sync(rtm_ctx* c) {
    if (!c) return fail(RTM_EINVAL, "ctx is NULL");
    DeviceGuard g;
    Slab& s = c->slabs[0];
    CK(cudaSetDevice(s.dev));
    if (c->s_copy) {  // the context's stream ends after the last asynchronous copies
        CK(cudaEventRecord(c->ev_d2h, c->s_copy));
        CK(cudaStreamWaitEvent(s.stream(), c->ev_d2h, 0));
        CK(cudaEventRecord(c->ev_h2d, c->s_h2d));
        CK(cudaStreamWaitEvent(s.stream(), c->ev_h2d, 0));
    }
    RET(sync_all(c));
    if (c->s_copy) {
        CK(cudaStreamSynchronize(c->s_copy));
        CK(cudaStreamSynchronize(c->s_h2d));
    }
    return async_vcheck(c);
}

}  // extern "C"
