// Device helpers shared by the stencil kernels (rtm_kernels.cu, rtm_tb.cu): the per-point
// update (ONE arithmetic expression for every kernel, so all variants are bitwise identical),
// mbarrier / TMA / cache-policy PTX wrappers, and the fused source epilogue.
#pragma once
#include "rtm_internal.h"

#include <type_traits>

namespace rtm {

// ------------------------------------------------------------------------------------
// The per-point update.  z[k], y[k], x[k] are u at offsets k-5 along each axis (index 5 is
// the point itself, shared by all three).  ONE expression for every kernel, so all
// variants are bitwise identical.  Order: centre * 3c0, then z, y, x pairs from the
// nearest to the farthest offset, then the leapfrog.
__device__ __forceinline__ float rtm_point(const float (&z)[11], const float (&y)[11],
                                           const float (&x)[11], float up, float C,
                                           const float (&c)[6]) {
    float acc = __fmul_rn(c[0], z[5]);
#pragma unroll
    for (int m = 1; m <= 5; ++m) acc = __fmaf_rn(c[m], __fadd_rn(z[5 - m], z[5 + m]), acc);
#pragma unroll
    for (int m = 1; m <= 5; ++m) acc = __fmaf_rn(c[m], __fadd_rn(y[5 - m], y[5 + m]), acc);
#pragma unroll
    for (int m = 1; m <= 5; ++m) acc = __fmaf_rn(c[m], __fadd_rn(x[5 - m], x[5 + m]), acc);
    return __fmaf_rn(C, acc, __fmaf_rn(2.0f, z[5], -up));
}

// The same expression for two x-adjacent points at once with Blackwell's packed fp32x2
// instructions (FFMA2/FADD2/FMUL2: one issue slot for two lanes).  Each lane performs exactly
// rtm_point's IEEE operations in rtm_point's order, so results are bitwise identical.  The x
// pair sums c_m * (x[-m] + x[+m]) are passed in precomputed (xsum[m-1]).
__device__ __forceinline__ float2 rtm_point2(const float2 (&z)[11], const float2 (&y)[11],
                                             const float2 (&xsum)[5], float2 up, float2 C,
                                             const float (&c)[6]) {
    float2 acc = __fmul2_rn(make_float2(c[0], c[0]), z[5]);
#pragma unroll
    for (int m = 1; m <= 5; ++m)
        acc = __ffma2_rn(make_float2(c[m], c[m]), __fadd2_rn(z[5 - m], z[5 + m]), acc);
#pragma unroll
    for (int m = 1; m <= 5; ++m)
        acc = __ffma2_rn(make_float2(c[m], c[m]), __fadd2_rn(y[5 - m], y[5 + m]), acc);
#pragma unroll
    for (int m = 1; m <= 5; ++m) acc = __ffma2_rn(make_float2(c[m], c[m]), xsum[m - 1], acc);
    const float2 lf = __ffma2_rn(make_float2(2.0f, 2.0f), z[5], make_float2(-up.x, -up.y));
    return __ffma2_rn(C, acc, lf);
}
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }

// ------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ float4 ld_stream4(const float* p) {  // read-once stream, evict-first
    return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_stream4(float* p, float4 v) {
    __stcs(reinterpret_cast<float4*>(p), v);
}
__device__ __forceinline__ float comp(const float4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Fused halo push: mirror a finished boundary-plane value into the neighbour slab's z-halo.
__device__ __forceinline__ void push_halo4(const StencilParams& p, int z, long long col, float4 v) {
    if (z < 5 && p.push_lo) st_stream4(p.push_lo + (long long)z * p.plane + col, v);
    if (z >= p.nzl - 5 && p.push_hi) st_stream4(p.push_hi + (long long)(z - p.nzl + 5) * p.plane + col, v);
}

// Add the samples of the sources owned by this thread's 4-point column at plane z.  step()
// returns the global index of the step being computed (sample n is added after the stencil of
// step n); it is evaluated only when a source lies in plane z — a device-counter read must not
// stall the owning warp on every plane (it would throttle the whole CTA pipeline).
template <class StepFn>
__device__ __forceinline__ void add_sources_f(const StencilParams& p, uint64_t mask, int x, int z,
                                              StepFn step, float (&out)[4]) {
    while (mask) {
        const int s = __ffsll(static_cast<long long>(mask)) - 1;
        mask &= mask - 1;
        const DevSource& src = p.src[s];
        if (src.z == z) {
            const int n = step();
            if (n < src.nsamples) {
                const float w = p.samples[src.offset + n];
                const int i = src.x - x;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k == i) out[k] = __fadd_rn(out[k], w);
            }
        }
    }
}
// ... n known (multi-step launches: step0 + k)
__device__ __forceinline__ void add_sources_n(const StencilParams& p, uint64_t mask, int x, int z,
                                              int n, float (&out)[4]) {
    add_sources_f(p, mask, x, z, [n]() { return n; }, out);
}
// ... n from the device step counter (graph-replayable launches)
__device__ __forceinline__ void add_sources(const StencilParams& p, uint64_t mask, int x, int z,
                                            float (&out)[4]) {
    add_sources_f(p, mask, x, z,
                  [&p]() { return *reinterpret_cast<volatile const int*>(&p.d_step[p.parity]); }, out);
}

// ---- gpu-scope acquire / release, proxy fence, watchdog (inter-CTA flags) ------------------
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr unsigned long long kWatchdogNs = 4000000000ull;

__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t addr) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
// Run f(integral_constant<O>), f(<O+1>), ... f(<U-1>) while iterations remain; false when the
// unit ended inside the unrolled group.
template <int O, int U, class F>
__device__ __forceinline__ bool unrolled(F& f, int i, int n) {
    f(std::integral_constant<int, O>{});
    if constexpr (O + 1 < U) {
        if (i + O + 1 >= n) return false;
        return unrolled<O + 1, U>(f, i, n);
    }
    return true;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// cache_mode (StencilParams): bits 0-1 L2 prefetch of u_prev/C (0 none, 1 evict_last,
// 2 evict_normal); bit 2 u TMA loads with an evict_last L2 policy; bit 3 plain (not
// evict-first) u_prev/C loads and u_next stores; bits 4-7 prefetch distance in planes;
// bits 8-9 L2 promotion of the u box (host side); bit 10 u_prev/C TMA loads evict_first;
// bit 11 C TMA loads evict_last (C kept in L2 across steps where it fits).
__device__ __forceinline__ void prefetch_l2(const void* p, int mode) {
    if (mode == 1)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
    else if (mode == 2)
        asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(p));
}
__device__ __forceinline__ float4 ld_mode4(const float* p, bool plain) {
    return plain ? __ldcg(reinterpret_cast<const float4*>(p)) : ld_stream4(p);
}
__device__ __forceinline__ void st_mode4(float* p, float4 v, bool plain) {
    if (plain)
        __stcg(reinterpret_cast<float4*>(p), v);
    else
        st_stream4(p, v);
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* tm, int x, int y,
                                                 int z, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Rows are pitched to a multiple of 4 floats; the padding columns x >= nx must stay zero (they
// are the Dirichlet x-halo for every load that reaches them), so a 4-point group that straddles
// nx stores zeros in its padding lanes.
__device__ __forceinline__ void zero_pad(float (&out)[4], int x, int nx) {
    if (x + 4 > nx) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (x + k >= nx) out[k] = 0.0f;
    }
}

// The k_stream per-thread update of 4 x-consecutive points, split into the operand gather
// (from shared memory in k_stream / k_tb2s, from L2 in k_resident) and ONE arithmetic core, so
// every kernel performs the same operations in the same order (bitwise-identical results).
// q[O + k] = u at z offset k - 5 (register queue); yv[5 +- m] = u at y offset +-m (yv[5] =
// q[O + 5]); xs[0..13] = u at x offsets -5 .. +8 of the first point; upv/cv = u_prev and C.
template <int O, int N>
__device__ __forceinline__ void star4_core(const float4 (&q)[N], const float4 (&yv)[11],
                                           const float (&xs)[14], float4 upv, float4 cv,
                                           const float (&c)[6], float (&out)[4]) {
    const float4 L4 = make_float4(xs[1], xs[2], xs[3], xs[4]);
    const float4 R4 = make_float4(xs[9], xs[10], xs[11], xs[12]);
    float2 xa[5], xb[5];
    xa[0] = make_float2(__fadd_rn(xs[4], xs[6]), __fadd_rn(xs[5], xs[7]));
    xa[1] = __fadd2_rn(hi2(L4), hi2(q[O + 5]));
    xa[2] = make_float2(__fadd_rn(xs[2], xs[8]), __fadd_rn(xs[3], xs[9]));
    xa[3] = __fadd2_rn(lo2(L4), lo2(R4));
    xa[4] = make_float2(__fadd_rn(xs[0], xs[10]), __fadd_rn(xs[1], xs[11]));
    xb[0] = make_float2(__fadd_rn(xs[6], xs[8]), __fadd_rn(xs[7], xs[9]));
    xb[1] = __fadd2_rn(lo2(q[O + 5]), lo2(R4));
    xb[2] = make_float2(__fadd_rn(xs[4], xs[10]), __fadd_rn(xs[5], xs[11]));
    xb[3] = __fadd2_rn(hi2(L4), hi2(R4));
    xb[4] = make_float2(__fadd_rn(xs[2], xs[12]), __fadd_rn(xs[3], xs[13]));
    float2 za[11], zb[11], ya[11], yb[11];
#pragma unroll
    for (int o = 0; o < 11; ++o) {
        za[o] = lo2(q[O + o]);
        zb[o] = hi2(q[O + o]);
        ya[o] = lo2(yv[o]);
        yb[o] = hi2(yv[o]);
    }
    const float2 ra = rtm_point2(za, ya, xa, lo2(upv), lo2(cv), c);
    const float2 rb = rtm_point2(zb, yb, xb, hi2(upv), hi2(cv), c);
    out[0] = ra.x; out[1] = ra.y; out[2] = rb.x; out[3] = rb.y;
}

// Operands from a staged plane: `row` points at the thread's own 4 points in the (RS-float
// rows, 5-row y halo, 8-float x halo) shared-memory copy of the centre plane.
template <int RS, int O, int N>
__device__ __forceinline__ void star4(const float* row, const float4 (&q)[N], float4 upv, float4 cv,
                                      const float (&c)[6], float (&out)[4]) {
    float xs[14];
    {
        const float4 l = *reinterpret_cast<const float4*>(row - 4);
        const float4 rr = *reinterpret_cast<const float4*>(row + 4);
        xs[0] = row[-5];
        xs[1] = l.x; xs[2] = l.y; xs[3] = l.z; xs[4] = l.w;
        xs[5] = q[O + 5].x; xs[6] = q[O + 5].y; xs[7] = q[O + 5].z; xs[8] = q[O + 5].w;
        xs[9] = rr.x; xs[10] = rr.y; xs[11] = rr.z; xs[12] = rr.w;
        xs[13] = row[8];
    }
    float4 yv[11];
#pragma unroll
    for (int m = 1; m <= 5; ++m) {
        yv[5 - m] = *reinterpret_cast<const float4*>(row - m * RS);
        yv[5 + m] = *reinterpret_cast<const float4*>(row + m * RS);
    }
    yv[5] = q[O + 5];
    star4_core<O>(q, yv, xs, upv, cv, c, out);
}

// ---- work units of the persistent streaming kernels (k_stream, k_stream2) ----------------
struct UnitGeom {
    int x0, y0, zs, ze;
    int shot;
    long long soff;  // buffer-plane offset of the shot: shot * (nzl + 10)
};
// unit = ((chunk * ntiles) + tile) * nshots + shot: shots fastest (concurrent CTAs share the
// C tile through L2), then tiles (co-running xy neighbours share halos), then z-chunks.
__device__ __forceinline__ UnitGeom unit_geom(const StencilParams& p, int unit, int TX, int TY) {
    const int ntiles = p.tiles_x * p.tiles_y;
    int shot;
    if (p.shot_major) {
        const int per_shot = ntiles * (p.r_chunks[0] + (p.nranges > 1 ? p.r_chunks[1] : 0));
        shot = unit / per_shot;
        unit -= shot * per_shot;
    } else {
        shot = unit % p.nshots;
        unit /= p.nshots;
    }
    int chunk = unit / ntiles;
    const int tile = unit - chunk * ntiles;
    int r = 0;
    if (chunk >= p.r_chunks[0]) {
        r = 1;
        chunk -= p.r_chunks[0];
    }
    UnitGeom g;
    g.zs = p.r_begin[r] + static_cast<int>((long long)chunk * p.r_len[r] / p.r_chunks[r]);
    g.ze = p.r_begin[r] + static_cast<int>((long long)(chunk + 1) * p.r_len[r] / p.r_chunks[r]);
    const int tyi = tile / p.tiles_x;
    g.x0 = (tile - tyi * p.tiles_x) * TX;
    g.y0 = tyi * TY;
    g.shot = shot;
    g.soff = (long long)shot * (p.nzl + 10);
    return g;
}

// z sweep direction of a unit (RTM_OPT_ZDIR bits): bit 0 — downward on odd-parity steps (a step
// starts where the previous one ended); bit 1 — downward on every other unit of a CTA (wave w + 1
// starts where wave w ended, so the halo rows its boxes share with wave w's tiles are still in
// L2).  Every unit is computed identically either way (bitwise).
__device__ __forceinline__ bool sweep_down(const StencilParams& p, int step_parity, int unit) {
    int d = 0;
    if (p.zalt & 1) d ^= step_parity & 1;
    if (p.zalt & 2) d ^= ((unit - (int)blockIdx.x) / (int)gridDim.x) & 1;
    if (p.zalt & 4) {  // odd z-chunks sweep downward: neighbouring chunks start and end on the
                       // planes they share, so each z-halo plane is read by both at the same time
        const int ntiles = p.tiles_x * p.tiles_y;
        const int per_shot = ntiles * (p.r_chunks[0] + (p.nranges > 1 ? p.r_chunks[1] : 0));
        const int u = p.shot_major ? unit % per_shot : unit / p.nshots;
        d ^= (u / ntiles) & 1;
    }
    return d != 0;
}

}  // namespace rtm
