// =====================================================================================
// sm_100a kernels of the RTM 3D-model step (arxiv 1310.8232, §2
// Algorithm 1 "calculate 3D model"): radius-5 31-point star, 2nd-order leapfrog, fused
// point-source injection.
//
//   k_tiled  (K1/K2/K3): one CTA per (xy tile, z-chunk) work unit.  The u planes of the
//            tile plus a 5-cell x/y halo are staged into a K-deep shared-memory ring by TMA
//            (cp.async.bulk.tensor.3d, OOB zero fill = the x/y Dirichlet halo), completion
//            tracked by one mbarrier per slot.  Each thread owns 4 consecutive x points
//            (128-bit accesses) of one row and streams along z with an 11-plane register
//            queue; y/x neighbours come from the staged plane.  u_prev and C are streamed
//            with 128-bit loads one plane ahead; u_next is stored in place over u_prev.
//            Sources registered on the slab are added in the epilogue (fused a3).
//   k_naive  (K5): one thread per point, global loads; same per-point expression, so its
//            output is bitwise identical to k_tiled's.
//   k_velocity (a1): C(p) = fp32((double(v)*dt/dx)^2) + max|v| and validity for the CFL check.
//
// The blocked traversal replaces the paper's CPU cache blocking (the
// (b_i, b_j, b_k) blocksize) by an xy tile streamed along z; see DESIGN.md §Kernels.
// =====================================================================================
#include "rtm_internal.h"
#include "rtm_device.cuh"

#include <cstdio>
#include <type_traits>

// 1 (default): single-step k_stream reads the 5 leading z-halo planes of a unit (only the z
// register queue uses them) with 128-bit global loads of the thread's own points instead of
// halo'd TMA boxes through the ring; 0: all planes through the ring (round-2 A/B:
// profiles/ldgq_ab_r02.log, C2 -0.4..-1.4 %, C3 -0.7 %, C4 -0.5 %, bitwise identical)
#ifndef RTM_LDGQ
#define RTM_LDGQ 1
#endif

namespace rtm {

// ------------------------------------------------------------------------------------
template <int TX, int TY, int K>
struct TiledShape {
    static constexpr int NT = TX * TY / 4;     // threads per CTA
    static constexpr int TXV = TX / 4;         // threads per tile row
    static constexpr int RS = TX + 16;         // staged row: x0-8 .. x0+TX+7 (16B aligned)
    static constexpr int ROWS = TY + 10;       // y0-5 .. y0+TY+4
    static constexpr int BOX_FLOATS = RS * ROWS;
    static constexpr int SLOT = (BOX_FLOATS + 31) / 32 * 32;  // 128-byte aligned slots
    static constexpr uint32_t BOX_BYTES = BOX_FLOATS * 4;
    static constexpr size_t SMEM = size_t(K) * SLOT * 4 + size_t(K) * 8;
    static_assert(TX % 4 == 0 && RS <= 256 && ROWS <= 256, "TMA box limits");
    static_assert(K >= 10, "ring must hold the 10 prologue planes");
};

template <int TX, int TY, int K, int MINB>
__global__ void __launch_bounds__(TX * TY / 4, MINB)
    k_tiled(const __grid_constant__ CUtensorMap tm, const __grid_constant__ StencilParams p) {
    using S = TiledShape<TX, TY, K>;
    extern __shared__ __align__(128) float smem[];
    float* ring = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + K * S::SLOT);

    const int tid = threadIdx.x;
    const int tx = tid % S::TXV, ty = tid / S::TXV;

    // ---- work unit: (z-chunk, tile), chunk-major so concurrently running CTAs are xy
    // neighbours at similar z (their halo re-reads hit L2)
    const int nunits_shot = p.tiles_x * p.tiles_y * (p.r_chunks[0] + (p.nranges > 1 ? p.r_chunks[1] : 0));
    const int shot = p.shot_major ? (int)(blockIdx.x / nunits_shot) : (int)(blockIdx.x % p.nshots);
    const int ublk = p.shot_major ? (int)(blockIdx.x - shot * nunits_shot) : (int)(blockIdx.x / p.nshots);
    const long long soff = (long long)shot * (p.nzl + 10);
    const int ntiles = p.tiles_x * p.tiles_y;
    int chunk = ublk / ntiles;
    const int tile = ublk - chunk * ntiles;
    int r = 0;
    if (chunk >= p.r_chunks[0]) {
        r = 1;
        chunk -= p.r_chunks[0];
    }
    const int zs = p.r_begin[r] + static_cast<int>((long long)chunk * p.r_len[r] / p.r_chunks[r]);
    const int ze = p.r_begin[r] + static_cast<int>((long long)(chunk + 1) * p.r_len[r] / p.r_chunks[r]);
    const int tyi = tile / p.tiles_x;
    const int x0 = (tile - tyi * p.tiles_x) * TX;
    const int y0 = tyi * TY;
    const int x = x0 + 4 * tx;
    const int y = y0 + ty;
    const bool active = (x < p.nx) && (y < p.ny);

    if (tid == 0) {
#pragma unroll 1
        for (int k = 0; k < K; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
    }
    __syncthreads();

    // plane j of this unit = owned plane zs-5+j = buffer plane zs+j
    const int L = ze - zs + 10;
    auto issue = [&](int j) {
        const int slot = j % K;
        mbar_expect_tx(&bars[slot], S::BOX_BYTES);
        tma_load_3d(ring + slot * S::SLOT, &tm, x0 - 8, y0 - 5, (int)soff + zs + j, &bars[slot]);
    };
    if (tid == 0) {
        const int first = L < K ? L : K;
#pragma unroll 1
        for (int j = 0; j < first; ++j) issue(j);
    }

    // sources in this thread's column within the unit (registration order = bit order)
    uint64_t smask = 0;
    if (active) {
#pragma unroll 1
        for (int s = 0; s < p.nsrc; ++s) {
            const DevSource& src = p.src[s];
            if (src.shot == shot && src.y == y && src.x >= x && src.x < x + 4 && src.z >= zs &&
                src.z < ze)
                smask |= (1ull << s);
        }
    }
    if (p.write_next && blockIdx.x == 0 && tid == 0)
        p.d_step[p.parity ^ 1] = p.d_step[p.parity] + 1;

    const int own = (5 + ty) * S::RS + 8 + 4 * tx;
    const long long col = (long long)y * p.pitch + x;

    // ---- prologue: queue <- planes zs-5 .. zs+4
    float4 q[11];
#pragma unroll
    for (int j = 0; j < 10; ++j) {
        mbar_wait(&bars[j % K], (j / K) & 1);
        q[j] = *reinterpret_cast<const float4*>(ring + (j % K) * S::SLOT + own);
    }
    __syncthreads();  // planes zs-5 .. zs-1 fully consumed
    if (tid == 0) {
        fence_proxy_async();
#pragma unroll 1
        for (int j = 0; j < 5; ++j)
            if (j + K < L) issue(j + K);
    }

    float4 upv = make_float4(0.f, 0.f, 0.f, 0.f), cv = upv;
    if (active) {
        upv = ld_stream4(p.next + (soff + zs + 5) * p.plane + col);
        cv = ld_stream4(p.C + (long long)zs * p.plane + col);
    }
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};

#pragma unroll 1
    for (int z = zs; z < ze; ++z) {
        const int i = z - zs;
        float4 upn = upv, cn = cv;
        if (active && z + 1 < ze) {  // one plane ahead
            upn = ld_stream4(p.next + (soff + z + 6) * p.plane + col);
            cn = ld_stream4(p.C + (long long)(z + 1) * p.plane + col);
        }
        const int jn = i + 10, jc = i + 5;
        mbar_wait(&bars[jn % K], (jn / K) & 1);
        q[10] = *reinterpret_cast<const float4*>(ring + (jn % K) * S::SLOT + own);

        const float* row = ring + (jc % K) * S::SLOT + own;
        float xs[14];
        {
            const float4 l = *reinterpret_cast<const float4*>(row - 4);
            const float4 rr = *reinterpret_cast<const float4*>(row + 4);
            xs[0] = row[-5];
            xs[1] = l.x; xs[2] = l.y; xs[3] = l.z; xs[4] = l.w;
            xs[5] = q[5].x; xs[6] = q[5].y; xs[7] = q[5].z; xs[8] = q[5].w;
            xs[9] = rr.x; xs[10] = rr.y; xs[11] = rr.z; xs[12] = rr.w;
            xs[13] = row[8];
        }
        float4 yv[11];
#pragma unroll
        for (int m = 1; m <= 5; ++m) {
            yv[5 - m] = *reinterpret_cast<const float4*>(row - m * S::RS);
            yv[5 + m] = *reinterpret_cast<const float4*>(row + m * S::RS);
        }
        yv[5] = q[5];

        float out[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float zl[11], yl[11], xl[11];
#pragma unroll
            for (int o = 0; o < 11; ++o) {
                zl[o] = comp(q[o], k);
                yl[o] = comp(yv[o], k);
                xl[o] = xs[k + o];
            }
            out[k] = rtm_point(zl, yl, xl, comp(upv, k), comp(cv, k), c);
        }
        if (smask) add_sources(p, smask, x, z, out);
        if (active) {
            zero_pad(out, x, p.nx);
            const float4 o4 = make_float4(out[0], out[1], out[2], out[3]);
            st_stream4(p.next + (soff + z + 5) * p.plane + col, o4);
            push_halo4(p, z, col, o4);
        }

#pragma unroll
        for (int o = 0; o < 10; ++o) q[o] = q[o + 1];
        upv = upn;
        cv = cn;
        __syncthreads();  // plane jc fully consumed -> its slot takes plane jc + K
        if (tid == 0 && jc + K < L) {
            fence_proxy_async();
            issue(jc + K);
        }
    }
}

// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_naive(const __grid_constant__ StencilParams p) {
    long long per_shot = (long long)p.r_len[0] * p.plane;
    if (p.nranges > 1) per_shot += (long long)p.r_len[1] * p.plane;
    const long long total = per_shot * p.nshots;
    if (p.write_next && blockIdx.x == 0 && threadIdx.x == 0)
        p.d_step[p.parity ^ 1] = p.d_step[p.parity] + 1;
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int shot = static_cast<int>(t / per_shot);
        long long tt = t - shot * per_shot;
        int z;
        const long long n0 = (long long)p.r_len[0] * p.plane;
        if (tt < n0) {
            z = p.r_begin[0] + static_cast<int>(tt / p.plane);
        } else {
            tt -= n0;
            z = p.r_begin[1] + static_cast<int>(tt / p.plane);
        }
        const long long inplane = tt % p.plane;
        const int y = static_cast<int>(inplane / p.pitch);
        const int x = static_cast<int>(inplane - (long long)y * p.pitch);
        if (x >= p.nx) continue;  // padding column: stays zero
        const long long pb = ((long long)shot * (p.nzl + 10) + z + 5) * p.plane + inplane;  // buffer index
        float zl[11], yl[11], xl[11];
#pragma unroll
        for (int o = -5; o <= 5; ++o) {
            zl[o + 5] = p.u[pb + o * p.plane];  // z-halo planes are explicit
            const int yy = y + o, xx = x + o;
            yl[o + 5] = (yy >= 0 && yy < p.ny) ? p.u[pb + (long long)o * p.pitch] : 0.0f;
            xl[o + 5] = (xx >= 0 && xx < p.nx) ? p.u[pb + o] : 0.0f;
        }
        float out = rtm_point(zl, yl, xl, p.next[pb], p.C[(long long)z * p.plane + inplane], c);
        for (int s = 0; s < p.nsrc; ++s) {
            const DevSource& src = p.src[s];
            if (src.x == x && src.y == y && src.z == z && src.shot == shot) {
                const int n = p.d_step[p.parity];
                if (n < src.nsamples) out = __fadd_rn(out, p.samples[src.offset + n]);
            }
        }
        p.next[pb] = out;
        if (z < 5 && p.push_lo) p.push_lo[(long long)z * p.plane + inplane] = out;
        if (z >= p.nzl - 5 && p.push_hi) p.push_hi[(long long)(z - p.nzl + 5) * p.plane + inplane] = out;
    }
}

// ------------------------------------------------------------------------------------
__device__ __forceinline__ float c_of_v(float vi, double dt, double dx, float& vmax, unsigned& bad) {
    if (!(isfinite(vi) && vi > 0.0f))
        ++bad;
    else
        vmax = fmaxf(vmax, vi);
    // (double(v) * double(dt)) / double(dx), squared, rounded once to fp32 (a1)
    const double nu = __ddiv_rn(__dmul_rn(static_cast<double>(vi), dt), dx);
    return __double2float_rn(__dmul_rn(nu, nu));
}

// vec4: n % 4 == 0 and 16-byte aligned pointers -> 128-bit loads/stores, 4 independent
// fp64 chains per thread (the scalar form was latency-bound at ~2 TB/s).  Padding columns
// (x = i mod pitch >= nx) get C = 0 and stay out of the statistics.
__global__ void __launch_bounds__(256) k_velocity(const float* v, float* C, long long n, int nx,
                                                  int pitch, double dt, double dx,
                                                  unsigned int* stats, int vec4) {
    float vmax = 0.0f;
    unsigned int bad = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (vec4) {
        const float4* v4 = reinterpret_cast<const float4*>(v);
        float4* c4 = reinterpret_cast<float4*>(C);
        for (long long i = t0; i < n / 4; i += stride) {
            const float4 a = __ldcs(v4 + i);
            float4 r;
            const int x = static_cast<int>((4 * i) % pitch);
            if (x + 4 <= nx) {
                r.x = c_of_v(a.x, dt, dx, vmax, bad);
                r.y = c_of_v(a.y, dt, dx, vmax, bad);
                r.z = c_of_v(a.z, dt, dx, vmax, bad);
                r.w = c_of_v(a.w, dt, dx, vmax, bad);
            } else {  // the group holding the last columns and the padding
                float o[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = x + k < nx ? c_of_v(o[k], dt, dx, vmax, bad) : 0.0f;
                r = make_float4(o[0], o[1], o[2], o[3]);
            }
            c4[i] = r;
        }
    } else {
        for (long long i = t0; i < n; i += stride)
            C[i] = (int)(i % pitch) < nx ? c_of_v(v[i], dt, dx, vmax, bad) : 0.0f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&stats[0], __float_as_uint(vmax));  // v > 0: uint order == float order
        if (bad) atomicAdd(&stats[1], bad);
    }
}

// ------------------------------------------------------------------------------------
// k_stream: warp-specialised persistent version of k_tiled.  One producer warp streams,
// unit after unit, the halo'd u planes (TMA, K-slot ring) and — when D > 0 — the u_prev and
// C tiles (TMA, D-slot ring) into shared memory; NW consumer warps compute.  Slots are
// handed over with full/empty mbarriers only (no CTA-wide barrier in the loop), so each
// consumer warp runs ahead as far as the data allows and the producer prefetches across
// unit boundaries.  Work units are (z-chunk, tile) pairs, chunk-major, dealt round-robin
// to the persistent CTAs (unit = blockIdx.x + k * gridDim.x) so co-running CTAs are xy
// neighbours at similar z.
template <int TX, int TY, int K, int D, int U = 4>
struct StreamShape {
    // U == 11: modulo-scheduled z queue (q[11], register names rotate with the unrolled
    // iteration, no copies at the loop back-edge) and per-lane empty-slot arrivals (no warp
    // sync / elected-lane branch per plane): the empty barriers count every consumer lane
    static constexpr bool MQ = (U == 11);
    static constexpr int NW = TX * TY / 128;      // consumer warps (4 points per thread)
    static constexpr int EMPTY_COUNT = MQ ? NW * 32 : NW;
    static constexpr int NT = NW * 32 + 32;       // + 1 producer warp
    static constexpr int TXV = TX / 4;
    static constexpr int RS = TX + 16;
    static constexpr int ROWS = TY + 10;
    static constexpr int USLOT = (RS * ROWS + 31) / 32 * 32;
    static constexpr uint32_t UBYTES = RS * ROWS * 4;
    static constexpr int CSLOT = 2 * TX * TY;     // u_prev tile then C tile
    static constexpr uint32_t CBYTES = CSLOT * 4;
    static constexpr size_t BAR_OFF = (size_t(K) * USLOT + size_t(D) * CSLOT) * 4;
    static constexpr size_t SMEM = BAR_OFF + size_t(2 * K + 2 * D) * 8;
    static_assert((TX * TY) % 128 == 0, "whole consumer warps");
    static_assert(K >= 7, "6 live planes + 1 in flight");
    static_assert(TX % 4 == 0 && RS <= 256 && ROWS <= 256 && TX <= 256 && TY <= 256, "TMA box");
};

// Multi-step launches (MS): the unit index of (shot, chunk, tile) — the inverse of unit_geom.
__device__ __forceinline__ int unit_index(const StencilParams& p, int shot, int chunk, int tile) {
    const int ntiles = p.tiles_x * p.tiles_y;
    if (p.shot_major) return shot * ntiles * p.r_chunks[0] + chunk * ntiles + tile;
    return (chunk * ntiles + tile) * p.nshots + shot;
}
// Spin (acquire, gpu scope) until flags[unit] and the flags of its face neighbours (x +- 1,
// y +- 1 tiles of the same chunk; chunks +- 1 of the same tile; same shot) reach target, i.e.
// until every unit whose u^{n+1} planes this unit's box reads has stored them (RAW) and has
// finished reading the u^{n-1} planes this unit overwrites (WAR).  Then order the following
// TMA (async-proxy) loads after the acquired generic-proxy stores.  4 s watchdog -> trap.
__device__ __noinline__ void wait_unit_flags(const StencilParams& p, int unit, unsigned long long target) {
    const int ntiles = p.tiles_x * p.tiles_y;
    int shot, rest;
    if (p.shot_major) {
        const int per_shot = ntiles * p.r_chunks[0];
        shot = unit / per_shot;
        rest = unit - shot * per_shot;
    } else {
        shot = unit % p.nshots;
        rest = unit / p.nshots;
    }
    const int chunk = rest / ntiles, tile = rest - chunk * ntiles;
    const int ty = tile / p.tiles_x, tx = tile - ty * p.tiles_x;
    // chunk c covers planes [zb(c), zb(c+1)); its u boxes read planes [zb(c) - 5, zb(c+1) + 5), so
    // every chunk of the same tile that intersects that range is a z-neighbour (more than one on
    // each side when chunks are shorter than the 5-plane halo)
    auto zb = [&](int c2) {
        return p.r_begin[0] + static_cast<int>((long long)c2 * p.r_len[0] / p.r_chunks[0]);
    };
    const int lo = zb(chunk) - RADIUS, hi = zb(chunk + 1) + RADIUS;
    auto check = [&](int v, unsigned long long t0) {
        const unsigned long long* f = p.flags + v;
        if (ld_acquire_gpu_u64(f) >= target) return;
        unsigned spins = 0;
        while (ld_acquire_gpu_u64(f) < target) {
            __nanosleep(64);
            if ((++spins & 255) == 0 && globaltimer_ns() - t0 > kWatchdogNs) __trap();
        }
    };
    const unsigned long long t0 = globaltimer_ns();
    check(unit, t0);
    if (tx > 0) check(unit_index(p, shot, chunk, tile - 1), t0);
    if (tx + 1 < p.tiles_x) check(unit_index(p, shot, chunk, tile + 1), t0);
    if (ty > 0) check(unit_index(p, shot, chunk, tile - p.tiles_x), t0);
    if (ty + 1 < p.tiles_y) check(unit_index(p, shot, chunk, tile + p.tiles_x), t0);
    for (int c2 = chunk - 1; c2 >= 0 && zb(c2 + 1) > lo; --c2) check(unit_index(p, shot, c2, tile), t0);
    for (int c2 = chunk + 1; c2 < p.r_chunks[0] && zb(c2) < hi; ++c2) check(unit_index(p, shot, c2, tile), t0);
    fence_proxy_async_global();
}

template <int TX, int TY, int K, int D, int MINB, int U, bool MS>
__global__ void __launch_bounds__(StreamShape<TX, TY, K, D, U>::NT, MINB)
    k_stream(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_up,
             const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ StencilParams p,
             const __grid_constant__ CUtensorMap tm_u2, const __grid_constant__ CUtensorMap tm_up2) {
    using S = StreamShape<TX, TY, K, D, U>;
    constexpr bool MQ = S::MQ;
    // queue slot of z offset k - 5 in unrolled iteration O
    constexpr auto QI = [](int O, int k) constexpr { return MQ ? (O + k) % 11 : O + k; };
    // z-halo planes at the start of a unit that bypass the ring (consumer global loads); only
    // in single-step launches, where the u buffer is read-only for the whole kernel
    constexpr int QS = (RTM_LDGQ && !MS) ? 5 : 0;
    extern __shared__ __align__(128) float smem[];
    float* uring = smem;
    float* cring = smem + K * S::USLOT;
    uint64_t* full_u = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + S::BAR_OFF);
    uint64_t* empty_u = full_u + K;
    uint64_t* full_c = empty_u + K;
    uint64_t* empty_c = full_c + D;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < K; ++k) {
            mbar_init(&full_u[k], 1);
            mbar_init(&empty_u[k], S::EMPTY_COUNT);
        }
        for (int k = 0; k < D; ++k) {
            mbar_init(&full_c[k], 1);
            mbar_init(&empty_c[k], S::EMPTY_COUNT);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // Programmatic dependent launch: everything above overlapped the previous grid's tail;
    // every global access below depends on it (u, u_prev, the step counter), so wait for its
    // completion here (a no-op for a normal launch), then let the next grid be scheduled.
    // (The producer lane first issues the u_prev / C tiles of its first unit: under PDL they do
    // not depend on the previous grid — u^{n-1} was its input, not its output — so their loads
    // overlap the previous step's tail; it waits right after.)
    if (!(warp == S::NW && lane == 0)) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if constexpr (MS) {
        // the step counter after the launch (nothing in this launch reads it: step0 + k)
        if (blockIdx.x == 0 && tid == 0) {
            p.d_step[(p.parity + p.nsteps) & 1] = p.step0 + p.nsteps;
            p.d_step[(p.parity + p.nsteps + 1) & 1] = p.step0 + p.nsteps - 1;
        }
    } else {
        if (p.write_next && blockIdx.x == 0 && tid == 0)
            p.d_step[p.parity ^ 1] = p.d_step[p.parity] + 1;
    }

    const int units = p.tiles_x * p.tiles_y * (p.r_chunks[0] + (p.nranges > 1 ? p.r_chunks[1] : 0)) *
                      p.nshots;
    const int nst = MS ? p.nsteps : 1;

    if (warp == S::NW) {  // ---------------- producer warp
        if (lane == 0) {
            const bool hint = (p.cache_mode & 4) != 0;
            const bool chint = (p.cache_mode & 0x400) != 0;
            const bool clast = (p.cache_mode & 0x800) != 0;
            const uint64_t pol = policy_evict_last();
            const uint64_t cpol = policy_evict_first();
            uint32_t gu = 0, gc = 0;
            bool waited = false;  // griddepcontrol.wait done (see above)
            for (int k = 0; k < nst; ++k)
            for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
                const CUtensorMap* tmu = (MS && (k & 1)) ? &tm_u2 : &tm_u;
                const CUtensorMap* tmp = (MS && (k & 1)) ? &tm_up2 : &tm_up;
                if constexpr (MS) {
                    if (k > 0) wait_unit_flags(p, unit, p.epoch | (unsigned long long)k);
                }
                const UnitGeom g = unit_geom(p, unit, TX, TY);
                const int n = g.ze - g.zs;
                // z sweep direction of this step (RTM_OPT_ZDIR): down on odd-parity steps, so a
                // step starts on the planes the previous step touched last (still in L2).
                // Buffer plane of sweep position j of the u box / of output i (u_prev tile):
                const bool down = sweep_down(p, MS ? p.parity + k : p.parity, unit);
                const int ub0 = (int)g.soff + (down ? g.ze + 9 : g.zs), ustep = down ? -1 : 1;
                const int cz0 = down ? g.ze - 1 : g.zs;
                auto put_u = [&](int j) {  // sweep position j >= QS
                    const uint32_t seq = gu + j - QS, slot = seq % K;
                    if (seq >= K) mbar_wait(&empty_u[slot], ((seq / K) - 1) & 1);
                    mbar_expect_tx(&full_u[slot], S::UBYTES);
                    if (hint)
                        tma_load_3d_hint(uring + slot * S::USLOT, tmu, g.x0 - 8, g.y0 - 5,
                                         ub0 + ustep * j, &full_u[slot], pol);
                    else
                        tma_load_3d(uring + slot * S::USLOT, tmu, g.x0 - 8, g.y0 - 5,
                                    ub0 + ustep * j, &full_u[slot]);
                };
                auto put_c = [&](int i) {
                    const uint32_t seq = gc + i, slot = seq % D;
                    if (seq >= D) mbar_wait(&empty_c[slot], ((seq / D) - 1) & 1);
                    mbar_expect_tx(&full_c[slot], S::CBYTES);
                    float* dst = cring + slot * S::CSLOT;
                    const int cz = cz0 + ustep * i;  // owned plane of output i
                    if (chint)  // read-once stream: evict first, keep u's halo rows in L2
                        tma_load_3d_hint(dst, tmp, g.x0, g.y0, (int)g.soff + cz + 5, &full_c[slot], cpol);
                    else
                        tma_load_3d(dst, tmp, g.x0, g.y0, (int)g.soff + cz + 5, &full_c[slot]);
                    if (chint || clast)  // C: evict first (streams) or evict last (L2-resident C)
                        tma_load_3d_hint(dst + TX * TY, &tm_c, g.x0, g.y0, cz, &full_c[slot],
                                         clast ? pol : cpol);
                    else
                        tma_load_3d(dst + TX * TY, &tm_c, g.x0, g.y0, cz, &full_c[slot]);
                };
                int ci = 0;  // u_prev / C planes of this unit already issued
                if (!waited) {
                    if constexpr (D > 0) {
                        const int pre = n < D ? n : D;  // first ring pass: no empty-slot waits
                        for (; ci < pre; ++ci) put_c(ci);
                    }
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                }
                for (int j = QS; j < 10; ++j) put_u(j);
                for (int i = 0; i < n; ++i) {
                    if constexpr (D > 0) {
                        if (i >= ci) put_c(i);
                    }
                    put_u(i + 10);
                }
                gu += n + 10 - QS;
                gc += n;
            }
            if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
        }
        return;
    }

    // ---------------- consumer warps
    const int tx = tid % S::TXV, ty = tid / S::TXV;
    const int own = (5 + ty) * S::RS + 8 + 4 * tx;
    const int cown = ty * TX + 4 * tx;
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};
    const int pf_mode = p.cache_mode & 3;
    const int pf_dist = (p.cache_mode >> 4) & 15;
    const bool plain = (p.cache_mode & 8) != 0;
    const uint32_t fu = smem_u32(full_u), eu = smem_u32(empty_u);
    const uint32_t fc = smem_u32(full_c), ec = smem_u32(empty_c);
    const float* uown = uring + own;
    uint32_t gu = 0, gc = 0;
    int nstep = 0;  // MS: global index of the step being computed
    for (int k = 0; k < nst; ++k)
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const UnitGeom g = unit_geom(p, unit, TX, TY);
        const int n = g.ze - g.zs;
        float* const nextbuf = (MS && (k & 1)) ? const_cast<float*>(p.u) : p.next;
        if constexpr (MS) nstep = p.step0 + k;
        const int x = g.x0 + 4 * tx, y = g.y0 + ty;
        const bool active = (x < p.nx) && (y < p.ny);
        uint64_t smask = 0;
        if (active) {
            for (int s = 0; s < p.nsrc; ++s) {
                const DevSource& src = p.src[s];
                if (src.shot == g.shot && src.y == y && src.x >= x && src.x < x + 4 &&
                    src.z >= g.zs && src.z < g.ze)
                    smask |= (1ull << s);
            }
        }
        const long long col = (long long)y * p.pitch + x;
        // sweep direction (see the producer); the z register queue is filled in sweep order, so
        // a downward sweep mirrors it — the z pair sums u(z-m) + u(z+m) are commutative (IEEE
        // addition), so results are bitwise those of the upward sweep
        const bool down = sweep_down(p, MS ? p.parity + k : p.parity, unit);
        const int z0 = down ? g.ze - 1 : g.zs, zstep = down ? -1 : 1;
        const long long pstep = down ? -p.plane : p.plane;
        float* outp = nextbuf + (g.soff + z0 + 5) * p.plane + col;  // also u_prev (D == 0)
        const float* cp = p.C + (long long)z0 * p.plane + col;

        // register queue along z: q[QI(O, k)] = u(z - 5 + k) for the O-th unrolled iteration
        float4 q[MQ ? 11 : 10 + U];
        auto release_u = [&](uint32_t slot) {  // this warp is done with u-ring slot `slot`
            if constexpr (MQ) {
                mbar_arrive_u32(eu + 8 * slot);
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive_u32(eu + 8 * slot);
            }
        };
        if constexpr (QS > 0) {
            // the unit's leading z-halo planes feed only this thread's z queue: 128-bit loads of
            // its own 4 points, all in flight with the producer's first ring pass (the first
            // output then waits for one memory round trip instead of two ring passes)
            const float* ucol = p.u + col;
            const long long ub0 = g.soff + (down ? g.ze + 9 : g.zs);
#pragma unroll
            for (int j = 0; j < QS; ++j)
                q[j] = active ? __ldg(reinterpret_cast<const float4*>(ucol + (ub0 + (down ? -j : j)) * p.plane))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = QS; j < 10; ++j) {
            const uint32_t seq = gu + j - QS;
            mbar_wait_u32(fu + 8 * (seq % K), (seq / K) & 1);
            q[j] = *reinterpret_cast<const float4*>(uown + (seq % K) * S::USLOT);
            if (j < 5) release_u(seq % K);
        }
        // running ring positions: plane gu+i+10 (new), gu+i+5 (current), u_prev/C gc+i
        // (sweep positions; the ring sequence is QS behind)
        uint32_t sn = (gu + 10 - QS) % K, pn = ((gu + 10 - QS) / K) & 1;
        uint32_t sc = (gu + 5 - QS) % K;
        uint32_t sq = D > 0 ? gc % D : 0, pq = D > 0 ? (gc / D) & 1 : 0;
        float4 upv = make_float4(0.f, 0.f, 0.f, 0.f), cv = upv;
        if constexpr (D == 0) {
            if (active) {
                upv = ld_mode4(outp, plain);
                cv = ld_mode4(cp, plain);
            }
        }
        int it = 0;
        auto body = [&](auto OFF) {
            constexpr int O = decltype(OFF)::value;
            float4 upn = upv, cn = cv;
            if constexpr (D == 0) {
                if (active && it + 1 < n) {
                    upn = ld_mode4(outp + pstep, plain);
                    cn = ld_mode4(cp + pstep, plain);
                    if (pf_mode && it + pf_dist < n) {
                        prefetch_l2(outp + pf_dist * pstep, pf_mode);
                        prefetch_l2(cp + pf_dist * pstep, pf_mode);
                    }
                }
            }
            mbar_wait_u32(fu + 8 * sn, pn);
            q[QI(O, 10)] = *reinterpret_cast<const float4*>(uown + sn * S::USLOT);
            if constexpr (D > 0) {
                mbar_wait_u32(fc + 8 * sq, pq);
                const float* cb = cring + sq * S::CSLOT + cown;
                upv = *reinterpret_cast<const float4*>(cb);
                cv = *reinterpret_cast<const float4*>(cb + TX * TY);
            }
            const float* row = uown + sc * S::USLOT;
            float xs[14];
            {
                const float4 l = *reinterpret_cast<const float4*>(row - 4);
                const float4 rr = *reinterpret_cast<const float4*>(row + 4);
                xs[0] = row[-5];
                xs[1] = l.x; xs[2] = l.y; xs[3] = l.z; xs[4] = l.w;
                xs[5] = q[QI(O, 5)].x; xs[6] = q[QI(O, 5)].y; xs[7] = q[QI(O, 5)].z; xs[8] = q[QI(O, 5)].w;
                xs[9] = rr.x; xs[10] = rr.y; xs[11] = rr.z; xs[12] = rr.w;
                xs[13] = row[8];
            }
            float4 yv[11];
#pragma unroll
            for (int m = 1; m <= 5; ++m) {
                yv[5 - m] = *reinterpret_cast<const float4*>(row - m * S::RS);
                yv[5 + m] = *reinterpret_cast<const float4*>(row + m * S::RS);
            }
            yv[5] = q[QI(O, 5)];
            float out[4];
            {
                // x pair sums for points (0,1) and (2,3): even m are aligned register pairs
                // of the staged float4s (FADD2), odd m straddle them (two scalar FADDs)
                const float4 L4 = make_float4(xs[1], xs[2], xs[3], xs[4]);
                const float4 R4 = make_float4(xs[9], xs[10], xs[11], xs[12]);
                float2 xa[5], xb[5];
                xa[0] = make_float2(__fadd_rn(xs[4], xs[6]), __fadd_rn(xs[5], xs[7]));
                xa[1] = __fadd2_rn(hi2(L4), hi2(q[QI(O, 5)]));
                xa[2] = make_float2(__fadd_rn(xs[2], xs[8]), __fadd_rn(xs[3], xs[9]));
                xa[3] = __fadd2_rn(lo2(L4), lo2(R4));
                xa[4] = make_float2(__fadd_rn(xs[0], xs[10]), __fadd_rn(xs[1], xs[11]));
                xb[0] = make_float2(__fadd_rn(xs[6], xs[8]), __fadd_rn(xs[7], xs[9]));
                xb[1] = __fadd2_rn(lo2(q[QI(O, 5)]), lo2(R4));
                xb[2] = make_float2(__fadd_rn(xs[4], xs[10]), __fadd_rn(xs[5], xs[11]));
                xb[3] = __fadd2_rn(hi2(L4), hi2(R4));
                xb[4] = make_float2(__fadd_rn(xs[2], xs[12]), __fadd_rn(xs[3], xs[13]));
                float2 za[11], zb[11], ya[11], yb[11];
#pragma unroll
                for (int o = 0; o < 11; ++o) {
                    za[o] = lo2(q[QI(O, o)]);
                    zb[o] = hi2(q[QI(O, o)]);
                    ya[o] = lo2(yv[o]);
                    yb[o] = hi2(yv[o]);
                }
                const float2 ra = rtm_point2(za, ya, xa, lo2(upv), lo2(cv), c);
                const float2 rb = rtm_point2(zb, yb, xb, hi2(upv), hi2(cv), c);
                out[0] = ra.x; out[1] = ra.y; out[2] = rb.x; out[3] = rb.y;
            }
            if constexpr (MQ) {
                mbar_arrive_u32(eu + 8 * sc);
                if constexpr (D > 0) mbar_arrive_u32(ec + 8 * sq);
            } else {
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_u32(eu + 8 * sc);
                    if constexpr (D > 0) mbar_arrive_u32(ec + 8 * sq);
                }
            }
            if (smask) {
                if constexpr (MS)
                    add_sources_n(p, smask, x, z0 + zstep * it, nstep, out);
                else
                    add_sources(p, smask, x, z0 + zstep * it, out);
            }
            if (active) {
                zero_pad(out, x, p.nx);
                const float4 o4 = make_float4(out[0], out[1], out[2], out[3]);
                st_mode4(outp, o4, plain);
                if (p.push_lo || p.push_hi) push_halo4(p, z0 + zstep * it, col, o4);
            }
            if (++sn == K) sn = 0, pn ^= 1;
            if (++sc == K) sc = 0;
            if constexpr (D > 0) {
                if (++sq == D) sq = 0, pq ^= 1;
            } else {
                upv = upn;
                cv = cn;
            }
            outp += pstep;
            cp += pstep;
            ++it;
        };
#pragma unroll 1
        for (int i = 0; i < n; i += U) {
            if (!unrolled<0, U>(body, i, n)) break;
            if constexpr (!MQ) {
#pragma unroll
                for (int o = 0; o < 10; ++o) q[o] = q[o + U];
            }
        }
#pragma unroll 1
        for (int j = n + 5; j < n + 10; ++j) release_u((gu + j - QS) % K);  // planes used only by the queue
        gu += n + 10 - QS;
        gc += n;
        if constexpr (MS) {
            // publish "unit done with step k": every consumer thread orders its own stores of the
            // unit at gpu scope (fence), the CTA barrier collects them, one gpu-scope release is
            // read by the neighbours' producers (acquire + async-proxy fence before their TMA)
            __threadfence();
            asm volatile("bar.sync 1, %0;" ::"n"(S::NW * 32) : "memory");
            if (tid == 0) st_release_gpu_u64(p.flags + unit, p.epoch | (unsigned long long)(k + 1));
        }
    }
}

// ------------------------------------------------------------------------------------
// Variant table.  id 0 = naive; kind 1 = k_tiled; kind 2 = k_stream.
#define RTM_VARIANTS(X)                                  \
    X(1, "stream64x16k8d4u4", 2, 64, 16, 8, 4, 2, 4)     \
    X(2, "stream64x16k8d4", 2, 64, 16, 8, 4, 2, 1)       \
    X(3, "stream64x16k8d4u2", 2, 64, 16, 8, 4, 2, 2)     \
    X(4, "stream32x32k8d4u4", 2, 32, 32, 8, 4, 2, 4)     \
    X(5, "stream64x16k9d0u4", 2, 64, 16, 9, 0, 2, 4)     \
    X(6, "stream64x32k10d0u4", 2, 64, 32, 10, 0, 1, 4)   \
    X(7, "stream64x14k8d4u2", 2, 64, 14, 8, 4, 2, 2)     \
    X(8, "stream64x14k8d4u4", 2, 64, 14, 8, 4, 2, 4)     \
    X(9, "stream128x7k8d4u2", 2, 128, 7, 8, 4, 2, 2)     \
    X(10, "stream128x7k8d4u4", 2, 128, 7, 8, 4, 2, 4)    \
    X(11, "stream64x14k8d4u11", 2, 64, 14, 8, 4, 2, 11)  \
    X(12, "stream32x28k8d4u4", 2, 32, 28, 8, 4, 2, 4)    \
    X(13, "stream64x16k8d4u11", 2, 64, 16, 8, 4, 2, 11)  \
    X(14, "tma64x16k10", 1, 64, 16, 10, 0, 2, 1)         \
    X(15, "tma32x16k10", 1, 32, 16, 10, 0, 3, 1)         \
    X(16, "stream64x14k10d4u4", 2, 64, 14, 10, 4, 2, 4)  \
    X(17, "stream64x14k10d5u4", 2, 64, 14, 10, 5, 2, 4)  \
    X(18, "stream64x16k9d4u11", 2, 64, 16, 9, 4, 2, 11)  \
    X(19, "stream128x7k9d3u4", 2, 128, 7, 9, 3, 2, 4)    \
    X(20, "stream64x14k10d4u11", 2, 64, 14, 10, 4, 2, 11) \
    X(21, "stream64x14k12d3u4", 2, 64, 14, 12, 3, 2, 4)  \
    X(22, "stream64x16k8d5u11", 2, 64, 16, 8, 5, 2, 11)  \
    X(23, "stream64x14k9d6u4", 2, 64, 14, 9, 6, 2, 4)    \
    X(24, "stream64x14k8d7u4", 2, 64, 14, 8, 7, 2, 4)    \
    X(25, "stream32x28k10d5u4", 2, 32, 28, 10, 5, 2, 4)  \
    X(26, "stream64x14k10d5u11", 2, 64, 14, 10, 5, 2, 11) \
    X(27, "stream64x28k10d4u4", 2, 64, 28, 10, 4, 1, 4)   \
    X(28, "stream64x28k10d6u4", 2, 64, 28, 10, 6, 1, 4)   \
    X(29, "stream128x14k9d5u4", 2, 128, 14, 9, 5, 1, 4)   \
    X(30, "stream64x14k10d5u2", 2, 64, 14, 10, 5, 2, 2)   \
    X(31, "stream64x28k11d6u4", 2, 64, 28, 11, 6, 1, 4)   \
    X(32, "stream64x28k10d7u4", 2, 64, 28, 10, 7, 1, 4)   \
    X(33, "stream128x14k10d6u4", 2, 128, 14, 10, 6, 1, 4) \
    X(34, "stream64x24k11d7u4", 2, 64, 24, 11, 7, 1, 4)   \
    X(35, "stream64x30k10d6u4", 2, 64, 30, 10, 6, 1, 4)   \
    X(36, "stream64x28k10d6u11", 2, 64, 28, 10, 6, 1, 11)

// Multi-step (kind 6) variants: k_stream<..., MS = true>, same columns as RTM_VARIANTS.
// The last column is the single-step k_stream variant of the same shape, run where multi-step
// launches do not apply (slab contexts).
#define RTM_MS_VARIANTS(X)                                      \
    X(43, "ms64x30k10d6u4", 6, 64, 30, 10, 6, 1, 4, 35)         \
    X(44, "ms128x7k8d4u4", 6, 128, 7, 8, 4, 2, 4, 10)           \
    X(45, "ms64x16k8d4u4", 6, 64, 16, 8, 4, 2, 4, 1)            \
    X(46, "ms64x14k10d5u4", 6, 64, 14, 10, 5, 2, 4, 17)         \
    X(47, "ms64x28k10d6u4", 6, 64, 28, 10, 6, 1, 4, 28)         \
    X(50, "ms64x30k10d6u11", 6, 64, 30, 10, 6, 1, 11, 48)

// Later single-step (kind 2) variants, appended after the multi-step ids: the U = 11 forms
// (modulo-scheduled z queue, per-lane slot release) of the best tiles.
#define RTM_VARIANTS2(X)                                   \
    X(48, "stream64x30k10d6u11", 2, 64, 30, 10, 6, 1, 11)  \
    X(49, "stream128x7k8d4u11", 2, 128, 7, 8, 4, 2, 11)

static const TileVariant kVariants[] = {
    {"naive", 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0},
#define X(id, name, kind, tx, ty, k, d, mb, u) {name, kind, tx, ty, k, d, mb, u, 0, 0, 0, 0},
    RTM_VARIANTS(X)
#undef X
#define X(id, name, tx, ty, k, d, u, lmax, w, ch, pair) {name, 4, tx, ty, k, d, 2, u, w, ch, lmax, pair},
    RTM_TB2S_VARIANTS(X)
#undef X
#define X(id, name, threads, per_sm, pair) {name, 5, threads, 0, 0, 0, per_sm, 1, 0, 0, 0, pair},
    RTM_RESIDENT_VARIANTS(X)
#undef X
// (table order = id order: 43-47 multi-step, 48-49 single-step, 50 multi-step)
#define X(id, name, kind, tx, ty, k, d, mb, u, pair) \
    {name, kind, tx, ty, k, d, mb, u, 0, 0, 0, pair},
#define X2(id, name, kind, tx, ty, k, d, mb, u) {name, kind, tx, ty, k, d, mb, u, 0, 0, 0, 0},
    X(43, "ms64x30k10d6u4", 6, 64, 30, 10, 6, 1, 4, 35)
    X(44, "ms128x7k8d4u4", 6, 128, 7, 8, 4, 2, 4, 10)
    X(45, "ms64x16k8d4u4", 6, 64, 16, 8, 4, 2, 4, 1)
    X(46, "ms64x14k10d5u4", 6, 64, 14, 10, 5, 2, 4, 17)
    X(47, "ms64x28k10d6u4", 6, 64, 28, 10, 6, 1, 4, 28)
    RTM_VARIANTS2(X2)
    X(50, "ms64x30k10d6u11", 6, 64, 30, 10, 6, 1, 11, 48)
#undef X2
#undef X
#define X(id, name, tx, ty, k, d, mb) {name, 7, tx, ty, k, d, mb, 11, 0, 0, 0, 0},
    RTM_STREAM2_VARIANTS(X)
#undef X
};

int num_variants() { return static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0])); }
const TileVariant& variant(int id) { return kVariants[id]; }

template <int KIND, int TX, int TY, int K, int D, int MINB, int U>
static cudaError_t prepare(const void** fn, int* threads, size_t* smem) {
    if constexpr (KIND == 1) {
        using S = TiledShape<TX, TY, K>;
        *fn = reinterpret_cast<const void*>(&k_tiled<TX, TY, K, MINB>);
        *threads = S::NT;
        *smem = S::SMEM;
    } else {
        using S = StreamShape<TX, TY, K, D, U>;
        *fn = reinterpret_cast<const void*>(&k_stream<TX, TY, K, D, MINB, U, KIND == 6>);
        *threads = S::NT;
        *smem = S::SMEM;
    }
    return cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(*smem));
}

static cudaError_t variant_fn(int id, const void** fn, int* threads, size_t* smem) {
    if (id > 0 && id < num_variants() && variant(id).kind == 4) return tb2s_variant_fn(id, fn, threads, smem);
    if (id > 0 && id < num_variants() && variant(id).kind == 7) return stream2_variant_fn(id, fn, threads, smem);
    if (id > 0 && id < num_variants() && variant(id).kind == 5) {
        *fn = nullptr;
        *threads = variant(id).TX;
        *smem = 0;
        return cudaSuccess;
    }
    switch (id) {
#define X(vid, name, kind, tx, ty, k, d, mb, u) \
    case vid:                                   \
        return prepare<kind, tx, ty, k, d, mb, u>(fn, threads, smem);
        RTM_VARIANTS(X)
#undef X
#define X(vid, name, kind, tx, ty, k, d, mb, u, pair) \
    case vid:                                         \
        return prepare<kind, tx, ty, k, d, mb, u>(fn, threads, smem);
        RTM_MS_VARIANTS(X)
#undef X
#define X(vid, name, kind, tx, ty, k, d, mb, u) \
    case vid:                                   \
        return prepare<kind, tx, ty, k, d, mb, u>(fn, threads, smem);
        RTM_VARIANTS2(X)
#undef X
        default:
            return cudaErrorInvalidValue;
    }
}

size_t variant_smem_bytes(int id) {
    const void* fn;
    int threads;
    size_t smem = 0;
    if (variant_fn(id, &fn, &threads, &smem) != cudaSuccess) return 0;
    return smem;
}

int variant_occupancy(int id, int* threads_per_block) {
    const void* fn;
    int threads;
    size_t smem;
    if (variant_fn(id, &fn, &threads, &smem) != cudaSuccess) return -1;
    if (variant(id).kind == 5) {
        int nb = 0;
        if (resident_occupancy(threads, &nb) != cudaSuccess) return -1;
        if (threads_per_block) *threads_per_block = threads;
        return nb;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess)
        return -1;
    if (threads_per_block) *threads_per_block = threads;
    return nb;
}

cudaError_t launch_variant(int id, const CUtensorMap* tm_u, const CUtensorMap* tm_up,
                           const CUtensorMap* tm_c, const StencilParams& p, int max_ctas,
                           cudaStream_t s, bool pdl) {
    const void* fn;
    int threads;
    size_t smem;
    const int kind = variant(id).kind;
    if (kind >= 3 && kind != 7) return cudaErrorInvalidValue;  // two-step / resident / multi-step: own launchers
    cudaError_t e = variant_fn(id, &fn, &threads, &smem);
    if (e != cudaSuccess) return e;
    const long long units = (long long)p.tiles_x * p.tiles_y *
                            (p.r_chunks[0] + (p.nranges > 1 ? p.r_chunks[1] : 0)) * p.nshots;
    if (units <= 0) return cudaSuccess;
    if (variant(id).kind == 1) {
        void* args[] = {const_cast<CUtensorMap*>(tm_u), const_cast<StencilParams*>(&p)};
        return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(units)), dim3(threads), args, smem, s);
    }
    const long long grid = units < max_ctas ? units : max_ctas;
    void* args[] = {const_cast<CUtensorMap*>(tm_u), const_cast<CUtensorMap*>(tm_up),
                    const_cast<CUtensorMap*>(tm_c), const_cast<StencilParams*>(&p),
                    const_cast<CUtensorMap*>(tm_u), const_cast<CUtensorMap*>(tm_up)};  // k_stream2 reads the first 4
    if (!pdl) return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(threads), args, smem, s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_mstep(int id, const CUtensorMap* tm_u, const CUtensorMap* tm_up,
                         const CUtensorMap* tm_u2, const CUtensorMap* tm_up2, const CUtensorMap* tm_c,
                         const StencilParams& p, int max_ctas, cudaStream_t s) {
    if (variant(id).kind != 6 || p.nranges != 1 || !p.flags || p.nsteps < 1) return cudaErrorInvalidValue;
    const void* fn;
    int threads;
    size_t smem;
    cudaError_t e = variant_fn(id, &fn, &threads, &smem);
    if (e != cudaSuccess) return e;
    const long long units = (long long)p.tiles_x * p.tiles_y * p.r_chunks[0] * p.nshots;
    if (units <= 0) return cudaSuccess;
    // every CTA must be co-resident: units wait on their neighbours' flags (cooperative launch)
    const long long grid = units < max_ctas ? units : max_ctas;
    void* args[] = {const_cast<CUtensorMap*>(tm_u), const_cast<CUtensorMap*>(tm_up),
                    const_cast<CUtensorMap*>(tm_c), const_cast<StencilParams*>(&p),
                    const_cast<CUtensorMap*>(tm_u2), const_cast<CUtensorMap*>(tm_up2)};
    return cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(threads), args, smem, s);
}

cudaError_t launch_naive(const StencilParams& p, cudaStream_t s) {
    long long total = (long long)p.r_len[0] * p.plane;
    if (p.nranges > 1) total += (long long)p.r_len[1] * p.plane;
    total *= p.nshots;
    if (total <= 0) return cudaSuccess;
    long long blocks = (total + 255) / 256;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    k_naive<<<static_cast<unsigned>(blocks), 256, 0, s>>>(p);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_field_stats(const float* buf, long long plane, int nzl,
                                                     int nshots, unsigned int* stats) {
    float m = 0.0f;
    unsigned int bad = 0;
    const long long per_shot = plane * nzl;
    const long long n = per_shot * nshots;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const long long shot = t / per_shot;
        const float v = buf[(shot * (nzl + 10) + 5) * plane + (t - shot * per_shot)];
        if (!isfinite(v)) ++bad;
        else m = fmaxf(m, fabsf(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&stats[0], __float_as_uint(m));
        if (bad) atomicAdd(&stats[1], bad);
    }
}

cudaError_t launch_field_stats(const float* buf, long long plane, int nzl, int nshots,
                               unsigned int* stats, cudaStream_t s) {
    const long long n = plane * nzl * nshots;
    if (n <= 0) return cudaSuccess;
    long long blocks = (n + 255) / 256;
    if (blocks > 148LL * 8) blocks = 148LL * 8;
    k_field_stats<<<static_cast<unsigned>(blocks), 256, 0, s>>>(buf, plane, nzl, nshots, stats);
    return cudaGetLastError();
}

// Fused-push step signal (f1, flag protocol): after a slab's stencil launch has completed (stream
// order), publish "steps done" to the neighbours' flag words (peer / CUDA-IPC device memory) with
// a system-scope fence + release store, so their next step's stream wait (cuStreamWaitValue64)
// sees the halo planes this step pushed into them.
__global__ void k_signal(unsigned long long* lo, unsigned long long* hi, unsigned long long v) {
    __threadfence_system();
    if (lo) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(lo), "l"(v) : "memory");
    if (hi) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(hi), "l"(v) : "memory");
}

cudaError_t launch_signal(unsigned long long* lo, unsigned long long* hi, unsigned long long v,
                          cudaStream_t s) {
    if (!lo && !hi) return cudaSuccess;
    k_signal<<<1, 1, 0, s>>>(lo, hi, v);
    return cudaGetLastError();
}

cudaError_t launch_velocity(const float* v, float* C, long long n, int nx, int pitch, double dt,
                            double dx, unsigned int* stats, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int vec4 = (n % 4 == 0) && (reinterpret_cast<uintptr_t>(v) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(C) % 16 == 0);
    long long blocks = ((vec4 ? n / 4 : n) + 255) / 256;
    if (blocks > 148LL * 8) blocks = 148LL * 8;
    k_velocity<<<static_cast<unsigned>(blocks), 256, 0, s>>>(v, C, n, nx, pitch, dt, dx, stats, vec4);
    return cudaGetLastError();
}

}  // namespace rtm
