// =====================================================================================
// k_stream2: k_stream with TWO rows per consumer thread (4 x-points × 2 y-rows = 8 points).
// RTM 3D-model step (§2, Algorithm 1 "calculate 3D model").
//
// Same pipeline as k_stream (rtm_kernels.cu): persistent CTAs, one producer warp streaming the
// halo'd u box of every plane into a K-slot TMA ring and the (u_prev, C) tiles into a D-slot
// ring, consumer warps with a register queue along z.  What changes is the consumer mapping:
//   * a thread owns rows y and y+1 of a 4-point column, so its y-neighbour loads are shared —
//     rows y-5 .. y+6 are 10 LDS.128 for 8 points (two one-row threads issue 20);
//   * the per-thread bookkeeping (ring slots, barrier waits / arrivals, branches, address
//     arithmetic) is paid once per 8 points instead of once per 4;
//   * the two z queues are modulo-scheduled (q[r][(O + k) % 11], unrolled 11×: no register
//     copies) and empty slots are released by per-lane arrivals.
// Every point runs rtm_point2 (k_stream's expression, same operand order): results are
// bitwise identical to k_stream and the naive kernel.
// =====================================================================================
#include "rtm_internal.h"
#include "rtm_device.cuh"

#include <type_traits>

namespace rtm {

template <int TX, int TY, int K, int D>
struct Stream2Shape {
    static constexpr int R = 2;                     // rows per consumer thread
    static constexpr int TXV = TX / 4;              // threads per row pair
    static constexpr int NW = TX * TY / (128 * R);  // consumer warps
    static constexpr int NT = NW * 32 + 32;         // + producer warp
    static constexpr int RS = TX + 16;
    static constexpr int ROWS = TY + 10;
    static constexpr int USLOT = (RS * ROWS + 31) / 32 * 32;
    static constexpr uint32_t UBYTES = RS * ROWS * 4;
    static constexpr int CSLOT = 2 * TX * TY;
    static constexpr uint32_t CBYTES = CSLOT * 4;
    static constexpr size_t BAR_OFF = (size_t(K) * USLOT + size_t(D) * CSLOT) * 4;
    static constexpr size_t SMEM = BAR_OFF + size_t(2 * K + 2 * D) * 8;
    static constexpr int EMPTY_COUNT = NW * 32;     // per-lane releases
    // registers per thread that let MINB CTAs share the 64 K-register file (multiple of 8, <= 255)
    template <int MINB>
    static constexpr int maxreg() {
        const int r = 65536 / (NT * MINB) / 8 * 8;
        return r > 248 ? 248 : r;
    }
    static_assert((TX * TY) % (128 * R) == 0 && TY % R == 0, "whole consumer warps of row pairs");
    static_assert(K >= 7 && D >= 1, "ring depths");
    static_assert(TX % 4 == 0 && RS <= 256 && ROWS <= 256 && TX <= 256 && TY <= 256, "TMA box");
};

template <int TX, int TY, int K, int D, int MINB>
__global__ void __launch_bounds__(Stream2Shape<TX, TY, K, D>::NT, MINB)
    __maxnreg__((Stream2Shape<TX, TY, K, D>::template maxreg<MINB>()))
    k_stream2(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_up,
              const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ StencilParams p) {
    using S = Stream2Shape<TX, TY, K, D>;
    constexpr int R = S::R;
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
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (p.write_next && blockIdx.x == 0 && tid == 0) p.d_step[p.parity ^ 1] = p.d_step[p.parity] + 1;

    const int units = p.tiles_x * p.tiles_y * (p.r_chunks[0] + (p.nranges > 1 ? p.r_chunks[1] : 0)) *
                      p.nshots;

    if (warp == S::NW) {  // ---------------- producer warp (k_stream's)
        if (lane == 0) {
            const bool hint = (p.cache_mode & 4) != 0;
            const uint64_t pol = policy_evict_last();
            uint32_t gu = 0, gc = 0;
            for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
                const UnitGeom g = unit_geom(p, unit, TX, TY);
                const int n = g.ze - g.zs;
                const bool down = sweep_down(p, p.parity, unit);
                const int ub0 = (int)g.soff + (down ? g.ze + 9 : g.zs), ustep = down ? -1 : 1;
                const int cz0 = down ? g.ze - 1 : g.zs;
                auto put_u = [&](int j) {
                    const uint32_t seq = gu + j, slot = seq % K;
                    if (seq >= K) mbar_wait(&empty_u[slot], ((seq / K) - 1) & 1);
                    mbar_expect_tx(&full_u[slot], S::UBYTES);
                    if (hint)
                        tma_load_3d_hint(uring + slot * S::USLOT, &tm_u, g.x0 - 8, g.y0 - 5, ub0 + ustep * j,
                                         &full_u[slot], pol);
                    else
                        tma_load_3d(uring + slot * S::USLOT, &tm_u, g.x0 - 8, g.y0 - 5, ub0 + ustep * j,
                                    &full_u[slot]);
                };
                auto put_c = [&](int i) {
                    const uint32_t seq = gc + i, slot = seq % D;
                    if (seq >= D) mbar_wait(&empty_c[slot], ((seq / D) - 1) & 1);
                    mbar_expect_tx(&full_c[slot], S::CBYTES);
                    float* dst = cring + slot * S::CSLOT;
                    const int cz = cz0 + ustep * i;
                    tma_load_3d(dst, &tm_up, g.x0, g.y0, (int)g.soff + cz + 5, &full_c[slot]);
                    tma_load_3d(dst + TX * TY, &tm_c, g.x0, g.y0, cz, &full_c[slot]);
                };
                for (int j = 0; j < 10; ++j) put_u(j);
                for (int i = 0; i < n; ++i) {
                    put_c(i);
                    put_u(i + 10);
                }
                gu += n + 10;
                gc += n;
            }
        }
        return;
    }

    // ---------------- consumer warps: rows ty0 and ty0 + 1 of a 4-point column
    const int tx = tid % S::TXV, ty0 = (tid / S::TXV) * R;
    const int own0 = (5 + ty0) * S::RS + 8 + 4 * tx;  // row ty0 in a u slot; row ty0+1 is + RS
    const int cown0 = ty0 * TX + 4 * tx;
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};
    const bool plain = (p.cache_mode & 8) != 0;
    const uint32_t fu = smem_u32(full_u), eu = smem_u32(empty_u);
    const uint32_t fc = smem_u32(full_c), ec = smem_u32(empty_c);
    const float* uown = uring + own0;
    constexpr auto QI = [](int O, int k) constexpr { return (O + k) % 11; };
    uint32_t gu = 0, gc = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const UnitGeom g = unit_geom(p, unit, TX, TY);
        const int n = g.ze - g.zs;
        const int x = g.x0 + 4 * tx;
        bool active[R];
        uint64_t smask[R];
        long long col[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int y = g.y0 + ty0 + r;
            active[r] = (x < p.nx) && (y < p.ny);
            col[r] = (long long)y * p.pitch + x;
            smask[r] = 0;
            if (active[r]) {
                for (int s = 0; s < p.nsrc; ++s) {
                    const DevSource& src = p.src[s];
                    if (src.shot == g.shot && src.y == y && src.x >= x && src.x < x + 4 && src.z >= g.zs &&
                        src.z < g.ze)
                        smask[r] |= (1ull << s);
                }
            }
        }
        const bool down = sweep_down(p, p.parity, unit);
        const int z0 = down ? g.ze - 1 : g.zs, zstep = down ? -1 : 1;
        const long long pstep = down ? -p.plane : p.plane;
        float* outp = p.next + (g.soff + z0 + 5) * p.plane + col[0];  // row 1: + (col[1] - col[0])
        const long long dcol = col[1] - col[0];

        float4 q[R][11];  // q[r][QI(O, k)] = u(z - 5 + k) at row r, unrolled iteration O
#pragma unroll
        for (int j = 0; j < 10; ++j) {
            const uint32_t seq = gu + j;
            mbar_wait_u32(fu + 8 * (seq % K), (seq / K) & 1);
#pragma unroll
            for (int r = 0; r < R; ++r)
                q[r][j] = *reinterpret_cast<const float4*>(uown + (seq % K) * S::USLOT + r * S::RS);
            if (j < 5) mbar_arrive_u32(eu + 8 * (seq % K));
        }
        uint32_t sn = (gu + 10) % K, pn = ((gu + 10) / K) & 1;
        uint32_t sc = (gu + 5) % K;
        uint32_t sq = gc % D, pq = (gc / D) & 1;
        int it = 0;
        auto body = [&](auto OFF) {
            constexpr int O = decltype(OFF)::value;
            mbar_wait_u32(fu + 8 * sn, pn);
#pragma unroll
            for (int r = 0; r < R; ++r)
                q[r][QI(O, 10)] = *reinterpret_cast<const float4*>(uown + sn * S::USLOT + r * S::RS);
            mbar_wait_u32(fc + 8 * sq, pq);
            float4 upv[R], cv[R];
            {
                const float* cb = cring + sq * S::CSLOT + cown0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    upv[r] = *reinterpret_cast<const float4*>(cb + r * TX);
                    cv[r] = *reinterpret_cast<const float4*>(cb + TX * TY + r * TX);
                }
            }
            const float* row0 = uown + sc * S::USLOT;
            // rows ty0-5 .. ty0+R+4 of the centre plane; the thread's own rows from its queues
            float4 yall[10 + R];
#pragma unroll
            for (int m = -5; m < R + 5; ++m) {
                if (m >= 0 && m < R)
                    yall[m + 5] = q[m][QI(O, 5)];
                else
                    yall[m + 5] = *reinterpret_cast<const float4*>(row0 + m * S::RS);
            }
            float out[R][4];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float* row = row0 + r * S::RS;
                const float4 ctr = q[r][QI(O, 5)];
                float xs[14];
                {
                    const float4 l = *reinterpret_cast<const float4*>(row - 4);
                    const float4 rr = *reinterpret_cast<const float4*>(row + 4);
                    xs[0] = row[-5];
                    xs[1] = l.x; xs[2] = l.y; xs[3] = l.z; xs[4] = l.w;
                    xs[5] = ctr.x; xs[6] = ctr.y; xs[7] = ctr.z; xs[8] = ctr.w;
                    xs[9] = rr.x; xs[10] = rr.y; xs[11] = rr.z; xs[12] = rr.w;
                    xs[13] = row[8];
                }
                // k_stream's pairing: x pair sums of points (0,1) and (2,3)
                const float4 L4 = make_float4(xs[1], xs[2], xs[3], xs[4]);
                const float4 R4 = make_float4(xs[9], xs[10], xs[11], xs[12]);
                float2 xa[5], xb[5];
                xa[0] = make_float2(__fadd_rn(xs[4], xs[6]), __fadd_rn(xs[5], xs[7]));
                xa[1] = __fadd2_rn(hi2(L4), hi2(ctr));
                xa[2] = make_float2(__fadd_rn(xs[2], xs[8]), __fadd_rn(xs[3], xs[9]));
                xa[3] = __fadd2_rn(lo2(L4), lo2(R4));
                xa[4] = make_float2(__fadd_rn(xs[0], xs[10]), __fadd_rn(xs[1], xs[11]));
                xb[0] = make_float2(__fadd_rn(xs[6], xs[8]), __fadd_rn(xs[7], xs[9]));
                xb[1] = __fadd2_rn(lo2(ctr), lo2(R4));
                xb[2] = make_float2(__fadd_rn(xs[4], xs[10]), __fadd_rn(xs[5], xs[11]));
                xb[3] = __fadd2_rn(hi2(L4), hi2(R4));
                xb[4] = make_float2(__fadd_rn(xs[2], xs[12]), __fadd_rn(xs[3], xs[13]));
                float2 za[11], zb[11], ya[11], yb[11];
#pragma unroll
                for (int o = 0; o < 11; ++o) {
                    za[o] = lo2(q[r][QI(O, o)]);
                    zb[o] = hi2(q[r][QI(O, o)]);
                    ya[o] = lo2(yall[r + o]);
                    yb[o] = hi2(yall[r + o]);
                }
                const float2 ra = rtm_point2(za, ya, xa, lo2(upv[r]), lo2(cv[r]), c);
                const float2 rb = rtm_point2(zb, yb, xb, hi2(upv[r]), hi2(cv[r]), c);
                out[r][0] = ra.x; out[r][1] = ra.y; out[r][2] = rb.x; out[r][3] = rb.y;
            }
            mbar_arrive_u32(eu + 8 * sc);  // per-lane releases (EMPTY_COUNT = consumer lanes)
            mbar_arrive_u32(ec + 8 * sq);
            const int z = z0 + zstep * it;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (smask[r]) add_sources(p, smask[r], x, z, out[r]);
                if (active[r]) {
                    zero_pad(out[r], x, p.nx);
                    const float4 o4 = make_float4(out[r][0], out[r][1], out[r][2], out[r][3]);
                    st_mode4(outp + r * dcol, o4, plain);
                    if (p.push_lo || p.push_hi) push_halo4(p, z, col[r], o4);
                }
            }
            if (++sn == K) sn = 0, pn ^= 1;
            if (++sc == K) sc = 0;
            if (++sq == D) sq = 0, pq ^= 1;
            outp += pstep;
            ++it;
        };
#pragma unroll 1
        for (int i = 0; i < n; i += 11) {
            if (!unrolled<0, 11>(body, i, n)) break;
        }
#pragma unroll 1
        for (int j = n + 5; j < n + 10; ++j) mbar_arrive_u32(eu + 8 * ((gu + j) % K));
        gu += n + 10;
        gc += n;
    }
}

// Variant launcher: kind 7 (k_stream2) with the kind-2 argument list.
template <int TX, int TY, int K, int D, int MINB>
static cudaError_t prepare2(const void** fn, int* threads, size_t* smem) {
    using S = Stream2Shape<TX, TY, K, D>;
    *fn = reinterpret_cast<const void*>(&k_stream2<TX, TY, K, D, MINB>);
    *threads = S::NT;
    *smem = S::SMEM;
    return cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(*smem));
}

cudaError_t stream2_variant_fn(int id, const void** fn, int* threads, size_t* smem) {
    switch (id) {
#define X(vid, name, tx, ty, k, d, mb) \
    case vid:                          \
        return prepare2<tx, ty, k, d, mb>(fn, threads, smem);
        RTM_STREAM2_VARIANTS(X)
#undef X
        default:
            return cudaErrorInvalidValue;
    }
}

}  // namespace rtm
