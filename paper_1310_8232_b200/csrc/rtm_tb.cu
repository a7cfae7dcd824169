// =====================================================================================
// k_tb2: two time steps of the RTM 3D-model update (§2, Algorithm 1)
// per HBM pass — temporal blocking, SURVEY.md §8(f) f4 (§4 names time blocking
// among the related stencil optimisations).
//
// The single-step kernel (k_stream) moves 16 B per point update and runs at the HBM copy
// peak.  k_tb2 reads u^n, u^{n-1}, C once and writes u^{n+1}, u^{n+2}: 20 B per two updates.
// The intermediate level u^{n+1} is consumed from L2 shortly after it is produced:
//
//   * The grid is cut into y-bands; one launch per band.  The band's CTAs (all co-resident,
//     cooperative launch, one per SM) own fixed xy tiles of the band's A region = the band's
//     rows plus 5 rows each side, and sweep z from 0 to nz together.
//   * Stage A (step n -> n+1) on plane z: the k_stream algorithm (TMA ring of halo'd u^n
//     planes, 11-plane register queue along z, packed FP32x2 point update), result stored to
//     outA (L2-resident for now; it is also the next pass's u_prev).  Each consumer warp
//     arrives (release.cta) on a per-plane mbarrier; a publisher warp waits for the CTA's
//     completed planes and releases flags[cta] = epoch<<32 | planes done at gpu scope.
//   * Stage B (step n+1 -> n+2) on plane z-L: a second producer warp waits (acquire) until
//     this CTA and its four edge neighbours have published A through plane z-L+5, then TMAs
//     the halo'd u^{n+1} box (from L2) into a second ring; the same consumer threads compute
//     u^{n+2} on the band's own rows and stream it to outB.
//   * Rows of the A region outside the band are recomputed by the neighbouring band
//     (redundant work ~ 10 / band rows); both bands store bitwise-identical values.
//
// Every point is computed by star4() = the exact arithmetic of k_stream (rtm_device.cuh), so
// k_tb2 results are bitwise identical to two k_stream steps (tests/test_gpu_parity.py).
// Deadlock freedom: stage A never waits on other CTAs; stage B of plane j waits only for A
// planes <= j+5 < the plane the slowest warp anywhere is working on (lag L >= 6), and all CTAs
// are resident.  Every spin has a 4 s watchdog that traps (a launch error, never a hang).
// =====================================================================================
#include "rtm_internal.h"
#include "rtm_device.cuh"

namespace rtm {

// ---- gpu/cta-scope acquire/release, proxy fence, watchdog --------------------------------
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

// mbarrier wait with a watchdog on the slow path only
__device__ __forceinline__ void mbar_wait_wd(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    const unsigned long long t0 = globaltimer_ns();
    unsigned spins = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
        if (!ok && (++spins & 1023) == 0 && globaltimer_ns() - t0 > kWatchdogNs) __trap();
    } while (!ok);
}

// Sources of this thread's 4-point column at plane z with sample index n (a3, fused).
__device__ __forceinline__ void add_sources_n(const TBParams& p, uint64_t mask, int x, int z,
                                              int n, float (&out)[4]) {
    while (mask) {
        const int s = __ffsll(static_cast<long long>(mask)) - 1;
        mask &= mask - 1;
        const DevSource& src = p.src[s];
        if (src.z == z && n < src.nsamples) {
            const float w = p.samples[src.offset + n];
            const int i = src.x - x;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k == i) out[k] = __fadd_rn(out[k], w);
        }
    }
}

template <int TX, int TY, int KA, int KB, int DA, int DB>
struct TBShape {
    static constexpr int NW = TX * TY / 128;  // consumer warps (4 points per thread)
    static constexpr int NT = (NW + 3) * 32;  // + producer A, producer B, publisher
    static constexpr int TXV = TX / 4;
    static constexpr int RS = TX + 16;
    static constexpr int ROWS = TY + 10;
    static constexpr int USLOT = (RS * ROWS + 31) / 32 * 32;
    static constexpr uint32_t UBYTES = RS * ROWS * 4;
    static constexpr int CSLOT = 2 * TX * TY;  // u_prev tile then C tile
    static constexpr uint32_t CBYTES = CSLOT * 4;
    static constexpr int OFF_UB = KA * USLOT;
    static constexpr int OFF_CA = OFF_UB + KB * USLOT;
    static constexpr int OFF_CB = OFF_CA + DA * CSLOT;
    static constexpr size_t BAR_OFF = size_t(OFF_CB + DB * CSLOT) * 4;
    static constexpr int NPUB = 64;  // stage-A completion ring (> lag + 8: see the publisher)
    static constexpr int NBAR = 2 * (KA + KB + DA + DB) + NPUB;
    static constexpr size_t SMEM = BAR_OFF + size_t(NBAR) * 8;
    static_assert((TX * TY) % 128 == 0, "whole consumer warps");
    static_assert(KA >= 7 && KB >= 7, "6 live planes + 1 in flight");
    static_assert(DA >= 1 && DB >= 1, "u_prev/C rings");
    static_assert(TX >= 8 && TY >= 5, "halo reaches only the 4 edge-neighbour tiles");
    static_assert(TX % 4 == 0 && RS <= 256 && ROWS <= 256 && TX <= 256 && TY <= 256, "TMA box");
    static_assert(SMEM <= 232448, "shared memory");
};

template <int TX, int TY, int KA, int KB, int DA, int DB, int L, int U>
__global__ void __launch_bounds__(TBShape<TX, TY, KA, KB, DA, DB>::NT, 1)
    k_tb2(const __grid_constant__ CUtensorMap tmA_u, const __grid_constant__ CUtensorMap tmA_up,
          const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tmB_u,
          const __grid_constant__ CUtensorMap tmB_up, const __grid_constant__ TBParams p) {
    using S = TBShape<TX, TY, KA, KB, DA, DB>;
    static_assert(L >= 6 && L % U == 0, "lag: B plane j needs A planes <= j+5; B starts on a group");
    static_assert(S::NPUB >= L + 16, "consumers run at most L + 6 planes ahead of the publisher");
    extern __shared__ __align__(128) float smem[];
    float* uA = smem;
    float* uB = smem + S::OFF_UB;
    float* cA = smem + S::OFF_CA;
    float* cB = smem + S::OFF_CB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + S::BAR_OFF);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + KA;
    uint64_t* fullB = emptyA + KA;
    uint64_t* emptyB = fullB + KB;
    uint64_t* fullCA = emptyB + KB;
    uint64_t* emptyCA = fullCA + DA;
    uint64_t* fullCB = emptyCA + DA;
    uint64_t* emptyCB = fullCB + DB;
    uint64_t* pubA = emptyCB + DB;  // pubA[i % NPUB]: all consumer warps finished A plane i

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < KA; ++k) mbar_init(&fullA[k], 1), mbar_init(&emptyA[k], S::NW);
        for (int k = 0; k < KB; ++k) mbar_init(&fullB[k], 1), mbar_init(&emptyB[k], S::NW);
        for (int k = 0; k < DA; ++k) mbar_init(&fullCA[k], 1), mbar_init(&emptyCA[k], S::NW);
        for (int k = 0; k < DB; ++k) mbar_init(&fullCB[k], 1), mbar_init(&emptyCB[k], S::NW);
        for (int k = 0; k < S::NPUB; ++k) mbar_init(&pubA[k], S::NW);
        fence_mbar_init();
    }
    __syncthreads();

    const int n = p.nzl;
    const int tile = blockIdx.x;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int x0 = txi * TX, y0 = p.ya_lo + tyi * TY;
    const unsigned long long E =
        (*reinterpret_cast<volatile const unsigned long long*>(p.d_epoch) * p.nbands + p.band + 1) << 32;

    if (warp == S::NW) {  // ---------------- producer A: u^n boxes, (u^{n-1}, C) tiles
        if (lane == 0) {
            const uint64_t pol_first = policy_evict_first();
            auto put_u = [&](int j) {  // box plane j = buffer plane j (z = j - 5)
                const uint32_t slot = j % KA;
                if (j >= KA) mbar_wait_wd(smem_u32(&emptyA[slot]), ((j / KA) - 1) & 1);
                mbar_expect_tx(&fullA[slot], S::UBYTES);
                tma_load_3d(uA + slot * S::USLOT, &tmA_u, x0 - 8, y0 - 5, j, &fullA[slot]);
            };
            auto put_c = [&](int i) {  // u^{n-1} (read once) and C at plane i
                const uint32_t slot = i % DA;
                if (i >= DA) mbar_wait_wd(smem_u32(&emptyCA[slot]), ((i / DA) - 1) & 1);
                mbar_expect_tx(&fullCA[slot], S::CBYTES);
                float* dst = cA + slot * S::CSLOT;
                tma_load_3d_hint(dst, &tmA_up, x0, y0, i + 5, &fullCA[slot], pol_first);
                tma_load_3d(dst + TX * TY, &tm_c, x0, y0, i, &fullCA[slot]);
            };
            for (int j = 0; j < 10; ++j) put_u(j);
            for (int i = 0; i < n; ++i) {
                put_c(i);
                put_u(i + 10);
            }
        }
        return;
    }
    if (warp == S::NW + 1) {  // ---------------- producer B: u^{n+1} boxes, (u^n, C) tiles
        if (lane == 0) {
            const uint64_t pol_first = policy_evict_first();
            // stage-A progress of this CTA and its edge neighbours (the box's x/y halo)
            const unsigned long long* fl[5];
            int nfl = 0;
            fl[nfl++] = p.flags + tile;
            if (txi > 0) fl[nfl++] = p.flags + tile - 1;
            if (txi + 1 < p.tiles_x) fl[nfl++] = p.flags + tile + 1;
            if (tyi > 0) fl[nfl++] = p.flags + tile - p.tiles_x;
            if (tyi + 1 < p.tiles_y) fl[nfl++] = p.flags + tile + p.tiles_x;
            unsigned long long seen[5] = {0, 0, 0, 0, 0};
            auto wait_flags = [&](int need) {
                const unsigned long long want = E | (unsigned)need;
                bool fenced = true;
                for (int k = 0; k < nfl; ++k) {
                    if (seen[k] >= want) continue;
                    fenced = false;
                    unsigned long long v = ld_acquire_gpu_u64(fl[k]);
                    if (v < want) {
                        const unsigned long long t0 = globaltimer_ns();
                        do {
                            __nanosleep(32);
                            v = ld_acquire_gpu_u64(fl[k]);
                            if (v < want && globaltimer_ns() - t0 > kWatchdogNs) __trap();
                        } while (v < want);
                    }
                    seen[k] = v;
                }
                // generic-proxy stores (published) -> async-proxy (TMA) reads
                if (!fenced) fence_proxy_async_global();
            };
            auto put_u = [&](int j) {
                const uint32_t slot = j % KB;
                if (j >= KB) mbar_wait_wd(smem_u32(&emptyB[slot]), ((j / KB) - 1) & 1);
                mbar_expect_tx(&fullB[slot], S::UBYTES);
                tma_load_3d(uB + slot * S::USLOT, &tmB_u, x0 - 8, y0 - 5, j, &fullB[slot]);
            };
            auto put_c = [&](int i) {  // u^n and C at plane i: their last use
                const uint32_t slot = i % DB;
                if (i >= DB) mbar_wait_wd(smem_u32(&emptyCB[slot]), ((i / DB) - 1) & 1);
                mbar_expect_tx(&fullCB[slot], S::CBYTES);
                float* dst = cB + slot * S::CSLOT;
                tma_load_3d_hint(dst, &tmB_up, x0, y0, i + 5, &fullCB[slot], pol_first);
                tma_load_3d_hint(dst + TX * TY, &tm_c, x0, y0, i, &fullCB[slot], pol_first);
            };
            wait_flags(n < 5 ? n : 5);
            for (int j = 0; j < 10; ++j) put_u(j);
            for (int i = 0; i < n; ++i) {
                wait_flags(i + 6 < n ? i + 6 : n);
                put_c(i);
                put_u(i + 10);
            }
        }
        return;
    }
    if (warp == S::NW + 2) {  // ---------------- publisher: stage-A planes completed by the CTA
        // Waits (acquire.cta) for plane i on pubA, folds in any later planes already complete,
        // then releases flags[cta] at gpu scope: cumulative over the consumers' u^{n+1} stores.
        // Safe ring reuse: a consumer reaches A plane i + NPUB only after B plane i + NPUB - L,
        // which needs this CTA's flag >= i + NPUB - L + 6 > i + 1 (NPUB >= L + 16).
        if (lane == 0) {
            const uint32_t pb = smem_u32(pubA);
            int i = 0;
            while (i < n) {
                mbar_wait_wd(pb + 8 * (i % S::NPUB), (i / S::NPUB) & 1);
                ++i;
                while (i < n && mbar_try_wait(&pubA[i % S::NPUB], (i / S::NPUB) & 1)) ++i;
                st_release_gpu_u64(p.flags + tile, E | (unsigned)i);
            }
        }
        return;
    }

    // ---------------- consumer warps: stage A on plane it, stage B on plane it - L
    const int tx = tid % S::TXV, ty = tid / S::TXV;
    const int own = (5 + ty) * S::RS + 8 + 4 * tx;
    const int cown = ty * TX + 4 * tx;
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool inx = x < p.nx;
    const bool actA = inx && y < p.ya_hi && y < p.ny;
    const bool actB = inx && y >= p.yb_lo && y < p.yb_hi;
    const int nA = p.d_step[p.parity];  // samples of step n (A) and n+1 (B)
    uint64_t smask = 0;
    if (actA) {
        for (int s = 0; s < p.nsrc; ++s) {
            const DevSource& src = p.src[s];
            if (src.shot == 0 && src.y == y && src.x >= x && src.x < x + 4) smask |= (1ull << s);
        }
    }
    const long long col = (long long)y * p.nx + x;
    float* outA = p.outA + 5 * p.plane + col;
    float* outB = p.outB + 5 * p.plane + col;
    const uint32_t fA = smem_u32(fullA), eA = smem_u32(emptyA);
    const uint32_t fB = smem_u32(fullB), eB = smem_u32(emptyB);
    const uint32_t fCA = smem_u32(fullCA), eCA = smem_u32(emptyCA);
    const uint32_t fCB = smem_u32(fullCB), eCB = smem_u32(emptyCB);
    const uint32_t pub0 = smem_u32(pubA);
    const float* uAown = uA + own;
    const float* uBown = uB + own;

    float4 qA[10 + U], qB[10 + U];
#pragma unroll
    for (int j = 0; j < 10; ++j) {
        mbar_wait_wd(fA + 8 * (j % KA), (j / KA) & 1);
        qA[j] = *reinterpret_cast<const float4*>(uAown + (j % KA) * S::USLOT);
        if (j < 5) {
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(eA + 8 * (j % KA));
        }
    }
    uint32_t snA = 10 % KA, pnA = (10 / KA) & 1, scA = 5 % KA, sqA = 0, pqA = 0;
    uint32_t snB = 10 % KB, pnB = (10 / KB) & 1, scB = 5 % KB, sqB = 0, pqB = 0;
    const int total = n + L;
    int it = 0;
    auto body = [&](auto OFF) {
        constexpr int O = decltype(OFF)::value;
        if (it < n) {  // ---- stage A: u^{n+1} at plane it
            mbar_wait_wd(fA + 8 * snA, pnA);
            qA[O + 10] = *reinterpret_cast<const float4*>(uAown + snA * S::USLOT);
            mbar_wait_wd(fCA + 8 * sqA, pqA);
            const float* cb = cA + sqA * S::CSLOT + cown;
            const float4 upv = *reinterpret_cast<const float4*>(cb);
            const float4 cv = *reinterpret_cast<const float4*>(cb + TX * TY);
            float out[4];
            star4<S::RS, O>(uAown + scA * S::USLOT, qA, upv, cv, c, out);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_u32(eA + 8 * scA);
                mbar_arrive_u32(eCA + 8 * sqA);
            }
            if (smask) add_sources_n(p, smask, x, it, nA, out);
            if (actA) __stcg(reinterpret_cast<float4*>(outA), make_float4(out[0], out[1], out[2], out[3]));
            __syncwarp();  // the lanes' stores, then one release.cta arrive for the warp
            if (lane == 0) mbar_arrive_u32(pub0 + 8 * (it % S::NPUB));
            if (++snA == KA) snA = 0, pnA ^= 1;
            if (++scA == KA) scA = 0;
            if (++sqA == DA) sqA = 0, pqA ^= 1;
            outA += p.plane;
        }
        if (it >= L) {  // ---- stage B: u^{n+2} at plane it - L
            mbar_wait_wd(fB + 8 * snB, pnB);
            qB[O + 10] = *reinterpret_cast<const float4*>(uBown + snB * S::USLOT);
            mbar_wait_wd(fCB + 8 * sqB, pqB);
            const float* cb = cB + sqB * S::CSLOT + cown;
            const float4 upv = *reinterpret_cast<const float4*>(cb);
            const float4 cv = *reinterpret_cast<const float4*>(cb + TX * TY);
            float out[4];
            star4<S::RS, O>(uBown + scB * S::USLOT, qB, upv, cv, c, out);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_u32(eB + 8 * scB);
                mbar_arrive_u32(eCB + 8 * sqB);
            }
            if (smask) add_sources_n(p, smask, x, it - L, nA + 1, out);
            if (actB) st_stream4(outB, make_float4(out[0], out[1], out[2], out[3]));
            if (++snB == KB) snB = 0, pnB ^= 1;
            if (++scB == KB) scB = 0;
            if (++sqB == DB) sqB = 0, pqB ^= 1;
            outB += p.plane;
        }
        ++it;
    };
#pragma unroll 1
    for (int i = 0; i < total; i += U) {
        if (i == L) {  // stage-B queue prologue: u^{n+1} planes z = -5 .. 4
#pragma unroll
            for (int j = 0; j < 10; ++j) {
                mbar_wait_wd(fB + 8 * (j % KB), (j / KB) & 1);
                qB[j] = *reinterpret_cast<const float4*>(uBown + (j % KB) * S::USLOT);
                if (j < 5) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(eB + 8 * (j % KB));
                }
            }
        }
        if (!unrolled<0, U>(body, i, total)) break;
#pragma unroll
        for (int o = 0; o < 10; ++o) {
            qA[o] = qA[o + U];
            qB[o] = qB[o + U];
        }
    }
}

__global__ void k_tb_advance(int* d_step, int parity, unsigned long long* d_epoch) {
    d_step[parity] += 2;
    *d_epoch += 1;
}

// ------------------------------------------------------------------------------------
template <int TX, int TY, int KA, int KB, int DA, int DB, int L, int U>
static cudaError_t tb_prepare(const void** fn, int* threads, size_t* smem) {
    using S = TBShape<TX, TY, KA, KB, DA, DB>;
    *fn = reinterpret_cast<const void*>(&k_tb2<TX, TY, KA, KB, DA, DB, L, U>);
    *threads = S::NT;
    *smem = S::SMEM;
    return cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(*smem));
}

cudaError_t tb_variant_fn(int id, const void** fn, int* threads, size_t* smem) {
    switch (id) {
#define X(vid, name, tx, ty, ka, kb, da, db, l, u, pair) \
    case vid:                                            \
        return tb_prepare<tx, ty, ka, kb, da, db, l, u>(fn, threads, smem);
        RTM_TB_VARIANTS(X)
#undef X
        default:
            return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tb2(int id, const CUtensorMap tm[5], const TBParams& p, cudaStream_t s) {
    const void* fn;
    int threads;
    size_t smem;
    cudaError_t e = tb_variant_fn(id, &fn, &threads, &smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<CUtensorMap*>(&tm[0]), const_cast<CUtensorMap*>(&tm[1]),
                    const_cast<CUtensorMap*>(&tm[2]), const_cast<CUtensorMap*>(&tm[3]),
                    const_cast<CUtensorMap*>(&tm[4]), const_cast<TBParams*>(&p)};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(p.tiles_x * p.tiles_y));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident, or a launch error
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_tb_advance(int* d_step, int parity, unsigned long long* d_epoch, cudaStream_t s) {
    k_tb_advance<<<1, 1, 0, s>>>(d_step, parity, d_epoch);
    return cudaGetLastError();
}

}  // namespace rtm
