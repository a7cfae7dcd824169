// =====================================================================================
// k_tb2s: two time steps of the RTM 3D-model update (§2, Algorithm 1)
// per HBM pass — temporal blocking, SURVEY.md §8(f) f4 (§4 names time blocking
// among the related stencil optimisations).
//
// The single-step kernel (k_stream) moves 16 B per point update and runs at the HBM copy
// peak.  A two-step pass reads u^n, u^{n-1}, C once and writes u^{n+1}, u^{n+2}: 20 B per two
// updates, with the intermediate level u^{n+1} produced and consumed through L2:
//
//   * The grid is cut into y-bands; one launch per band.  Each tile of the band's A region
//     (the band's rows plus 5 rows each side) has a stage-A CTA (step n -> n+1) and a stage-B
//     CTA (step n+1 -> n+2); all CTAs are co-resident (cooperative launch, 2 per SM) and sweep
//     z from 0 to nz.  Rows of the A region outside the band are recomputed by the
//     neighbouring band (redundant work ~ 10 / band rows); both store bitwise-identical values.
//   * Both roles run k_stream's pipeline: a producer warp TMAs the halo'd u box and the
//     (u_prev, C) tiles into rings; consumer warps keep an 11-plane register queue along z and
//     compute star4() = k_stream's exact arithmetic, so results are bitwise identical to two
//     k_stream steps (tests/test_gpu_parity.py).
//   * Publication of u^{n+1} (stage A): consumers write each plane into a shared-memory
//     staging slot; a store warp issues one TMA tensor store per plane (async proxy end to
//     end) and, once the writes of plane i - W are complete (bulk wait_group), hands the plane
//     to a publisher warp that releases flagsA[tile] = epoch << 32 | planes at gpu scope.
//   * Stage-B producers acquire flagsA of their tile and its 4 edge neighbours (the box halo)
//     before each u^{n+1} load; stage B reports its progress (flagsB) to throttle stage A to
//     at most LMAX planes ahead, which bounds the L2 working set.
// Deadlock freedom: a throttled stage-A CTA still drains and publishes every plane it has
// loaded; stage B of plane j needs A planes <= j+5 < j + LMAX.  Every spin has a 4 s watchdog
// that traps (a launch error, never a hang).
// =====================================================================================
#include "rtm_internal.h"
#include "rtm_device.cuh"

namespace rtm {

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

// ====================================================================================
// k_tb2s: the same two-step pass with the two stages on separate CTAs (2 per SM).  CTA
// b < ntiles is the stage-A CTA of tile b, CTA ntiles + b the stage-B CTA of tile b; each is
// a k_stream pipeline (producer warp, TMA rings, consumer warps with the z register queue).
//   * Stage-A consumers write u^{n+1} into a shared-memory staging slot; a store warp issues
//     one TMA tensor store per plane (async proxy end to end: no per-warp memory fences),
//     and once bulk group i is complete publishes flagsA[tile] = E | (i+1) (proxy fence +
//     gpu-scope release).
//   * Stage-B producers acquire flagsA of the tile and its 4 edge neighbours before each TMA
//     load of the halo'd u^{n+1} box; stage-B CTAs publish their progress (flagsB, relaxed)
//     only to throttle stage A: A's producer keeps plane i within LMAX planes of B, which
//     bounds the L2 working set (u^{n+1} window and the u^n/C re-reads of stage B).
// Deadlock freedom: a throttled stage-A CTA still drains every plane it has loaded, so its
// published count reaches the plane its producer waits at; stage B of plane j needs A planes
// <= j+5 < j + LMAX (LMAX >= 7).  All CTAs are co-resident (cooperative launch).

template <int TX, int TY, int K, int D, int S>
struct TB2SShape {
    static constexpr int NW = TX * TY / 128;
    static constexpr int NT = (NW + 3) * 32;  // + producer, store warp, publisher warp
    static constexpr int TXV = TX / 4;
    static constexpr int RS = TX + 16;
    static constexpr int ROWS = TY + 10;
    static constexpr int USLOT = (RS * ROWS + 31) / 32 * 32;
    static constexpr uint32_t UBYTES = RS * ROWS * 4;
    static constexpr int CSLOT = 2 * TX * TY;
    static constexpr uint32_t CBYTES = CSLOT * 4;
    static constexpr int STSLOT = TX * TY;
    static constexpr int OFF_C = K * USLOT;
    static constexpr int OFF_ST = OFF_C + D * CSLOT;
    static constexpr size_t BAR_OFF = size_t(OFF_ST + S * STSLOT) * 4;
    static constexpr int NPUB = 32;  // B: per-plane completion; A: store-group completion
    static constexpr int NBAR = 2 * (K + D + S) + NPUB;
    static constexpr size_t SMEM = BAR_OFF + size_t(NBAR) * 8;
    static_assert((TX * TY) % 128 == 0 && K >= 7 && D >= 1 && S >= 2, "shape");
    static_assert(TX >= 8 && TY >= 5 && TX % 4 == 0 && RS <= 256 && ROWS <= 256, "TMA box / halo");
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const void* src, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(tm)),
        "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void add_sources_2s(const TB2SParams& p, uint64_t mask, int x, int z,
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

// W: TMA store groups whose writes may still be in flight when a plane is published (the
// publication lag); staging slots (S_ = 4) are recycled as soon as a store has read them.
// CH bit 0: stage A loads the u^n box and C with an evict_last L2 policy (stage B re-reads
// u^n and C with evict_first: their last use).
template <int TX, int TY, int K, int D, int U, int LMAX, int W, int CH>
__global__ void __launch_bounds__(TB2SShape<TX, TY, K, D, 4>::NT, 2)
    k_tb2s(const __grid_constant__ CUtensorMap tmA_u, const __grid_constant__ CUtensorMap tmA_up,
           const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tmB_u,
           const __grid_constant__ CUtensorMap tmB_up, const __grid_constant__ CUtensorMap tmA_st,
           const __grid_constant__ TB2SParams p) {
    constexpr int S_ = 4;
    using S = TB2SShape<TX, TY, K, D, S_>;
    static_assert(LMAX >= 7, "stage A may run at most LMAX planes ahead of stage B");
    static_assert(W >= 1 && W < S::NPUB, "store groups in flight");
    extern __shared__ __align__(128) float smem[];
    float* uring = smem;
    float* cring = smem + S::OFF_C;
    float* stg = smem + S::OFF_ST;
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + S::BAR_OFF);
    uint64_t* full_u = bars;
    uint64_t* empty_u = full_u + K;
    uint64_t* full_c = empty_u + K;
    uint64_t* empty_c = full_c + D;
    uint64_t* staged = empty_c + D;
    uint64_t* stfree = staged + S_;
    uint64_t* pub = stfree + S_;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < K; ++k) mbar_init(&full_u[k], 1), mbar_init(&empty_u[k], S::NW);
        for (int k = 0; k < D; ++k) mbar_init(&full_c[k], 1), mbar_init(&empty_c[k], S::NW);
        for (int k = 0; k < S_; ++k) mbar_init(&staged[k], S::NW), mbar_init(&stfree[k], 1);
        for (int k = 0; k < S::NPUB; ++k) mbar_init(&pub[k], (int)blockIdx.x < p.ntiles ? 1 : S::NW);
        fence_mbar_init();
    }
    __syncthreads();

    const bool isA = (int)blockIdx.x < p.ntiles;
    const int tile = isA ? blockIdx.x : blockIdx.x - p.ntiles;
    const int n = p.nzl;
    const int tyi = tile / p.tiles_x, txi = tile - tyi * p.tiles_x;
    const int x0 = txi * TX, y0 = p.ya_lo + tyi * TY;
    const unsigned long long E =
        (*reinterpret_cast<volatile const unsigned long long*>(p.d_epoch) * p.nbands + p.band + 1) << 32;
    const CUtensorMap* tm_u = isA ? &tmA_u : &tmB_u;
    const CUtensorMap* tm_up = isA ? &tmA_up : &tmB_up;

    if (warp == S::NW) {  // ---------------- producer
        if (lane == 0) {
            const uint64_t pol_first = policy_evict_first();
            const uint64_t pol_last = policy_evict_last();
            const bool keep = isA && (CH & 1);
            const unsigned long long* fl[5];
            int nfl = 0;
            if (isA) {
                fl[nfl++] = p.flagsB + tile;
            } else {
                fl[nfl++] = p.flagsA + tile;
                if (txi > 0) fl[nfl++] = p.flagsA + tile - 1;
                if (txi + 1 < p.tiles_x) fl[nfl++] = p.flagsA + tile + 1;
                if (tyi > 0) fl[nfl++] = p.flagsA + tile - p.tiles_x;
                if (tyi + 1 < p.tiles_y) fl[nfl++] = p.flagsA + tile + p.tiles_x;
            }
            unsigned long long seen[5] = {0, 0, 0, 0, 0};
            // A: throttle to B's progress (relaxed); B: acquire A's published planes
            auto wait_flags = [&](int need) {
                if (need <= 0) return;
                const unsigned long long want = E | (unsigned)need;
                bool fresh = false;
                for (int k = 0; k < nfl; ++k) {
                    if (seen[k] >= want) continue;
                    fresh = true;
                    unsigned long long v = isA ? ld_relaxed_gpu_u64(fl[k]) : ld_acquire_gpu_u64(fl[k]);
                    if (v < want) {
                        const unsigned long long t0 = globaltimer_ns();
                        do {
                            __nanosleep(32);
                            v = isA ? ld_relaxed_gpu_u64(fl[k]) : ld_acquire_gpu_u64(fl[k]);
                            if (v < want && globaltimer_ns() - t0 > kWatchdogNs) __trap();
                        } while (v < want);
                    }
                    seen[k] = v;
                }
                if (fresh && !isA) fence_proxy_async_global();
            };
            auto put_u = [&](int j) {
                const uint32_t slot = j % K;
                if (j >= K) mbar_wait_wd(smem_u32(&empty_u[slot]), ((j / K) - 1) & 1);
                mbar_expect_tx(&full_u[slot], S::UBYTES);
                if (keep)
                    tma_load_3d_hint(uring + slot * S::USLOT, tm_u, x0 - 8, y0 - 5, j, &full_u[slot], pol_last);
                else
                    tma_load_3d(uring + slot * S::USLOT, tm_u, x0 - 8, y0 - 5, j, &full_u[slot]);
            };
            auto put_c = [&](int i) {  // u_prev (read once) and C at plane i
                const uint32_t slot = i % D;
                if (i >= D) mbar_wait_wd(smem_u32(&empty_c[slot]), ((i / D) - 1) & 1);
                mbar_expect_tx(&full_c[slot], S::CBYTES);
                float* dst = cring + slot * S::CSLOT;
                tma_load_3d_hint(dst, tm_up, x0, y0, i + 5, &full_c[slot], pol_first);
                if (keep)
                    tma_load_3d_hint(dst + TX * TY, &tm_c, x0, y0, i, &full_c[slot], pol_last);
                else if (isA)
                    tma_load_3d(dst + TX * TY, &tm_c, x0, y0, i, &full_c[slot]);
                else
                    tma_load_3d_hint(dst + TX * TY, &tm_c, x0, y0, i, &full_c[slot], pol_first);
            };
            if (!isA) wait_flags(n < 5 ? n : 5);
            for (int j = 0; j < 10; ++j) put_u(j);
            for (int i = 0; i < n; ++i) {
                if (isA) wait_flags(i - LMAX);
                else wait_flags(i + 6 < n ? i + 6 : n);
                put_c(i);
                put_u(i + 10);
            }
        }
        return;
    }
    if (warp == S::NW + 1) {  // ---------------- A: TMA stores; B: progress (throttle)
        if (lane == 0) {
            if (isA) {
                // store plane i, recycle the slot of plane i - S_ + 1 once read, and signal
                // pub[(i - W) % NPUB] once the writes of plane i - W are complete.  The gpu-scope
                // release is left to the publisher warp: a release here would wait for every
                // store this thread has in flight (MEMBAR.GPU), serialising the W-deep pipeline.
                for (int i = 0; i < n; ++i) {
                    const int slot = i % S_;
                    mbar_wait_wd(smem_u32(&staged[slot]), (i / S_) & 1);
                    tma_store_3d(&tmA_st, stg + slot * S::STSLOT, x0, y0, i + 5);
                    bulk_commit();
                    bulk_wait_read<S_ - 1>();  // the store of plane i - S_ + 1 has read its slot
                    if (i >= S_ - 1) mbar_arrive(&stfree[(i - S_ + 1) % S_]);
                    if (i >= W) {
                        bulk_wait<W>();  // the writes of planes <= i - W are complete
                        fence_proxy_async_global();
                        mbar_arrive(&pub[(i - W) % S::NPUB]);
                    }
                }
                bulk_wait<0>();
                fence_proxy_async_global();
                for (int i = n - W < 0 ? 0 : n - W; i < n; ++i) mbar_arrive(&pub[i % S::NPUB]);
            } else {
                int i = 0;
                while (i < n) {
                    mbar_wait_wd(smem_u32(&pub[i % S::NPUB]), (i / S::NPUB) & 1);
                    ++i;
                    while (i < n && mbar_try_wait(&pub[i % S::NPUB], (i / S::NPUB) & 1)) ++i;
                    st_relaxed_gpu_u64(p.flagsB + tile, E | (unsigned)i);
                }
            }
        }
        return;
    }
    if (warp == S::NW + 2) {  // ---------------- A: publish completed u^{n+1} planes (acquire
        if (lane == 0 && isA) {  // the store warp's completion, release at gpu scope)
            int i = 0;
            while (i < n) {
                mbar_wait_wd(smem_u32(&pub[i % S::NPUB]), (i / S::NPUB) & 1);
                ++i;
                while (i < n && mbar_try_wait(&pub[i % S::NPUB], (i / S::NPUB) & 1)) ++i;
                fence_proxy_async_global();
                st_release_gpu_u64(p.flagsA + tile, E | (unsigned)i);
            }
        }
        return;
    }

    // ---------------- consumers (k_stream's loop, one stage)
    const int tx = tid % S::TXV, ty = tid / S::TXV;
    const int own = (5 + ty) * S::RS + 8 + 4 * tx;
    const int cown = ty * TX + 4 * tx;
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};
    const int x = x0 + 4 * tx, y = y0 + ty;
    const bool inx = x < p.nx;
    const bool actB = !isA && inx && y >= p.yb_lo && y < p.yb_hi;
    const int nS = p.d_step[p.parity] + (isA ? 0 : 1);  // sample index of this stage's step
    uint64_t smask = 0;
    if (inx && y < p.ny) {  // A: every grid row it stores is exact (sources included)
        for (int s = 0; s < p.nsrc; ++s) {
            const DevSource& src = p.src[s];
            if (src.shot == 0 && src.y == y && src.x >= x && src.x < x + 4) smask |= (1ull << s);
        }
    }
    const long long col = (long long)y * p.pitch + x;
    float* outB = p.outB + 5 * p.plane + col;
    const uint32_t fu = smem_u32(full_u), eu = smem_u32(empty_u);
    const uint32_t fc = smem_u32(full_c), ec = smem_u32(empty_c);
    const uint32_t stg0 = smem_u32(staged), sfr0 = smem_u32(stfree), pub0 = smem_u32(pub);
    const float* uown = uring + own;

    float4 q[10 + U];
#pragma unroll
    for (int j = 0; j < 10; ++j) {
        mbar_wait_wd(fu + 8 * (j % K), (j / K) & 1);
        q[j] = *reinterpret_cast<const float4*>(uown + (j % K) * S::USLOT);
        if (j < 5) {
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(eu + 8 * (j % K));
        }
    }
    uint32_t sn = 10 % K, pn = (10 / K) & 1, sc = 5 % K, sq = 0, pq = 0;
    int it = 0;
    auto body = [&](auto OFF) {
        constexpr int O = decltype(OFF)::value;
        mbar_wait_wd(fu + 8 * sn, pn);
        q[O + 10] = *reinterpret_cast<const float4*>(uown + sn * S::USLOT);
        mbar_wait_wd(fc + 8 * sq, pq);
        const float* cb = cring + sq * S::CSLOT + cown;
        const float4 upv = *reinterpret_cast<const float4*>(cb);
        const float4 cv = *reinterpret_cast<const float4*>(cb + TX * TY);
        float out[4];
        star4<S::RS, O>(uown + sc * S::USLOT, q, upv, cv, c, out);
        __syncwarp();
        if (lane == 0) {
            mbar_arrive_u32(eu + 8 * sc);
            mbar_arrive_u32(ec + 8 * sq);
        }
        if (smask) add_sources_2s(p, smask, x, it, nS, out);
        zero_pad(out, x, p.nx);  // (A: the TMA store clips at nx anyway)
        const float4 o4 = make_float4(out[0], out[1], out[2], out[3]);
        if (isA) {
            const int slot = it % S_;
            if (it >= S_) mbar_wait_wd(sfr0 + 8 * slot, ((it / S_) - 1) & 1);
            *reinterpret_cast<float4*>(stg + slot * S::STSLOT + cown) = o4;
            fence_proxy_async_smem();  // generic smem writes -> the TMA store's async reads
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(stg0 + 8 * slot);
        } else {
            if (actB) st_stream4(outB, o4);
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(pub0 + 8 * (it % S::NPUB));
        }
        if (++sn == K) sn = 0, pn ^= 1;
        if (++sc == K) sc = 0;
        if (++sq == D) sq = 0, pq ^= 1;
        outB += p.plane;
        ++it;
    };
#pragma unroll 1
    for (int i = 0; i < n; i += U) {
        if (!unrolled<0, U>(body, i, n)) break;
#pragma unroll
        for (int o = 0; o < 10; ++o) q[o] = q[o + U];
    }
}

__global__ void k_tb_advance(int* d_step, int parity, unsigned long long* d_epoch) {
    d_step[parity] += 2;
    *d_epoch += 1;
}

// ------------------------------------------------------------------------------------
template <int TX, int TY, int K, int D, int U, int LMAX, int W, int CH>
static cudaError_t tb2s_prepare(const void** fn, int* threads, size_t* smem) {
    using S = TB2SShape<TX, TY, K, D, 4>;
    *fn = reinterpret_cast<const void*>(&k_tb2s<TX, TY, K, D, U, LMAX, W, CH>);
    *threads = S::NT;
    *smem = S::SMEM;
    return cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(*smem));
}

cudaError_t tb2s_variant_fn(int id, const void** fn, int* threads, size_t* smem) {
    switch (id) {
#define X(vid, name, tx, ty, k, d, u, lmax, w, ch, pair) \
    case vid:                                              \
        return tb2s_prepare<tx, ty, k, d, u, lmax, w, ch>(fn, threads, smem);
        RTM_TB2S_VARIANTS(X)
#undef X
        default:
            return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tb2s(int id, const CUtensorMap tm[6], const TB2SParams& p, cudaStream_t s) {
    const void* fn;
    int threads;
    size_t smem;
    cudaError_t e = tb2s_variant_fn(id, &fn, &threads, &smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<CUtensorMap*>(&tm[0]), const_cast<CUtensorMap*>(&tm[1]),
                    const_cast<CUtensorMap*>(&tm[2]), const_cast<CUtensorMap*>(&tm[3]),
                    const_cast<CUtensorMap*>(&tm[4]), const_cast<CUtensorMap*>(&tm[5]),
                    const_cast<TB2SParams*>(&p)};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * p.ntiles));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
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
