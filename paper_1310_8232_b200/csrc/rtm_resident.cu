// =====================================================================================
// k_resident: many time steps of the RTM 3D-model update (§2
// Algorithm 1) in ONE cooperative launch, for grids whose three fields live in L2 (C1 64^3:
// 3 MB of the 126 MB).  Per-step launches of k_stream are latency-bound there (~12 us per
// step for 16 us of work spread over 148 SMs); here all CTAs stay resident, each thread
// updates 4 x-consecutive points per step from L2 (ld.global.cg: 128-bit z / y neighbours and
// centre, 4 loads for the x neighbours, u_prev, C), the sources are added in the same
// epilogue, and a grid barrier separates the time steps.  The arithmetic is star4_core(),
// the same operations in the same order as k_stream, so results are bitwise identical.
// Zero Dirichlet halo: explicit z-halo planes, predicated x / y neighbours.
// =====================================================================================
#include "rtm_internal.h"
#include "rtm_device.cuh"

namespace rtm {

__device__ __forceinline__ float4 ldcg4(const float* p) {
    return __ldcg(reinterpret_cast<const float4*>(p));
}

__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier on a monotonically increasing arrival counter bar[0] (zeroed before the launch):
// barrier k of the launch is passed when bar[0] >= (k+1) * gridDim.x.  One release-add per CTA
// (its stores of the step happen-before the arrival) and acquire-polling; no reset and no
// generation flip by the last arriver (one L2 round trip less than a sense-reversing barrier).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = (gen + 1) * gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned long long t0 = 0;
        unsigned spins = 0;
        while (ld_acquire_gpu_u32(bar) < target) {
            if ((++spins & 255) == 0) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (!t0) t0 = t;
                else if (t - t0 > 4000000000ull) __trap();  // watchdog: error, never a hang
            }
        }
    }
    ++gen;
    __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT) k_resident(const __grid_constant__ ResParams p) {
    const float c[6] = {p.coef[0], p.coef[1], p.coef[2], p.coef[3], p.coef[4], p.coef[5]};
    const int nxq = p.pitch >> 2;  // 4-point groups per pitched row
    const long long per_shot = (long long)p.nzl * p.ny * nxq;
    const long long total = per_shot * p.nshots;
    const int n0 = p.d_step[p.parity0];
    unsigned gen = 0;
    for (int k = 0; k < p.nsteps; ++k) {
        const int par = (p.parity0 + k) & 1;
        const float* u = par ? p.buf1 : p.buf0;
        float* nxt = par ? p.buf0 : p.buf1;
        const int n = n0 + k;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
             t += (long long)gridDim.x * blockDim.x) {
            const int shot = static_cast<int>(t / per_shot);
            long long r = t - shot * per_shot;
            const int z = static_cast<int>(r / ((long long)p.ny * nxq));
            r -= (long long)z * p.ny * nxq;
            const int y = static_cast<int>(r / nxq);
            const int x = 4 * static_cast<int>(r - (long long)y * nxq);
            if (x >= p.nx) continue;  // a group of padding columns: stays zero
            const long long inpl = (long long)y * p.pitch + x;
            const long long base = ((long long)shot * (p.nzl + 10) + z + 5) * p.plane + inpl;
            float4 q[11];
#pragma unroll
            for (int o = 0; o < 11; ++o) q[o] = ldcg4(u + base + (long long)(o - 5) * p.plane);
            float4 yv[11];
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int m = 1; m <= 5; ++m) {
                yv[5 - m] = y - m >= 0 ? ldcg4(u + base - (long long)m * p.pitch) : zero;
                yv[5 + m] = y + m < p.ny ? ldcg4(u + base + (long long)m * p.pitch) : zero;
            }
            yv[5] = q[5];
            float xs[14];
            {
                const float4 l = x >= 4 ? ldcg4(u + base - 4) : zero;
                const float4 rr = x + 4 < p.nx ? ldcg4(u + base + 4) : zero;
                xs[0] = x >= 5 ? __ldcg(u + base - 5) : 0.0f;
                xs[1] = l.x; xs[2] = l.y; xs[3] = l.z; xs[4] = l.w;
                xs[5] = q[5].x; xs[6] = q[5].y; xs[7] = q[5].z; xs[8] = q[5].w;
                xs[9] = rr.x; xs[10] = rr.y; xs[11] = rr.z; xs[12] = rr.w;
                xs[13] = x + 8 < p.nx ? __ldcg(u + base + 8) : 0.0f;
            }
            const float4 upv = ldcg4(nxt + base);
            const float4 cv = ldcg4(p.C + (long long)z * p.plane + inpl);
            float out[4];
            star4_core<0>(q, yv, xs, upv, cv, c, out);
            for (int s = 0; s < p.nsrc; ++s) {  // a3, registration order
                const DevSource& src = p.src[s];
                if (src.shot == shot && src.z == z && src.y == y && src.x >= x && src.x < x + 4 &&
                    n < src.nsamples) {
                    const float w = p.samples[src.offset + n];
                    const int i = src.x - x;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        if (kk == i) out[kk] = __fadd_rn(out[kk], w);
                }
            }
            zero_pad(out, x, p.nx);
            __stcg(reinterpret_cast<float4*>(nxt + base), make_float4(out[0], out[1], out[2], out[3]));
        }
        grid_barrier(p.bar, gen);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) p.d_step[(p.parity0 + p.nsteps) & 1] = n0 + p.nsteps;
}

static const void* resident_fn(int threads) {
    switch (threads) {
        case 128: return reinterpret_cast<const void*>(&k_resident<128>);
        case 256: return reinterpret_cast<const void*>(&k_resident<256>);
        case 512: return reinterpret_cast<const void*>(&k_resident<512>);
        default: return nullptr;
    }
}

cudaError_t resident_occupancy(int threads, int* per_sm) {
    const void* fn = resident_fn(threads);
    if (!fn) return cudaErrorInvalidValue;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fn, threads, 0);
}

cudaError_t launch_resident(const ResParams& p, int ctas, int threads, cudaStream_t s) {
    if (p.nsteps <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(p.bar, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<ResParams*>(&p)};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(ctas));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident, or a launch error
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const void* fn = resident_fn(threads);
    if (!fn) return cudaErrorInvalidValue;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace rtm
