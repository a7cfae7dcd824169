// Internal interface between the host library (rtm_host.cpp) and the kernels (rtm_kernels.cu).
// Not installed, not part of the C ABI (include/rtm.h is).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/rtm.h"

namespace rtm {

constexpr int RADIUS = 5;  // "five points (cells) in each direction"

struct DevSource {       // a source owned by this slab, LOCAL coordinates
    int x, y, z;         // z = owned plane index (0..nzl-1)
    int shot;            // wavefield index in a batched (multi-shot) context
    int nsamples;
    long long offset;    // into StencilParams::samples
};

// Everything a stencil launch needs.  Passed by value (__grid_constant__).
struct StencilParams {
    int nx, ny, nzl;           // interior extents of this slab
    int pitch;                 // row stride in floats: nx rounded up to a multiple of 4; the
                               // padding columns [nx, pitch) are zero at all times
    long long plane;           // pitch*ny
    int nshots;                // independent wavefields sharing C (batched shots); shot k's
                               // planes start at buffer plane k*(nzl+10)
    float coef[6];             // coef[0] = 3*c0 (fp32, host-folded), coef[1..5] = c1..c5
    const float* u;            // u^n buffer base (nzl+10 planes, plane 0 = first halo plane)
    float* next;               // u^{n-1} buffer base, overwritten in place by u^{n+1}
    const float* C;            // C(p), nzl planes
    int* d_step;               // step counter slots [2]; this launch reads d_step[parity]
    int parity;                // (global step) & 1
    int write_next;            // 1: block 0 writes d_step[parity^1] = n + 1
    int nranges;               // 1 or 2 z-ranges of owned planes
    int r_begin[2], r_len[2];  // ranges [r_begin, r_begin + r_len)
    int r_chunks[2];           // z-chunks per range (tiled kernel work units)
    int tiles_x, tiles_y;      // tiled kernel: xy tiles
    int cache_mode;            // k_stream L2 policy knobs (see rtm_kernels.cu)
    int zalt;                  // k_stream: RTM_OPT_ZDIR bits (downward sweeps: odd steps / odd waves)
    int shot_major;            // 1: units ordered shot-slowest (each shot's tiles co-run);
                               // 0: shot-fastest (co-running CTAs share the C tile)
    // fused halo push (f1, in-process multi-slab): when non-null, owned planes [0,5) are also
    // stored to push_lo + z*plane and planes [nzl-5, nzl) to push_hi + (z-nzl+5)*plane — the
    // neighbours' z-halo planes of their u^{n+1} buffers (peer or same-device pointers)
    float* push_lo;
    float* push_hi;
    // multi-step launches (kind 6, k_stream<..., MS = true>): nsteps time steps in ONE
    // cooperative launch, step k reading buf (parity + k) & 1 (u = k even ? u : next); the step
    // index of step k is step0 + k; a unit may start step k once it and its x/y/z neighbour
    // units have published flags[unit] >= epoch | k (epoch: a per-launch tag in the upper 32 bits)
    int nsteps;
    int step0;
    unsigned long long epoch;
    unsigned long long* flags;
    int nsrc;
    DevSource src[RTM_MAX_SOURCES];
    const float* samples;
};

struct TileVariant {
    const char* name;
    int kind;                  // 0 naive, 1 k_tiled (CTA per unit), 2 k_stream (persistent, producer
                               // warp), 4 k_tb2s (two time steps per HBM pass),
                               // 5 k_resident (many steps per launch, L2-resident grids),
                               // 6 k_stream multi-step (many steps per cooperative launch, units
                               //   ordered by neighbour flags instead of launch boundaries),
                               // 7 k_stream2 (two rows per consumer thread, rtm_stream2.cu)
    int TX, TY, K, D, MINB;    // tile (x, y), u ring depth, u_prev/C ring depth (0: LDG), min CTAs/SM
    int U;                     // z-loop unroll (register-queue rotation amortised over U planes)
    int KB, DB, L;             // kind 4: KB = W (store groups in flight before publication),
                               // DB = L2 hint bits, L = LMAX (stage-A lead bound, planes)
    int pair;                  // kind 4: the k_stream variant that runs single (odd) steps
};


// Split-role two-step (kind 4) variants: X(id, name, TX, TY, K, D, U, LMAX, W, CH, pair)
#define RTM_TB2S_VARIANTS(X)                                              \
    X(37, "tb2s_64x16k8d3l24w6u4", 64, 16, 8, 3, 4, 24, 6, 0, 35)         \
    X(38, "tb2s_64x16k8d3l40w6u4", 64, 16, 8, 3, 4, 40, 6, 0, 35)         \
    X(39, "tb2s_64x16k8d3l56w16u4", 64, 16, 8, 3, 4, 56, 16, 0, 35)

// Resident (kind 5) variants: X(id, name, threads, ctas_per_sm, pair)
#define RTM_RESIDENT_VARIANTS(X)                          \
    X(40, "resident256x2", 256, 2, 35)                    \
    X(41, "resident128x4", 128, 4, 35)                    \
    X(42, "resident512x1", 512, 1, 35)

// Two-row streaming (kind 7, k_stream2 in rtm_stream2.cu) variants: X(id, name, TX, TY, K, D, MINB).
// Warps per SM stay a multiple of 4 (8): the register file is split per SM sub-partition, so a
// 9th warp would cap every thread at 168 registers and spill the two z queues.
#define RTM_STREAM2_VARIANTS(X)                        \
    X(51, "s2r64x28k10d6", 64, 28, 10, 6, 1)            \
    X(52, "s2r128x14k8d4", 128, 14, 8, 4, 1)            \
    X(53, "s2r64x12k10d6", 64, 12, 10, 6, 2)            \
    X(54, "s2r128x6k8d5", 128, 6, 8, 5, 2)
cudaError_t stream2_variant_fn(int id, const void** fn, int* threads, size_t* smem);

// Variant table: index 0 is the naive kernel.
int num_variants();
const TileVariant& variant(int id);

size_t variant_smem_bytes(int id);
// Max resident blocks per SM (after opting in to the variant's smem), or < 0 on error.
int variant_occupancy(int id, int* threads_per_block);

// tm_u: u^n with the (TX+16) x (TY+10) halo box; tm_up: u^{n-1} and tm_c: C with TX x TY
// boxes (k_stream with D > 0).  max_ctas bounds the persistent grid.
// pdl: programmatic dependent launch (k_stream only): the grid may be scheduled while the
// previous kernel on the stream drains; it waits (griddepcontrol.wait) before touching memory.
cudaError_t launch_variant(int id, const CUtensorMap* tm_u, const CUtensorMap* tm_up,
                           const CUtensorMap* tm_c, const StencilParams& p, int max_ctas,
                           cudaStream_t s, bool pdl = false);
cudaError_t launch_naive(const StencilParams& p, cudaStream_t s);
// kind 6: p.nsteps steps from buffers (p.u, p.next) in one cooperative launch; tm_u / tm_up
// over p.u's buffer as the u box / u_prev tile at even steps (tm_u over p.u, tm_up over
// p.next), tm_u2 / tm_up2 the same for odd steps (tm_u2 over p.next, tm_up2 over p.u).
cudaError_t launch_mstep(int id, const CUtensorMap* tm_u, const CUtensorMap* tm_up,
                         const CUtensorMap* tm_u2, const CUtensorMap* tm_up2, const CUtensorMap* tm_c,
                         const StencilParams& p, int max_ctas, cudaStream_t s);

// Resident multi-step kernel (kind 5, k_resident in rtm_resident.cu): nsteps time steps of a
// single-slab context in one cooperative launch, grid barrier (bar[0..1], zeroed by the
// launcher) between steps; buffers alternate starting from buf[parity0] = u^n.
struct ResParams {
    int nx, ny, nzl, nshots;
    int pitch;
    long long plane;
    float coef[6];
    float* buf0;
    float* buf1;
    const float* C;
    int* d_step;
    int parity0;
    int nsteps;
    unsigned* bar;             // [2]: grid barrier arrival counter (zeroed per launch), spare
    int nsrc;
    DevSource src[RTM_MAX_SOURCES];
    const float* samples;
};
cudaError_t launch_resident(const ResParams& p, int ctas, int threads, cudaStream_t s);
cudaError_t resident_occupancy(int threads, int* per_sm);

// Split-role two-step pass (kind 4, k_tb2s in rtm_tb.cu): stage-A and stage-B CTAs of each
// tile (2 per SM); stage A publishes u^{n+1} planes through TMA stores (flagsA), stage B
// reports progress (flagsB) that throttles stage A.
struct TB2SParams {
    int nx, ny, nzl;
    int pitch;
    long long plane;
    float coef[6];
    float* outB;                        // u^{n+2} (stage-B STG stores, band rows only)
    const int* d_step;
    int parity;
    unsigned long long* flagsA;         // [ntiles] stage-A published planes
    unsigned long long* flagsB;         // [ntiles] stage-B completed planes (throttle only)
    const unsigned long long* d_epoch;
    int band, nbands, ntiles;
    int tiles_x, tiles_y;
    int ya_lo, ya_hi, yb_lo, yb_hi;
    int nsrc;
    DevSource src[RTM_MAX_SOURCES];
    const float* samples;
};

// kind 4: tm[0] u^n box (TX+16)x(TY+10), tm[1] u^{n-1} tile, tm[2] C tile, tm[3] u^{n+1} box,
// tm[4] u^n tile, tm[5] u^{n+1} TX x TY box (TMA store).  Grid 2 * p.ntiles, cooperative.
cudaError_t launch_tb2s(int id, const CUtensorMap tm[6], const TB2SParams& p, cudaStream_t s);
cudaError_t tb2s_variant_fn(int id, const void** fn, int* threads, size_t* smem);
// after the last band of a pass: d_step[parity] += 2, ++*d_epoch
cudaError_t launch_tb_advance(int* d_step, int parity, unsigned long long* d_epoch, cudaStream_t s);

// a1: C = fp32((double(v)*dt/dx)^2), stats[0] = max(v) bits (v > 0), stats[1] = count of
// invalid (non-finite or <= 0) velocities.  v and C may alias.
// Field check: stats[0] = max |u| bits (uint order of non-negative floats), stats[1] = number of
// non-finite values, over the owned planes of every shot in a slab buffer.
cudaError_t launch_field_stats(const float* buf, long long plane, int nzl, int nshots,
                               unsigned int* stats, cudaStream_t s);
// v and C are pitched (row stride pitch floats, n = pitch * rows); padding columns x >= nx get
// C = 0 and do not enter the statistics.
cudaError_t launch_velocity(const float* v, float* C, long long n, int nx, int pitch, double dt,
                            double dx, unsigned int* stats, cudaStream_t s);
// st.release.sys of v into *lo and *hi (either may be null) after a system fence
cudaError_t launch_signal(unsigned long long* lo, unsigned long long* hi, unsigned long long v,
                          cudaStream_t s);

}  // namespace rtm
