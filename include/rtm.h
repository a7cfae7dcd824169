/* =====================================================================================
 * rtm.h — C ABI of the B200-native RTM 3D-model time step (arxiv 1310.8232).
 *
 * The operation (§2 "3D Stencil Computations": finite differences, "10th
 * order in space and 2nd order in time", a stencil that "refers to five points (cells)
 * in each direction for each dimension"; Algorithm 1 line "forall points:
 * calculate 3D model", 99% of RTM time):
 *
 *     u^{n+1}(p) = 2 u^n(p) - u^{n-1}(p) + C(p) * sum_{axis} sum_{o=-5..5} c_|o| u^n(p + o e_axis)
 *     C(p)       = fp32( (double(v(p)) * double(dt) / double(dx))^2 )        (a1)
 *     u^{n+1}(p_s) += w_s[n]   for each registered source s, in registration order (a3)
 *
 * with a 5-cell zero (Dirichlet) halo around the nx*ny*nz interior.  Coefficients, halo,
 * source form and precision are the readings R1-R16 of DESIGN.md (the paper is silent on
 * them; BASELINE.json configs[0] fixes c0..c5).  Arithmetic is fp32 on the GPU.
 *
 * Layout: every host array is the unpadded interior, x fastest, then y, then z:
 *     index(x, y, z) = (z * ny + y) * nx + x          (float32)
 *
 * Conventions
 *  - Every int-returning call returns RTM_OK (0) or a negative RTM_E* code.  Nothing
 *    throws or aborts across the ABI.  rtm_last_error() returns a thread-local message
 *    naming the offending argument or the failing CUDA/NCCL call.
 *  - Ownership: the caller owns every host (and user device) buffer it passes; the library
 *    copies what it needs before returning.  The context owns its device memory, streams,
 *    events, graphs and NCCL communicator; rtm_destroy releases them.
 *  - A context is used by one host thread at a time ("confined to one worker").
 *  - No CPU fallback: every step of the path runs in the library's sm_100a kernels.  A
 *    context cannot be created without a CUDA device (rtm_create returns NULL, RTM_ECUDA).
 * ===================================================================================== */
#ifndef RTM_H_
#define RTM_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rtm_ctx rtm_ctx; /* opaque; owned by the library */

enum {
    RTM_OK = 0,
    RTM_EINVAL = -1, /* invalid argument (sizes, non-finite values, coordinates, ids)       */
    RTM_ECFL = -2,   /* max(v)*dt/dx exceeds nu_crit(coeffs) = 2/sqrt(3*S_max)              */
    RTM_ENOMEM = -3, /* device or host allocation failed                                    */
    RTM_ECUDA = -4,  /* a CUDA runtime/driver call or kernel failed                          */
    RTM_ENCCL = -5,  /* an NCCL call failed                                                  */
    RTM_ESTATE = -6, /* call not valid in this state (e.g. rtm_step before rtm_set_velocity) */
    RTM_EUNSTABLE = -7 /* the field check (RTM_OPT_CHECK_EVERY) found a non-finite value      */
};

#define RTM_MAX_SOURCES 64

/* ---- north-star entry points (BASELINE.json north_star) ------------------------------ */

/* Create a single-GPU context on the current CUDA device for an nx*ny*nz interior grid.
 * dx > 0 (m), dt > 0 (s) finite; coeffs[0..5] = c0..c5 finite, with S_max > 0 (a valid
 * negative-definite 2nd difference).  Allocates u, u_prev (each px*ny*(nz+10) floats:
 * 5 explicit zero z-halo planes per side) and C (px*ny*nz floats), zero-initialised, where
 * px = nx rounded up to a multiple of 4 is the device row pitch (any nx >= 1 runs every
 * kernel; the padding columns stay zero; host arrays are always unpadded, nx per row).
 * Returns NULL on error (see rtm_last_error()). */
rtm_ctx* rtm_create(int nx, int ny, int nz, float dx, float dt, const float coeffs[6]);

/* Host velocity v (m/s), nx*ny*nz_local floats (the whole grid, or this rank's slab for
 * rtm_create_dist).  Copied to the device, where a kernel computes C(p) in fp64 and rounds
 * once to fp32 (a1).  Every v must be finite and > 0 (RTM_EINVAL) and
 * max(v)*dt/dx <= nu_crit (RTM_ECFL, nu_crit = 5/sqrt(128) for the configs' coefficients).
 * On error no velocity is installed. */
int rtm_set_velocity(rtm_ctx* ctx, const float* v);

/* Register a point source at GLOBAL interior coordinates (ix, iy, iz).  samples[n]
 * (nsamples >= 0 floats, host, copied) is added to u^{n+1}(p_s) right after the stencil of
 * step n (n counted from the last rtm_reset/rtm_set_fields), for n < nsamples (a3).
 * Sources at the same point add in registration order.  At most RTM_MAX_SOURCES.
 * Coordinates outside the interior or a non-finite sample -> RTM_EINVAL.  In a distributed
 * context every rank registers every source; a rank keeps the ones it owns. */
int rtm_inject_source(rtm_ctx* ctx, int ix, int iy, int iz, const float* samples, int nsamples);

/* Advance nsteps >= 0 time steps.  Returns after device completion (surfaces asynchronous
 * errors).  RTM_ESTATE before rtm_set_velocity. */
int rtm_step(rtm_ctx* ctx, int nsteps);

/* Copy the current field u^n to host out (nx*ny*nz_local floats; the whole grid for
 * multi-slab contexts, this rank's slab for distributed ones). */
int rtm_read_field(rtm_ctx* ctx, float* out);

void rtm_destroy(rtm_ctx* ctx);
const char* rtm_last_error(void);

/* ---- extensions (tests, bench, multi-GPU; not in the north-star list) ----------------- */

/* Initial conditions / resume: u^0 = u, u^{-1} = u_prev (host, nx*ny*nz_local each; either
 * may be NULL = zero).  Resets the step counter to 0. */
int rtm_set_fields(rtm_ctx* ctx, const float* u, const float* u_prev);
/* Read both time levels (u^n, u^{n-1}); either pointer may be NULL. */
int rtm_read_fields(rtm_ctx* ctx, float* u, float* u_prev);
/* u = u_prev = 0 and step = 0; keeps velocity, sources and tile choice. */
int rtm_reset(rtm_ctx* ctx);
/* Extents of the host arrays this context reads and writes (host-only query, no device
 * work): *nx, *ny, *nzl (this rank's / slab set's planes: nz for single-GPU, batched and
 * multi-slab contexts, the slab's nzl for a distributed rank) and *nshots (1 unless batched).
 * Field arrays hold nshots*nzl*ny*nx floats, the velocity nzl*ny*nx.  Any pointer may be
 * NULL.  The Python binding validates every host array against it. */
int rtm_get_dims(rtm_ctx* ctx, int* nx, int* ny, int* nzl, int* nshots);
/* Number of steps taken since the last reset / set_fields. */
long long rtm_step_count(rtm_ctx* ctx);
/* Checkpoint / resume: after rtm_set_fields(u^n, u^{n-1}) of a saved state, set the step index
 * n so source samples continue at samples[n] (n >= 0). */
int rtm_set_step_count(rtm_ctx* ctx, long long n);
/* Failure detection: max |u^n| and the number of non-finite values of the current field
 * (device reduction; all slabs).  With RTM_OPT_CHECK_EVERY = k > 0, rtm_step runs this check
 * every k steps and returns RTM_EUNSTABLE at the first non-finite value. */
int rtm_field_stats(rtm_ctx* ctx, double* max_abs, long long* nonfinite);

/* Device-resident variants (the bench's kernel-only leg): d_v / d_out are device pointers
 * on the context's device (single-slab contexts only), same layout as the host versions.
 * Enqueued on the context's stream; d_v must stay valid until the next synchronising call. */
int rtm_set_velocity_device(rtm_ctx* ctx, const float* d_v);
int rtm_read_field_device(rtm_ctx* ctx, float* d_out);

/* Asynchronous host-buffer pipeline (single-slab contexts: single-GPU, batched, or one rank of
 * a distributed context).  These calls only ENQUEUE work and return; host buffers must stay
 * valid and unmodified (v) / unread (out) until the next rtm_sync.  Pinned host memory makes
 * the copies truly asynchronous: the H2D of the next velocity and the D2H of the previous result
 * then overlap the stencil steps (an H2D and a D2H copy stream plus a device staging buffer and
 * a device snapshot buffer, each nx*ny*nz floats, allocated on first use).
 *   rtm_set_velocity_async: H2D of v into the staging buffer, then a1 (C(p) and the validity /
 *       CFL reduction) on the context's stream after the work already enqueued; steps enqueued
 *       afterwards use the new model.  The verdict (RTM_EINVAL non-finite/non-positive values,
 *       RTM_ECFL) is DEFERRED to the next rtm_sync (or synchronising call: rtm_step,
 *       rtm_set_velocity), which then returns it and marks the velocity unset; steps run in
 *       between used the rejected model.
 *   rtm_step_async: rtm_step without the final synchronisation (no field check / profiling).
 *   rtm_read_field_async: snapshot of u^n (device copy, ordered after the steps enqueued so
 *       far) and its D2H into out on the copy stream.
 *   rtm_sync: waits for everything enqueued (the context's stream is made to wait for the copy
 *       streams) and returns the first deferred error. */
int rtm_set_velocity_async(rtm_ctx* ctx, const float* v);
int rtm_step_async(rtm_ctx* ctx, int nsteps);
int rtm_read_field_async(rtm_ctx* ctx, float* out);
int rtm_sync(rtm_ctx* ctx);

/* Kernel variant ("tile", the GPU analogue of the paper's blocksize):
 * -1 = automatic (default), 0 = naive one-thread-per-point kernel, 1..rtm_num_tiles()-1 =
 * TMA-staged xy tiles.  Unknown id -> RTM_EINVAL.  Every variant computes bitwise-identical
 * results (one per-point expression).  Variants named "tb2_*" advance TWO time steps per HBM
 * pass (temporal blocking) on single-GPU single-shot contexts: u^{n+1} is
 * produced and consumed through L2 by co-resident CTAs of a y-band; the context then keeps a
 * second pair of field buffers (2 x nx*ny*(nz+10) floats more).  Odd remainders, multi-slab
 * and batched contexts run the variant's paired single-step kernel. */
int rtm_set_tile(rtm_ctx* ctx, int tile_id);
int rtm_get_tile(rtm_ctx* ctx);          /* the variant rtm_step will use (resolves -1) */
int rtm_num_tiles(void);
/* z-chunk length (planes) of a tiled work unit; 0 = automatic (minimises wave quantisation
 * times chunk-halo re-reads). */
int rtm_set_zchunk(rtm_ctx* ctx, int planes);
const char* rtm_tile_name(int tile_id);  /* e.g. "stream64x32k10d0"; NULL for unknown ids */

/* Tuning options (results are bitwise independent of all of them):
 *   RTM_OPT_ZCHUNK     z-chunk length in planes, 0 = automatic (same as rtm_set_zchunk)
 *   RTM_OPT_CACHE_MODE L2 policy bits of the stream kernels: bits 0-1 L2 prefetch of u_prev/C
 *                      (0 none, 1 evict_last, 2 evict_normal), bit 2 u TMA loads with an
 *                      evict_last policy, bit 3 plain (not evict-first) u_prev/C/u_next
 *                      accesses, bits 4-7 prefetch distance in planes, bits 8-9 L2 promotion
 *                      of the halo'd u TMA box (0 = 256B, 1 = 128B, 2 = 64B, 3 = none), bit 10
 *                      u_prev/C TMA loads with an evict_first policy, bit 11 C TMA loads with an
 *                      evict_last policy (C stays in L2 across steps when it fits)
 *   RTM_OPT_GRAPHS     1 (default) = capture runs of 16 steps in CUDA graphs, 0 = direct launches
 *   RTM_OPT_SHOT_ORDER batched contexts: 0 auto (shot-major when C fits in 40% of L2), 1 shot-major
 *                      (each shot's tiles co-run), 2 shot-fastest (co-running CTAs share C tiles)
 *   RTM_OPT_CHECK_EVERY 0 (default) off; k > 0: rtm_step checks the field for NaN/Inf every k steps
 *   RTM_OPT_HALO_MODE  slab contexts:
 *                      0 (default) boundary planes first, halo copies (in-process: copy engines;
 *                        distributed: NCCL send/recv on a comm stream) overlapped with the interior;
 *                      1 in-process only: fused push — one kernel per slab whose epilogue stores
 *                        the boundary planes straight into the neighbours' halos (peer stores over
 *                        NVLink), ordered by CUDA events;
 *                      2 fused push ordered by a flag protocol: after each step a 1-thread kernel
 *                        releases "steps done" (system scope) into the neighbours' flag words and
 *                        the next step's stream waits on its own flags (cuStreamWaitValue64; no
 *                        spinning kernel).  In a distributed context the neighbours' buffers and
 *                        flags are CUDA-IPC mappings (same node, peer access) set up by an NCCL
 *                        all-gather of the handles: setting it there is a COLLECTIVE call, as is
 *                        rtm_set_step_count while it is active.  Needs 64-bit stream memory ops.
 *                      3 copy-engine pull ordered by the flag protocol (SURVEY §8(e) "SM-free
 *                        alternative"): after its boundary planes each slab releases "boundary n
 *                        ready" into the neighbours' flag words; a neighbour's comm stream waits
 *                        on it and PULLS the 5 planes with cudaMemcpyAsync from the (peer /
 *                        CUDA-IPC mapped) buffer into its own halo, overlapped with its interior
 *                        kernel — no NCCL kernels, no SM time for the transfer, and every rank
 *                        writes only its own memory.  In-process or across processes (IPC); the
 *                        default of peer contexts (rtm_create_peer).
 *                      Peer access is required between neighbouring devices (else RTM_EINVAL).
 *                      Setting 2 or 3 in a distributed context is a COLLECTIVE call.
 *   RTM_OPT_HOST_ORDERED 1: before every device-side flag wait of halo modes 2/3 the library
 *                      synchronises its streams and calls the rank barrier (the NCCL
 *                      communicator or the rtm_set_host_barrier callback), so every wait is
 *                      already satisfied when it is enqueued.  This runs the cross-process data
 *                      plane with host ordering only — used to test several ranks on ONE GPU,
 *                      where device-side waits between processes are not allowed — at the cost
 *                      of one host barrier per step.  0 (default): device-ordered.
 *   RTM_OPT_TB_CTAS    two-step variants ("tb2_*"): max CTAs per y-band launch,
 *                      0 (default) = one per SM.  Smaller values force more, narrower bands
 *                      (used by the tests to cover band edges on small grids).
 *   RTM_OPT_PDL        1: launch consecutive k_stream steps with programmatic dependent launch
 *                      (the next step's CTAs are scheduled while the previous grid drains and
 *                      wait on griddepcontrol.wait before touching memory); 0: plain launches.
 *   RTM_OPT_ZDIR       k_stream z sweep direction bits (default 2): 0 = every unit sweeps z upward; bit 0 =
 *                      odd-parity steps sweep downward (each step starts on the planes the
 *                      previous step touched last); bit 1 = every other unit (wave) of a
 *                      persistent CTA sweeps downward (a wave starts where the previous one
 *                      ended, next to the halo rows it shares with it); bit 2 = odd z-chunks
 *                      sweep downward (neighbouring chunks start / end on the planes they share,
 *                      so each z-halo plane is read by both at the same time).  Bitwise identical
 *                      either way (the z pair sums are commutative).
 *   RTM_OPT_SLAB_SHARE 1: slabs of an in-process context that share a device (one-GPU decomposition
 *                      runs, devices = [0, 0, ...]) split its SMs — each slab's persistent grid
 *                      gets #SMs × occupancy / (slabs on the device) CTAs — so their kernels can run
 *                      concurrently; 0 (default): every launch gets all SMs.
 * Unknown key or out-of-range value -> RTM_EINVAL.  rtm_get_option returns -1 for unknown keys. */
enum { RTM_OPT_ZCHUNK = 1, RTM_OPT_CACHE_MODE = 2, RTM_OPT_GRAPHS = 3, RTM_OPT_SHOT_ORDER = 4,
       RTM_OPT_HALO_MODE = 5, RTM_OPT_CHECK_EVERY = 6, RTM_OPT_TB_CTAS = 7, RTM_OPT_PDL = 8,
       RTM_OPT_HOST_ORDERED = 9, RTM_OPT_ZDIR = 10, RTM_OPT_SLAB_SHARE = 11 };
int rtm_set_option(rtm_ctx* ctx, int key, long long value);
long long rtm_get_option(rtm_ctx* ctx, int key);

/* Run on the caller's CUDA stream (a cudaStream_t, e.g. torch.cuda.current_stream()); NULL
 * restores the library's own stream.  Single-GPU or distributed (one slab per process)
 * contexts only (RTM_EINVAL for multi-slab contexts). */
int rtm_set_stream(rtm_ctx* ctx, void* cuda_stream);

/* CUDA-event time of the last rtm_step call (ms). */
float rtm_last_elapsed_ms(rtm_ctx* ctx);

/* Per-launch stencil timing (bench roofline): when on, rtm_step records CUDA events around
 * every stencil launch (and does not use CUDA graphs); rtm_kernel_stats returns the
 * launches and summed device time (ms) since it was switched on / last read, then clears. */
int rtm_set_profiling(rtm_ctx* ctx, int on);
int rtm_kernel_stats(rtm_ctx* ctx, long long* launches, double* total_ms);
/* Stencil launches issued by the library since creation (all kernels of the step). */
long long rtm_launch_count(rtm_ctx* ctx);

/* ---- the paper's two-phase blocksize tuner, GPU analogue ----------
 * PAPER.md:112-126 ("A Framework for Profiling Technique"): a selection phase times every
 * candidate for nI iterations of the kernel and keeps the best (MinTime); a verification
 * phase re-times the winner (ActualTime); PAPER.md:276-281 rates the choice by
 * 100*(ActualTime - MinTime)/MinTime.  Candidates are (tile variant, z-chunk) pairs timed on
 * the context's real grid with all SMs busy.  With several slabs/ranks a candidate's time is
 * the worst over ranks and the winner minimises it — the MWMB rule, Eq. (2),
 * the paper's best procedure.  The wavefield, step counter and the
 * previous tile/z-chunk settings are restored afterwards (device snapshot; needs 2 extra
 * fields of device memory); the winner is installed.  Requires a velocity.
 * tiles/zchunks: ncand pairs; tiles == NULL -> every non-naive variant with z-chunk 0 (auto).
 * cand_ms (optional, ncand or rtm_num_tiles()-1 doubles) receives each candidate's time. */
typedef struct {
    int best_tile;
    int best_zchunk;
    int ncandidates;
    double min_time_ms;     /* MinTime: the winner's selection-phase time for nI steps      */
    double actual_time_ms;  /* ActualTime: verification-phase time of the winner (nI steps) */
    double quality_pct;     /* 100 * (ActualTime - MinTime) / MinTime        */
} rtm_tune_result;
int rtm_autotune(rtm_ctx* ctx, int nI, const int* tiles, const int* zchunks, int ncand,
                 rtm_tune_result* out, double* cand_ms);
/* The paper's candidate lattice for one dimension ("divided in P parts"):
 * b = < 1, S/(P-1) + 1, 2S/(P-1) + 1, ..., (P-1)S/(P-1) + 1 >, integer division, each value
 * clamped to [1, S] (the worked example at PAPER.md:301 lists 200 for S = 200, P = 5: the
 * formula's last term S+1 is read as S, R17) and duplicates (small S) removed.
 * Writes at most P values to out (ascending) and returns their count; P < 2 or S < 1 ->
 * RTM_EINVAL.  Host-only (no device).  On the GPU the runtime blocksize dimension is the
 * z-chunk length of a work unit (the xy block is the compile-time tile of a variant), so
 * rtm_autotune over {tiles} x rtm_blocksize_lattice(nz, P) is the paper's nC-candidate
 * selection phase. */
int rtm_blocksize_lattice(int S, int P, int* out);

/* MWMB selection (host-only): times[r*ncand + c] = time of candidate c on rank r; returns the
 * c minimising max_r times[r][c] (ties -> lowest c), or -1 on invalid input. */
int rtm_select_mwmb(const double* times, int nranks, int ncand);

/* ---- batched shots (the paper's production mode runs one independent
 * grid per process) ------------------------------------------------
 * One context, nshots independent wavefields on one velocity model (RTM shots share the
 * model, differ in sources).  Host field arrays become (nshots, nz, ny, nx); the velocity stays
 * (nz, ny, nx).  Work units are dealt shot-fastest, so co-running CTAs read the same C tile
 * (one HBM read serves all shots through L2).  rtm_inject_source registers on shot 0;
 * rtm_inject_source_shot on any shot (the RTM_MAX_SOURCES limit is per context).
 * Single-GPU only; across GPUs run one batch per GPU (replicas, no exchange). */
rtm_ctx* rtm_create_batch(int nx, int ny, int nz, float dx, float dt, const float coeffs[6],
                          int nshots);
int rtm_num_shots(rtm_ctx* ctx);
int rtm_inject_source_shot(rtm_ctx* ctx, int shot, int ix, int iy, int iz, const float* samples,
                           int nsamples);

/* ---- z-slab decomposition -------------------------------------------- */

/* One process, several slabs: the grid is split into nslabs z-slabs, slab r on CUDA device
 * devices[r] (devices may repeat, e.g. all 0, to run the decomposition on one GPU).  Halos
 * move by cudaMemcpyPeerAsync (copy engines) between slabs each step.  Host arrays are the
 * whole grid.  Requires nz/nslabs >= 10 for every slab. */
rtm_ctx* rtm_create_multi(int nx, int ny, int nz, float dx, float dt, const float coeffs[6],
                          int nslabs, const int* devices);

/* One process per GPU (torchrun): rank owns global planes [z0, z0+nzl) (rtm_slab_range).
 * id = 128-byte NCCL unique id from rtm_get_unique_id() on rank 0, broadcast by the caller
 * (torch.distributed).  Each step sends/receives the 5 boundary planes to/from rank-1 and
 * rank+1 with ncclSend/ncclRecv on a comm stream, overlapped with the interior planes. */
int rtm_get_unique_id(unsigned char id[128]);
rtm_ctx* rtm_create_dist(int nx, int ny, int nz_global, float dx, float dt,
                         const float coeffs[6], int rank, int world, const unsigned char id[128],
                         int device);

/* One process per GPU WITHOUT NCCL (peer context): the same z-slab of rank `rank` as
 * rtm_create_dist, on CUDA device `device`, whose neighbours are reached only through CUDA-IPC
 * mappings.  Bootstrap (any out-of-band channel, e.g. a torch.distributed gloo group):
 *   1. every rank calls rtm_ipc_export and sends its record to its neighbours;
 *   2. every rank calls rtm_ipc_import with the records of rank-1 and rank+1 (NULL where absent);
 *   3. every rank installs a rank barrier with rtm_set_host_barrier.
 * The default halo mode is 3 (copy-engine pull); 2 (fused push) is also available; 0 (NCCL)
 * is not (RTM_EINVAL).  rtm_reset / rtm_set_fields / rtm_set_step_count / rtm_set_option(
 * RTM_OPT_HALO_MODE) / rtm_autotune are collective (they call the barrier); rtm_step before the
 * import -> RTM_ESTATE.  Ranks may share a device (each then maps the others' buffers). */
rtm_ctx* rtm_create_peer(int nx, int ny, int nz_global, float dx, float dt, const float coeffs[6],
                         int rank, int world, int device);

/* The 512-byte CUDA-IPC record of a slab context (peer or NCCL-distributed): IPC handles of
 * its two time-level buffers and of its flag words, plus the grid extents, rank and world it
 * belongs to (checked on import).  Plain bytes: send them over any channel. */
#define RTM_IPC_RECORD_BYTES 512
int rtm_ipc_export(rtm_ctx* ctx, unsigned char rec[RTM_IPC_RECORD_BYTES]);
/* Open the neighbours' records (lo = rank-1, hi = rank+1; NULL for an absent neighbour).
 * RTM_EINVAL if a record belongs to another grid / world / rank, or a neighbour that exists is
 * passed NULL; RTM_ECUDA if a handle cannot be opened.  May be called once per context. */
int rtm_ipc_import(rtm_ctx* ctx, const unsigned char* lo, const unsigned char* hi);
/* Rank barrier of a peer context: fn(user) must return 0 once every rank of the context has
 * called it (non-zero aborts the calling operation with RTM_ESTATE).  Called from the thread
 * that calls the library.  fn = NULL removes it. */
typedef int (*rtm_barrier_fn)(void* user);
int rtm_set_host_barrier(rtm_ctx* ctx, rtm_barrier_fn fn, void* user);
/* Host time (ms) the last rtm_step spent enqueuing work (launches, waits, copies, graph
 * launches), excluding its final synchronisation; divide by the steps for a per-step cost. */
double rtm_last_enqueue_ms(rtm_ctx* ctx);

/* Host-only plan helpers (no GPU needed; shared by the library and the CPU tests).
 * rtm_slab_range: rank's owned global planes [*z0, *z0 + *nzl); balanced split
 *   z0 = rank*nz/world (floor).  RTM_EINVAL if world < 1, rank out of range, or a slab
 *   would have fewer than 10 planes when world > 1.
 * rtm_halo_plan: element offsets, within a slab buffer of nx*ny*(nzl+10) floats (pass the
 *   row pitch as nx for the device layout), of
 *   [0] send_lo  (owned planes 0..4   -> rank-1),  [1] recv_lo (halo planes -5..-1),
 *   [2] send_hi  (owned planes nzl-5.. -> rank+1), [3] recv_hi (halo planes nzl..nzl+4);
 *   *count = 5*nx*ny elements per message; an offset is -1 when that neighbour is absent. */
int rtm_slab_range(int nz_global, int world, int rank, int* z0, int* nzl);
int rtm_halo_plan(int nx, int ny, int nzl, int rank, int world, long long offsets[4],
                  long long* count);

/* Stability bound nu_crit = 2/sqrt(3*S_max), S_max = max_theta -(c0 + 2 sum c_m cos m theta)
 * (host-only; < 0 on invalid coefficients). */
double rtm_nu_crit(const float coeffs[6]);

#ifdef __cplusplus
}
#endif
#endif /* RTM_H_ */
