/*
 * firecell.h -- C ABI of the B200-native wildfire cellular-automaton path.
 *
 * Drop-in boundary for the reference's hot path (pyrocell 0.1.0; paths
 * below are relative to /root/reference/pkg/src/pyrocell/).  The reference
 * is pure Python/NumPy and has no FFI of its own: its "operator API" is the
 * functions re-exported by __init__.py:4-98.  Each launcher here replaces the
 * numerical core of one of those functions; the Python host layer
 * (paper_2502_18738_b200/) binds them with ctypes and keeps the reference's
 * signatures, argument meaning and exceptions.
 *
 * Rules: every pointer argument is DEVICE memory unless named host_*; the
 * library never allocates (callers size buffers with the fc_*_bytes helpers);
 * all launchers are asynchronous on the given stream and hold no global
 * mutable state.  Return value: FC_OK, or FC_EINVAL (bad argument, nothing
 * launched) / FC_ECUDA (launch error; fc_last_cuda_error() has the code).
 *
 * Data layout:
 *   fire state    bit planes, tile-major: a 32x32-cell tile is 32 uint32 words
 *                 (word r = row r, bit c = column c); planes are
 *                 [M][tiles_y][tiles_x][32]. burning is double-buffered by
 *                 step parity (burn[t & 1] holds pre-step-t state); burned is
 *                 updated in place.  Padding cells outside HxW are "burned".
 *   accumulator   fp32 [M][H][W]; t_ign int16 [M][H][W] (pre-step index of
 *                 the step a cell ignited in, minus fc_state.t_base; -1
 *                 initial/injected or before the base; 0x7FFF never);
 *                 jacobian fp32 [M][H][W][4] = dp/d(c1,c2,a,p_h)
 *                 captured at ignition on attached steps (0 elsewhere).
 *   landscape     env fp32 [H][W][4] = {wind speed m/s, wind vector east and
 *                 north m/s (speed * cos/sin of the direction, deg East-CCW),
 *                 vd=(1+canopy)(1+density)}; slope4 fp32 [H][W][4] forward
 *                 slopes from elevation (the fused slope_from_altitude);
 *                 env64 fp64 [H][W][5] = {elevation, speed, direction, canopy,
 *                 density} read only by the fp64 guard recompute; optional
 *                 slope tensors [H][W][8] (slot order NW,N,NE,W,E,SW,S,SE:
 *                 slope in degrees from the source in that slot toward the
 *                 target) replace the elevation-derived slope.
 *   activity      flags int32 [M][TY][TX] = last pre-step index at which the
 *                 tile must be visited; tile_list int32 [3][M*TY*TX] rotating
 *                 compacted lists of tiles active at steps t, t+1, t+2 with
 *                 list_count int32 [2 (max_steps+3) + 4] (zeroed by fc_state_init,
 *                 8-byte aligned): list lengths, per-launch work counters,
 *                 the neighbour-activation distance the current lists were
 *                 built with (0 = full 3x3 tile neighbourhoods), one unused
 *                 word, and last the dense scan's (ticket, count) pair, zero
 *                 between scans.
 *   params        fp64 [M][8] = {c1, c2, a, p_h, p_continue, norm_c, 0, 0}.
 */
#ifndef FIRECELL_H
#define FIRECELL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fc_stream_t; /* == cudaStream_t */

enum { FC_OK = 0, FC_EINVAL = 1, FC_ECUDA = 2 };

/* Random draws (pyrocell/rng.py).  SPLITMIX reproduces rng.py:35-75 bit for
 * bit (keyed by seed, step, absolute cell, channel); PHILOX is Philox4x32-10
 * keyed by (seed, step, cell, member); INJECT consumes caller-supplied fp64
 * draw tensors [nsteps][M][2][H][W] (channel 0 = ignite, 1 = continue). */
enum { FC_RNG_SPLITMIX = 0, FC_RNG_PHILOX = 1, FC_RNG_INJECT = 2 };

/* Slope source: on-the-fly from elevation (data_io.py:92-132 fused into the
 * stencil) or the caller's per-slot slope tensor (model.py:88-90). */
enum { FC_SLOPE_ELEVATION = 0, FC_SLOPE_TENSOR = 1 };

#define FC_TILE 32
#define FC_NPARAM 8
#define FC_NCOUNTER 4 /* per member and step: ignitions, burn-outs, tiles, candidates */
#define FC_T_NEVER 0x7FFF

typedef struct {
    int32_t height, width;    /* cells                                  */
    int32_t tiles_y, tiles_x; /* ceil(height/32), ceil(width/32)         */
    int32_t members;          /* independent simulations sharing the env */
} fc_grid;

typedef struct {
    const float* env;       /* [H][W][4] fp32 {V, wind east, north, vd}  */
    const float* slope4;    /* [H][W][4] fp32 slope in degrees (signed, slope_sign applied)
                               from each cell toward its E, SW, S, SE neighbour (0 off-grid);
                               the other four directions are the neighbours' negations
                               (exact antisymmetry, data_io.py:112-129).  Elevation mode. */
    const double* env64;    /* [H][W][5] fp64                           */
    const float* slope32;   /* [H][W][8] fp32, FC_SLOPE_TENSOR only     */
    const double* slope64;  /* [H][W][8] fp64, FC_SLOPE_TENSOR only     */
    const float* dir32;     /* [H][W][2] fp32 (cos, sin) of the wind direction; needed by
                               per-step wind schedules                   */
    double cell_side;       /* metres (kernel uses l and l*sqrt(2))     */
    int32_t slope_mode;     /* FC_SLOPE_*                                */
    int32_t slope_sign;     /* +1 downhill-positive, -1 uphill-positive */
    int32_t factor_source;  /* vd at the source (1) or target (0) cell  */
    int32_t pad_;
} fc_landscape;

typedef struct {
    uint32_t* burn0;        /* [M][TY][TX][32] burning, even launch phases */
    uint32_t* burn1;        /* [M][TY][TX][32] burning, odd launch phases  */
    uint32_t* burned0;      /* [M][TY][TX][32] burned, even launch phases  */
    uint32_t* burned1;      /* [M][TY][TX][32] burned, odd launch phases: a
                               launch reads the halo of neighbouring tiles
                               from the phase's input buffers while those
                               tiles' new states go to the output buffers */
    float* acc;             /* [M][H][W]                                */
    int16_t* t_ign;         /* [M][H][W]                                */
    float* jac;             /* [M][H][W][4], may be NULL (no gradients) */
    int32_t* flags;         /* [M][TY][TX] last pre-step index active   */
    int32_t* counters;      /* [M][max_steps][FC_NCOUNTER]              */
    int32_t* tile_list;     /* [3][M*TY*TX] rotating active-tile lists  */
    int32_t* list_count;    /* [2 (max_steps+3) + 4]: list length, then work-
                               distribution counter, of each launch; the
                               neighbour-activation distance of the lists; pad;
                               the dense scan's 64-bit (ticket, count) word */
    uint8_t* tile_fire;     /* [M][TY][TX] per-tile work estimate (log2), written by
                               the step kernel; orders ensemble lists (may be NULL) */
    int32_t* tile_first;    /* [M][TY][TX] earliest pre-step index at which a cell of the
                               tile ignited (-1: initial or injected fire), FC_T_NEVER
                               if none: no cell of the tile has t_ign < tile_first.  The
                               loss kernels skip tiles with no ignition before an
                               observation step.  May be NULL (no skipping). */
    uint8_t* live;          /* [M][H][W] bit k = slot k's neighbour burned pre-step, written
                               at every ignition (the tape mask of kernel.py:380-383); read
                               only where t_ign marks an ignition.  May be NULL. */
    void* sched;            /* fc_sched_workspace_bytes(g, max_steps) bytes, or NULL: with it,
                               an ensemble (M >= 2, keyed SplitMix draws, activity lists,
                               4- or 8-step windows) runs each fc_run call as one persistent
                               dataflow launch in which every member advances window by
                               window on its own (same bytes as one launch per window) */
    int64_t* init_burning;  /* [M] burning cells of each member's initial mask, written by
                               fc_state_init / fc_state_reset (the series' step-0 count,
                               kernel.py:431-439), or NULL */
    int32_t max_steps;
    int32_t t_base;         /* t_ign and tile_first hold (pre-step index - t_base): int16
                               t_ign spans 32766 steps from the base, and runs longer than
                               that move the base forward with fc_state_rebase */
} fc_state;

/* Position of this state in a partitioned job.  Row-sharded single domain
 * (BASELINE config 3 across GPUs): the local grid holds this rank's rows plus
 * ghost tile rows (32 rows each) copied from the neighbouring ranks after
 * every launch.  Ghost tiles are read as halo and never advanced; draws are
 * keyed by the global row = local row + row0.  Member-sharded ensembles
 * (configs 1 and 4): local member m is global member m + member0, the member
 * word of the Philox counter, so a member draws the same numbers on any rank. */
/* Peer-memory halo of a row shard (NVLink peers, or IPC mappings on one
 * device): the boundary pass writes its owned boundary tile rows straight
 * into the neighbours' ghost tile rows, tile by tile as it computes them, and
 * its last CTA then stores `seq` into the neighbours' flag words -- compute
 * and halo transfer in one kernel, no collective.  Protocol (every shard
 * issues the same sequence of events -- resets and boundary passes -- and
 * numbers them 1, 2, ...): before its event k a shard makes its stream wait
 * until both of its own flag words are >= k - 1 (fc_stream_wait_geq); a
 * boundary pass that is event k runs with seq = k; a reset that is event k
 * is followed by fc_peer_signal(k).  So a shard reads its ghost rows only
 * after the neighbours wrote them, writes a neighbour's ghost rows only after
 * the neighbour read the previous ones, and never races a neighbour's reset. */
typedef struct {
    uint32_t* up[4];        /* upper neighbour's {burn0, burn1, burned0, burned1}; NULL: none */
    uint32_t* down[4];      /* lower neighbour's planes; NULL: none                          */
    int32_t up_tiles_y;     /* the neighbours' local tile rows (ghost rows included)          */
    int32_t down_tiles_y;
    int32_t* up_flag;       /* the upper neighbour's word counting this shard's events        */
    int32_t* down_flag;     /* the lower neighbour's word                                     */
    int32_t seq;            /* the event number the next boundary pass stores                 */
    int32_t pad_;
} fc_peer_halo;

typedef struct {
    int32_t row0;           /* global row of local row 0                    */
    int32_t ghost_top;      /* ghost tile rows at the top (0 or 1)          */
    int32_t ghost_bottom;   /* ghost tile rows at the bottom (0 or 1)       */
    int32_t member0;        /* global index of local member 0               */
    const fc_peer_halo* peer; /* NULL, or the peer-memory halo (fc_run_pass pass 2) */
} fc_shard;

/* ------------------------------------------------------------ sizing --- */
void fc_grid_make(int32_t height, int32_t width, int32_t members, fc_grid* out);
size_t fc_plane_words(const fc_grid* g);              /* uint32 words per plane   */
size_t fc_loss_workspace_bytes(const fc_grid* g, int32_t n_targets);
size_t fc_sched_workspace_bytes(const fc_grid* g, int32_t max_steps);  /* fc_state.sched */

/* -------------------------------------------------------------- state --- */
/* new_fire_state (model.py:180-200) for every member: init is uint8 [M][H][W]
 * (member_stride = H*W) or one [H][W] mask broadcast (member_stride = 0).
 * t0 = pre-step index of the initial state.  Zeroes the counters.  jac is
 * not cleared: every ignition writes its J (zero on unattached steps) and J
 * is defined only where t_ign marks an ignition during the run. */
int fc_state_init(const fc_grid* g, const fc_state* s, const uint8_t* init,
                  int64_t member_stride, int32_t t0, fc_stream_t stream);

/* fc_state_init for a state previously initialised by fc_state_init whose
 * acc and t_ign have been written only by this library since (fc_run,
 * fc_inject, fc_state_reset): acc and t_ign are rewritten only in tiles that
 * held fire since the last reset (tile_first set) or hold initial fire now;
 * every other cell already has acc = 0, t_ign = FC_T_NEVER.  Same result as
 * fc_state_init at a fraction of the memory traffic.  tile_first must be set. */
int fc_state_reset(const fc_grid* g, const fc_state* s, const uint8_t* init,
                   int64_t member_stride, int32_t t0, fc_stream_t stream);

/* Unpack the current state to uint8 grids [M][H][W] (either may be NULL);
 * phase = number of fc_run launches since fc_state_init (selects the
 * burning buffer).  Mirrors FireState.burning / burned (model.py:158-160). */
int fc_state_unpack(const fc_grid* g, const fc_state* s, int32_t phase, uint8_t* burning,
                    uint8_t* burned, fc_stream_t stream);

/* Jaccard index per member of the affected cells (burning | burned) against a
 * uint8 target mask [H][W] per member (member_stride elements apart; 0 = one
 * mask shared by all members): out[m] = |A & T| / |A | T|, 1 when both are
 * empty -- the metric of calibration.py's iteration records, computed from the
 * bit planes (no unpack).  work: 2 M + 1 zero-initialised uint64 on the device,
 * left zeroed by the call.  Replaces jaccard_index (pyrocell/losses.py:89-98)
 * over unpacked grids in calibrate()'s records (calibration.py:204). */
int fc_state_jaccard(const fc_grid* g, const fc_state* s, int32_t phase, const uint8_t* targets,
                     int64_t member_stride, uint64_t* work, double* out, fc_stream_t stream);

/* Export the current state into [M][H][W] result arrays: burning / burned as
 * uint8 0/1 and the accumulator as fp32 (any may be NULL) -- the same values
 * fc_state_unpack and the acc plane hold.  The arrays may be pinned host
 * memory mapped into the device address space (fc_host_device_pointer), so
 * the kernel writes the results over PCIe without a device staging copy.
 * written: NULL = every tile is written; else uint8 [M][TY][TX] flags owned
 * by the destination (zero-initialised together with it): only tiles that are
 * affected now (tile_first set) or were written by the previous export into
 * the same destination are written, and the flags are updated.  The caller
 * keeps the destination's other cells zero.  Replaces the host-side copy of
 * FireState.burning / burned / accumulator (model.py:148-177) at the end of
 * run_simulation (kernel.py:525-529). */
int fc_state_export(const fc_grid* g, const fc_state* s, int32_t phase, uint8_t* burning,
                    uint8_t* burned, float* acc, uint8_t* written, fc_stream_t stream);

/* Device address of pinned host memory (cudaHostGetDevicePointer). */
int fc_host_device_pointer(void* host, void** device_ptr);

/* Long runs (kernel.py:453-468 has no step limit): every recorded ignition
 * becomes "before the base" (t_ign -1, tile_first -1); the caller then moves
 * fc_state.t_base to the current pre-step index, after which t_ign counts
 * steps from there.  Losses, contractions and fp64 recomputation address
 * ignitions after the last rebase only (recompute64 before rebasing). */
int fc_state_rebase(const fc_grid* g, const fc_state* s, fc_stream_t stream);

/* inject_ignitions (kernel.py:405-419) before pre-step t (launch phase
 * `phase`): cells is int32 [n][3] = (member, row, col), all in bounds
 * (checked by the caller).  Burnable cells start burning with accumulator
 * 1.0 (a constant). */
int fc_inject(const fc_grid* g, const fc_state* s, const int32_t* cells, int32_t n,
              int32_t t, int32_t phase, fc_stream_t stream);

/* ------------------------------------------------------------ forward --- */
/* Advance every member from pre-step index t0 by nsteps steps: the loop of
 * run_simulation (kernel.py:504-524) over step_forward (kernel.py:263-333).
 * host_attach: NULL or nsteps flags (step t0+i attaches when host_attach[i]).
 * draws: FC_RNG_INJECT only, [nsteps][M][2][H][W] fp64.
 * skip_inactive: 1 = only tiles near burning cells are visited (exact: the
 * analogue of the reference's bounding-box window, kernel.py:296-302);
 * 0 = dense sweep: every launch rescans the whole domain (fc_activity_scan)
 * instead of using incremental activity lists.  A state must not switch
 * between the two without fc_state_init.
 * window: steps fused per launch (temporal blocking; 1, 4, 8 or 16).
 * wind_schedule: NULL, or fp64 [max_steps][4] = {alpha, beta, gamma_deg, 0}
 * indexed by pre-step index: step t sees speed alpha*V + beta and direction
 * theta + gamma (a WindUpdate, kernel.py:422-428/505-511, for every step
 * without re-uploading fields; config 4's rotating, ramping wind).
 * shard: NULL, or the partition descriptor (global row / member offsets;
 * ghost rows are not advanced).
 * host_phase: in/out launch counter (see fc_state_unpack). */
int fc_run(const fc_grid* g, const fc_landscape* land, const fc_state* s,
           const double* params, const uint64_t* seeds, int32_t rng_mode,
           const double* draws, int32_t t0, int32_t nsteps, const uint8_t* host_attach,
           int32_t skip_inactive, int32_t window, const double* wind_schedule,
           const fc_shard* shard, int32_t* host_phase, fc_stream_t stream);

/* One launch of fc_run on a row shard, split so that the halo exchange of
 * the previous launch overlaps compute (activity-list sweep, keyed draws;
 * nsteps <= window steps from pre-step index t0 at launch *host_phase):
 *   pass 1: the listed tiles outside the boundary tile rows (the first and
 *           last owned tile rows, next to ghost rows) -- they read no ghost
 *           rows, so they may run while the ghost rows are being refreshed;
 *           *host_phase is unchanged;
 *   pass 2: every tile of the boundary tile rows (a dense sweep of at most
 *           two tile rows: fire arriving through a ghost row needs no
 *           activity marks), after the ghost rows hold the neighbours'
 *           state of this launch's input; advances *host_phase.
 * Pass 1 then pass 2 of every launch gives the same bytes as fc_run
 * (kernel.py:307-309 partition invariance; draws keyed by global cells).
 * With shard->peer, pass 2 also stores the boundary tile rows of its output
 * into the neighbours' ghost tile rows (their input of the next launch) and,
 * when its last CTA is done, stores peer->seq into the neighbours' flag words
 * (release, system scope; the protocol is at fc_peer_halo). */
int fc_run_pass(const fc_grid* g, const fc_landscape* land, const fc_state* s,
                const double* params, const uint64_t* seeds, int32_t rng_mode, int32_t t0,
                int32_t nsteps, const uint8_t* host_attach, int32_t window,
                const double* wind_schedule, const fc_shard* shard, int32_t pass,
                int32_t* host_phase, fc_stream_t stream);

/* Store `value` into the neighbours' flag words of `peer` once the work
 * queued before it on `stream` is done (release, system scope): the event
 * signal of a reset in the peer-halo protocol. */
int fc_peer_signal(const fc_peer_halo* peer, int32_t value, fc_stream_t stream);

/* Make `stream` wait (without a kernel) until the int32 at device address
 * `flag` is >= value (wrap-around compare; cuStreamWaitValue32 GEQ): the
 * peer-halo hand-off between row shards. */
int fc_stream_wait_geq(const int32_t* flag, int32_t value, fc_stream_t stream);

/* Dense-sweep activity scan for launch `phase` (the first half of every
 * skip_inactive = 0 launch, exposed for measurement): streams the burning
 * plane, lists every tile with fire in its 3x3 tile neighbourhood and writes
 * the all-zero next state of every other tile (HBM-bound).  One kernel
 * launch: the list length is set by the scan's last CTA. */
int fc_activity_scan(const fc_grid* g, const fc_state* s, int32_t phase, fc_stream_t stream);

/* After the ghost rows were refreshed with the neighbours' state at launch
 * phase `phase`, activate the owned tiles next to ghost tiles holding fire
 * (the marks a neighbour's tiles would have made in an unsharded run). */
int fc_mark_ghosts(const fc_grid* g, const fc_state* s, const fc_shard* shard, int32_t phase,
                   fc_stream_t stream);

/* ----------------------------------------------------------- backward --- */
/* backward_params (tape.py:118-148): out[m][4] = sum_j g[m][j] * J[m][j] in
 * (c1, c2, a, p_h) order; g is fp64 (g_is_f32 = 0) or fp32 [M][H][W].
 * workspace: fc_loss_workspace_bytes(g, 1) bytes. */
int fc_contract(const fc_grid* g, const fc_state* s, const void* dl_dacc, int32_t g_is_f32,
                double* out, void* workspace, fc_stream_t stream);

/* fp64 recomputation of the ignitions recorded at pre-step indices
 * t_lo <= t_ign < t_hi (those steps ran on this landscape / wind schedule):
 * p_ignite and J = dp/d(c1, c2, a, p_h) from the live-slot mask of each cell
 * (fc_state.live, required), in fp64 with the reference's operation order
 * (kernel.py:172-190, 232-240; tape.py:134-147).  acc64 [M][H][W] and jac64
 * [M][H][W][4] (may be NULL) are written for those cells only.  This gives
 * the pyrocell-signature API fp64 accumulators and tape caches. */
int fc_recompute64(const fc_grid* g, const fc_landscape* land, const fc_state* s,
                   const double* params, int32_t t_lo, int32_t t_hi,
                   const double* wind_schedule, double* acc64, double* jac64,
                   fc_stream_t stream);

/* backward_params (tape.py:118-148) over a subset of the run's tape blocks:
 * out[m][4] = sum over cells whose ignition step t_ign has step_flags[t_ign]
 * != 0 (device uint8 [n_flags]) of dl_dacc (fp64) * jac64 (fc_recompute64),
 * fixed-order fp64 reduction.  workspace: fc_loss_workspace_bytes(g, 1). */
int fc_contract_steps(const fc_grid* g, const fc_state* s, const double* dl_dacc,
                      const double* jac64, const uint8_t* step_flags, int32_t n_flags,
                      double* out, void* workspace, fc_stream_t stream);

/* combined_loss (losses.py:44-86) summed over n_targets observation steps of
 * one run, fused with the gradient contraction.  acc_s = acc where
 * t_ign < obs_steps[k] (the accumulator as it stood after step obs_steps[k]);
 * targets uint8 [n_targets][M][H][W] with member stride target_member_stride
 * (0 = shared by all members).  Outputs per member m:
 *   loss_out[m][2 + 2*n_targets] = {total, n_targets, bce_0, mse_0, bce_1, ...}
 *   crop_out[m][n_targets][4] (int32 r0, r1, c0, c1; may be NULL)
 *   grad_out[m][4]   (may be NULL: loss only)
 *   dl_dacc [M][H][W] fp64 of the single target (n_targets == 1; may be NULL)
 * workspace: fc_loss_workspace_bytes(g, n_targets) bytes. */
int fc_loss_grad(const fc_grid* g, const fc_state* s, const uint8_t* targets,
                 int64_t target_member_stride, const int32_t* host_obs_steps,
                 int32_t n_targets, double* loss_out, int32_t* crop_out, double* grad_out,
                 double* dl_dacc, void* workspace, fc_stream_t stream);

/* combined_loss (losses.py:44-86) of a caller-supplied fp64 accumulator
 * [H][W] and uint8 target: loss_out[4] = {total, 1, bce, mse}, crop_out[4],
 * dl_dacc [H][W] fp64 (may be NULL).  workspace: fc_loss_workspace_bytes of
 * a 1-member grid with 1 target. */
int fc_loss_dense(int32_t height, int32_t width, const double* acc, const uint8_t* target,
                  double* loss_out, int32_t* crop_out, double* dl_dacc, void* workspace,
                  fc_stream_t stream);

/* adamw_update + clamp_params (calibration.py:43-64, model.py:47-57) on the
 * device params [M][8] with per-member moments adam[M][8] = {m[4], v[4]}.
 * step = 1-based Adam step, or dev_step (device int32 [M], incremented by the
 * kernel) for CUDA-graph replays.  A non-finite gradient leaves that member's
 * params and step untouched and sets status[m] = 1 (else 0). */
int fc_adamw(const double* grads, double* params, double* adam, int32_t members,
             int32_t step, int32_t* dev_step, double lr, double weight_decay, double beta1,
             double beta2, double eps, int32_t clamp, int32_t* status, fc_stream_t stream);

/* ---------------------------------------------------------------- rng --- */
/* uniform_grid (rng.py:55-75) on the device: out [height][width] fp64. */
int fc_uniform_grid(uint64_t seed, int64_t t, int32_t channel, int64_t row0, int64_t col0,
                    int64_t height, int64_t width, double* out, fc_stream_t stream);
/* derive_epoch_seed (rng.py:83-88); host function. */
uint64_t fc_epoch_seed(uint64_t base_seed, uint64_t epoch);

/* ------------------------------------------------------------- fields --- */
/* build_fields (kernel.py:149-205) for the pyrocell API, evaluated in fp64
 * with the reference's operation order for params row 0: out fp64 [8][H][W]
 * (fp), or [5][8][H][W] (fp, raw, rest, cosm1, slope) with gradients. */
int fc_build_fields(const fc_grid* g, const fc_landscape* land, const double* params,
                    double* out, int32_t with_gradients, fc_stream_t stream);

/* ---------------------------------------------------------- landscape --- */
/* Kernel-layout landscape from the five rasters (Landscape, model.py:76-105;
 * slope_from_altitude, data_io.py:92-132) in one pass: inputs [H][W] fp32
 * (input_is_f64 = 0) or fp64; outputs env fp32 [H][W][4] = {V, V cos th,
 * V sin th, (1+canopy)(1+density)}, slope4 fp32 [H][W][4] = slope in degrees
 * toward the E, SW, S, SE neighbour (0 off the grid; negated when
 * slope_sign < 0), env64 fp64 [H][W][5] = the inputs widened, dir32 fp32
 * [H][W][2] = (cos th, sin th).  All arithmetic in fp64 before rounding,
 * like the reference (replaces the host-side torch preparation). */
int fc_landscape_build(int32_t height, int32_t width, const void* elevation,
                       const void* wind_speed, const void* wind_direction, const void* canopy,
                       const void* density, int32_t input_is_f64, double cell_side,
                       int32_t slope_sign, float* env, float* slope4, double* env64, float* dir32,
                       fc_stream_t stream);

/* fc_landscape_build on at most max_ctas CTAs (0 = as many as the grid
 * needs).  The e2e runner builds the next call's landscape with a few CTAs on
 * a low-priority stream while the current call's step kernels hold the SMs. */
int fc_landscape_build_ctas(int32_t height, int32_t width, const void* elevation,
                            const void* wind_speed, const void* wind_direction,
                            const void* canopy, const void* density, int32_t input_is_f64,
                            double cell_side, int32_t slope_sign, float* env, float* slope4,
                            double* env64, float* dir32, int32_t max_ctas, fc_stream_t stream);

/* ---------------------------------------------------------- diagnostics --- */
int fc_last_cuda_error(void);
const char* fc_version(void);
/* Builds compiled with -DFC_TRACE record per-CTA phase timestamps of the
 * window kernel into buf ([512][16][4] int64); NULL disables.  No effect in
 * regular builds. */
void fc_debug_set_trace(long long* buf);

#ifdef __cplusplus
}
#endif
#endif /* FIRECELL_H */
