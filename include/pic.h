/*
 * pic.h — C ABI of the B200-native particle hot path of the implicit-moment
 * PIC cycle (arXiv 2507.20719, iPIC3D): the implicit predictor-corrector
 * mover (Eq. 2) and the moment gatherer (Eq. 3), with slab decomposition,
 * ghost-node moment sums and particle migration over NVLink peer memory (or
 * NCCL), plus the NEXT rows built on it: the relativistic mover (NEXT-1), the
 * field solver's sources chi, rho-hat, J-hat (Eq. 5-6, NEXT-2), inflow
 * injection and particle control (NEXT-3), and the velocity-histogram
 * Gaussian-mixture fit of the GMM compression (NEXT-4).
 *
 *   PAPER.md:141-145  Eq. 1  equations of motion; q_s, m_s, x_p, v_p, E_p, B_p
 *   PAPER.md:149-165  Eq. 2  predictor-corrector mover, fixed-point on v-bar
 *   PAPER.md:184-187  Eq. 3  {rho, J, Pi}_g = sum_p q {1, v, vv} W(x - x_p)
 *   PAPER.md:235-236  §III-B open boundaries (outflow particles are removed)
 *   PAPER.md:256-261, 291-334  Alg. 1: mover -> interpolation -> MPI exchange
 *   PAPER.md:199-213  Eq. 5-6 susceptibility and corrected sources (NEXT-2)
 *   PAPER.md:232-249  §III-B injection and particle control (NEXT-3)
 *   PAPER.md:366-379  §IV GMM velocity binning and EM fit (NEXT-4)
 * Readings of the paper (R1..R33) are listed in DESIGN.md §3.
 *
 * Conventions (all calls):
 *  - Every entry point returns pic_status; none throws, exits or prints.
 *    The text of the last error is pic_last_error(ctx).
 *  - Units are the caller's code units (the generators use c = 1, lengths in
 *    d_i, time in 1/omega_pi).  Positions are absolute, origin 0, global.
 *  - Pointers documented "host or device" may be either (the library copies
 *    with cudaMemcpyDefault on the context stream).  Host pointers should be
 *    pinned for asynchronous copies.  Device pointers must be on the device
 *    that was current at pic_init.
 *  - All GPU work is enqueued on the context stream (pic_set_stream) and is
 *    asynchronous unless stated; device-side errors (non-finite values,
 *    particles beyond ghost reach, capacity overflow) are latched in device
 *    flags and surfaced by the next pic_sync.
 *  - Per cycle the call order is pic_mover -> pic_moments -> pic_exchange
 *    (for each species, mover before moments); other orders return
 *    PIC_ESTATE.  With nranks > 1, pic_mover and pic_exchange are COLLECTIVE
 *    over the nranks of the config (every rank calls them with the same s).
 */
#ifndef PIC_H
#define PIC_H

#include <stdint.h>

#if defined(__GNUC__)
#define PIC_API __attribute__((visibility("default")))
#else
#define PIC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PIC_ABI_VERSION 6
#define PIC_MAX_SPECIES 8
#define PIC_NCCL_ID_BYTES 128
#define PIC_N_MOMENTS 10  /* rho, Jx, Jy, Jz, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz (R16) */

typedef struct pic_ctx pic_ctx;

typedef enum {
  PIC_OK = 0,
  PIC_EINVAL = 1,       /* bad argument / config                                  */
  PIC_ECUDA = 2,        /* CUDA runtime error                                     */
  PIC_ENCCL = 3,        /* NCCL error                                             */
  PIC_ENOMEM = 4,       /* workspace too small                                    */
  PIC_ESTATE = 5,       /* call order violated (e.g. moments before mover)        */
  PIC_ERANGE = 6,       /* particle beyond ghost reach / > 1 periodic wrap /
                           particle capacity exceeded                            */
  PIC_ENONFINITE = 7    /* NaN/Inf seen in a field sample or particle update      */
} pic_status;

typedef enum { PIC_BC_PERIODIC = 0, PIC_BC_OPEN = 1 } pic_bc;

/* Kernel family selection (pic_config.kernel).                               */
typedef enum {
  PIC_KERNEL_AUTO = 0,     /* best available (tiled where the config allows)  */
  PIC_KERNEL_BASIC = 1,    /* one thread per particle, global field reads,
                              global fp64 atomics for the deposit              */
  PIC_KERNEL_TILED = 2     /* cell-ordered: TMA-staged tile mover, tensor-core
                              per-cell deposit                                 */
} pic_kernel;

/* Multi-rank transport (pic_config.transport).                              */
typedef enum {
  PIC_TRANSPORT_AUTO = 0,  /* peer memory when every rank can map its slab
                              neighbours' workspaces (CUDA IPC), else NCCL     */
  PIC_TRANSPORT_NCCL = 1,  /* NCCL point-to-point messages, host sync for the
                              migration counts                                 */
  PIC_TRANSPORT_PEER = 2,  /* the mover writes slab leavers into the
                              neighbour's buffer over NVLink and ghost planes
                              are read from peer memory; pic_init fails if the
                              neighbours cannot be mapped                      */
  PIC_TRANSPORT_LOOPBACK = 3  /* the nranks slab contexts live in ONE process
                              on ONE device (no NCCL, nccl_id ignored) and are
                              joined by pic_loopback_link; the peer transport's
                              data-path kernels then run unchanged (migration
                              stores from the mover, arrivals, ghost-plane
                              reads); its barriers become event handshakes
                              between the contexts' streams.  Each context
                              needs its own non-default stream and its own
                              host thread (a barrier blocks that thread until
                              the neighbours reach it, 20 s at most).  For
                              testing the multi-rank path on one GPU.         */
} pic_transport;

typedef struct {
  /* Global grid: cells [0, ncell) per axis, origin 0, Delta_d = len_d/ncell_d. */
  int64_t ncell[3];
  double  len[3];
  int32_t bc[3];                 /* pic_bc per axis                              */
  double  dt;                    /* time step Delta t                            */
  double  c;                     /* speed of light (Omega = q B /(m c), Eq. 2)   */
  int32_t n_species;             /* 1 .. PIC_MAX_SPECIES                          */
  double  qom[PIC_MAX_SPECIES];  /* q_s / m_s, signed (R8)                        */
  int32_t n_iter[PIC_MAX_SPECIES];   /* fixed PC iterations, >= 1 (R2; default 3) */
  int64_t capacity[PIC_MAX_SPECIES]; /* particle slots per species on this rank,
                                        including migration headroom             */
  double  planet_center[3];      /* absorbing sphere (R21); radius 0 = none       */
  double  planet_radius;
  int32_t rank, nranks;          /* slab decomposition along x                    */
  int64_t slab_lo, slab_hi;      /* this rank owns x-cells [slab_lo, slab_hi)     */
  int32_t ghost;                 /* G >= 1: field-window ghost nodes per side and
                                    moment ghost node planes per x-side (R22)     */
  int32_t transport;             /* pic_transport (nranks > 1)                    */
  int32_t kernel;                /* pic_kernel                                    */
  int32_t relativistic;          /* 0: gamma == 1 limit of Eq. 2 (R3, the hot path);
                                    1: relativistic Eq. 2 with gamma (NEXT-1, R4-R6);
                                    |v| >= c is then a non-finite update (R23)    */
  int32_t far_hops;              /* peer / loopback transports: extra forwarding
                                    rounds per pic_mover for particles that cross
                                    more than one slab in one step (R22); a
                                    particle still not home after them is dropped
                                    and counted as a far-flyer (PIC_ERANGE).  0
                                    (default): one hop; each extra round costs a
                                    barrier even when nothing is forwarded.
                                    0 <= far_hops < nranks.                       */
  int32_t barrier_timeout_ms;    /* peer / loopback transports: a neighbour that
                                    does not reach a barrier within this time is
                                    reported (PIC_ENCCL) instead of hanging; 0 =
                                    default 20000                                 */
} pic_config;

/* ABI version (PIC_ABI_VERSION).                                             */
PIC_API int32_t pic_abi_version(void);

/* Fill out[PIC_NCCL_ID_BYTES] with a fresh ncclUniqueId (call on rank 0 and
 * broadcast the bytes to the other ranks, e.g. with torch.distributed).      */
PIC_API pic_status pic_nccl_id(void *out);

/* Bytes of device workspace pic_init needs for this config (particle store
 * x2 for sorting, keys, field window, moments with ghost planes, exchange
 * buffers, sort scratch).  Needs the CUDA device that pic_init will use.     */
PIC_API pic_status pic_workspace_bytes(const pic_config *cfg, int64_t *bytes);

/* Create a context.  workspace: device pointer to >= bytes bytes (e.g. one
 * torch.empty(bytes, dtype=uint8, device='cuda')), 256-byte aligned, owned by
 * the caller and kept alive until pic_destroy; libpic never cudaMallocs.
 * nccl_id: PIC_NCCL_ID_BYTES bytes from pic_nccl_id on rank 0 (ignored and
 * may be NULL when nranks == 1).  The config is copied.                      */
PIC_API pic_status pic_init(const pic_config *cfg, const void *nccl_id, void *workspace,
                    int64_t bytes, pic_ctx **out);

/* Join the n contexts of a loopback decomposition (PIC_TRANSPORT_LOOPBACK):
 * ctxs[r] must be rank r of n, all on one device, their slabs tiling the x
 * axis in rank order.  Afterwards each context addresses its slab neighbours'
 * receive buffers, control words and moment planes directly, exactly as the
 * peer transport does over CUDA IPC (the particle
 * communication of Alg. 1 phase 2, here within one device).  Call once, after
 * pic_init of all n and before the first pic_mover.  Synchronises the device.
 * Errors: PIC_EINVAL (mismatched configs / devices), PIC_ESTATE (linked twice). */
PIC_API pic_status pic_loopback_link(pic_ctx *const *ctxs, int32_t n);

/* Stream for all subsequent work (a cudaStream_t, e.g. torch's current
 * stream).  NULL = the legacy default stream.                                */
PIC_API pic_status pic_set_stream(pic_ctx *ctx, void *stream);

/* Load n particles of species s, replacing the previous ones (the particle
 * state of Eq. 1: x_p, v_p and the charge q_s w_p of the
 * statistical weights; kept in GPU memory).
 * xyzuvwq[7]:
 * host or device fp64 arrays x, y, z, u, v, w (velocity) and q (per-particle
 * charge q_s w_p, R14); id: host or device int64 ids (may be NULL: ids
 * become 0..n-1).  Particles must lie in this rank's slab [slab_lo, slab_hi)
 * x [0, ncell_y) x [0, ncell_z) (in cells).  Returns PIC_ERANGE if
 * n > capacity[s].  Copied; the caller's buffers may be reused on return of
 * the next pic_sync.                                                         */
PIC_API pic_status pic_set_particles(pic_ctx *ctx, int32_t s, int64_t n,
                             const double *const xyzuvwq[7], const int64_t *id);

/* Append n particles to species s (same arrays and units as
 * pic_set_particles; id NULL: ids continue the store's
 * position count) and count them into the cell order (built once, by the next
 * call that needs it).  For loading stores too large to stage in one
 * piece (draw a sub-slab, append it, free it).  Between cycles only
 * (PIC_ESTATE between pic_mover and pic_exchange); PIC_ERANGE if the store
 * would exceed capacity[s].  Particles outside this rank's slab are counted
 * as far-flyers and dropped.  Synchronises the stream.                       */
PIC_API pic_status pic_add_particles(pic_ctx *ctx, int32_t s, int64_t n,
                             const double *const xyzuvwq[7], const int64_t *id);

/* Number of live particles of species s on this rank (synchronises the
 * stream).                                                                   */
PIC_API pic_status pic_count(pic_ctx *ctx, int32_t s, int64_t *n);

/* Copy the live particles of species s out (in store order — the order is
 * unspecified; compare by id, R20).  xyzuvwq[7]/id: host or device buffers of
 * >= pic_count elements (any entry may be NULL to skip it).  Synchronises.   */
PIC_API pic_status pic_get_particles(pic_ctx *ctx, int32_t s, double *const xyzuvwq[7],
                             int64_t *id);

/* Set E and B for the next mover call.  EB: host or device fp64 window
 * EB[kz][ky][kx][6] (Ex Ey Ez Bx By Bz) over global node indices
 *   x: [slab_lo - G, slab_hi + G],  y: [-G, ncell_y + G],  z: [-G, ncell_z + G]
 * i.e. (slab_hi - slab_lo + 1 + 2G) x (ncell_y + 1 + 2G) x (ncell_z + 1 + 2G)
 * nodes, periodic images replicated by the caller (R10, R11).  Copied into
 * the context (the caller's buffer may be reused after the next pic_sync).
 * Double-buffered: the copy goes to the buffer the NEXT pic_mover reads, on
 * an internal copy stream, so a host-to-device copy of the next cycle's
 * fields overlaps the current cycle (fields on the host for
 * discrete GPUs); a device source is first ordered after the context stream. */
PIC_API pic_status pic_set_fields(pic_ctx *ctx, const double *EB);

/* Advance species s (-1 = all) one cycle with Eq. 2 (R1-R3, R7-R9), then
 * apply the boundary conditions (R10, R11, R21).  With nranks > 1 this call
 * is COLLECTIVE: particles that left the slab migrate to their new owner rank
 * ("exiting particles are transferred using MPI"),
 * (with the NCCL transport this blocks the host once for the message counts;
 * the peer transport does not block).  Ends by building the
 * cell order of the new state that pic_moments deposits over.                */
PIC_API pic_status pic_mover(pic_ctx *ctx, int32_t s);

/* Gather rho_s, J_s, Pi_s (Eq. 3, R12-R18) of the current state of species s
 * (-1 = all) into the context's ghosted node arrays (owned values become
 * final after pic_exchange).                                                 */
PIC_API pic_status pic_moments(pic_ctx *ctx, int32_t s);

/* Alg. 1 phase 2, PAPER.md:256-261, 317-320 (the nodes a slab shares with its
 * neighbour; the paper's "particle communication" exchange point) and R18
 * (periodic node N == node 0).  COLLECTIVE when nranks > 1: adds the ghost
 * node planes deposited next to the slab face into their owner's planes
 * (peer transport: the owner reads its left neighbour's plane x = slab_lo
 * over NVLink; NCCL transport: one send/recv group), then folds the periodic
 * images along y, z (and along x when nranks == 1).  Requires pic_moments of
 * every species since the last pic_mover (PIC_ESTATE otherwise).  Afterwards
 * the owned node values are final (pic_get_moments / pic_moment_ptr).
 * Asynchronous; latched device errors are returned by pic_sync.              */
PIC_API pic_status pic_exchange(pic_ctx *ctx);

/* One full particle cycle of Alg. 1 (phases 1-2):
 * pic_mover(-1), pic_moments(-1), pic_exchange (errors as those calls; the
 * first failing status is returned).  Replayed from a CUDA graph when
 * pic_set_graph allows it.                                                    */
PIC_API pic_status pic_cycle(pic_ctx *ctx);

/* Implementation control (no paper passage).
 * CUDA graphs for pic_cycle (enable != 0; default off): the first pic_cycle
 * of each (field buffer, store buffer) combination is captured into a CUDA
 * graph and later cycles replay it — one launch instead of ~20 kernel launches
 * per cycle, for small per-GPU problems where launch gaps matter.  pic_cycle
 * falls back to plain launches (same results) whenever a host decision sits
 * inside the cycle: the NCCL or loopback transports, inflow injection,
 * pic_profile enabled, a species between pic_mover and pic_exchange, or the
 * legacy default stream as the context stream (capture needs its own stream).
 * The separate pic_mover / pic_moments / pic_exchange calls never use graphs. */
PIC_API pic_status pic_set_graph(pic_ctx *ctx, int32_t enable);

/* Node counts of the moment output of this rank: out[0] = owned x-planes
 * (slab_hi - slab_lo, +1 on the last rank when x is open), out[1], out[2] =
 * y, z unique nodes (ncell for periodic axes, ncell + 1 for open, R18).      */
PIC_API pic_status pic_moment_shape(const pic_ctx *ctx, int64_t out[3]);

/* Copy the owned moments of species s to out[10][nz][ny][nx] (shape from
 * pic_moment_shape; host or device).  Valid after pic_exchange.             */
PIC_API pic_status pic_get_moments(pic_ctx *ctx, int32_t s, double *out);

/* Wait for the stream and return counters accumulated since pic_init:
 * stats[0] removed (open faces / planet), [1] sent, [2] received,
 * [3] far-flyers (deposit fallback), [4] field samples clamped to the window,
 * [5] non-finite, [6] capacity overflow, [7] multi-wrap.  stats may be NULL.
 * Returns the first latched device error as a status.                        */
PIC_API pic_status pic_sync(pic_ctx *ctx, int64_t stats[8]);

/* Asynchronous pic_get_moments: the moments of species s are packed on the
 * context stream into one of two staging slots of the species and copied to
 * `out` (pinned host or device) on the internal copy stream, overlapping the
 * next cycle.  `out` is complete after pic_join_copies followed by a
 * synchronisation of the context stream, or after pic_sync.                  */
PIC_API pic_status pic_get_moments_async(pic_ctx *ctx, int32_t s, double *out);

/* NEXT-2 (Eq. 5-6; readings R24-R27): the implicit field
 * solver's particle sources from the moments of every species (after
 * pic_exchange) and B of the most recent pic_set_fields, over the owned nodes
 * (pic_moment_shape, layout [..][z][y][x]; host or device buffers, any may be
 * NULL):
 *   chi[9]      sum_s (1/2)(omega_ps dt)^2 R_s, row-major 3x3 per node,
 *               omega_ps^2 = 4 pi rho_s q_s/m_s, R_s = (I - [a]x + a a^T)/(1+a.a),
 *               a = q_s B dt / (2 m_s c)  (Gaussian units)
 *   J_hat[3]    sum_s R_s (J_s - (dt/2) div Pi_s)
 *   rho_hat[1]  sum_s rho_s - dt div J_hat
 * Central differences (periodic wrap; one-sided at open-axis boundary nodes).
 * nranks > 1: COLLECTIVE with the peer transport (the x derivatives at a slab
 * face read the neighbour's adjacent owned plane from its mapped workspace,
 * behind a flag barrier); the NCCL transport returns PIC_EINVAL.  Device
 * buffers for chi and rho_hat are written in place by the kernels; host
 * buffers (and J_hat, staged in the workspace for the neighbours) are filled
 * by copies.  Synchronises.                                                  */
PIC_API pic_status pic_implicit_sources(pic_ctx *ctx, double *chi, double *rho_hat, double *J_hat);

/* NEXT-3: inflow injection at the x = 0 face of an open x axis (PAPER.md:
 * 232-233, "wind electrons and protons are injected with a prescribed bulk
 * velocity"; reading R28).  From the next pic_mover on, every cycle places ppc
 * particles of species s uniformly in each ghost cell (-1, cy, cz) of the face,
 * velocities drift + vth * N(0,1)^3 (Box-Muller on Philox4x32-10 draws keyed by
 * seed, counter {face cell, index, cycle, species << 8 | draw}), charge q per
 * particle, id 2^62 | cycle << 40 | s << 37 | (face cell * ppc + index); each is
 * pushed one step with Eq. 2 and joins the store iff it ends inside the domain.
 * Applied on the rank whose slab starts at x = 0.  ppc = 0 switches it off.   */
PIC_API pic_status pic_set_injection(pic_ctx *ctx, int32_t s, int32_t ppc, double vth, const double drift[3],
                                     double q, uint64_t seed);

/* NEXT-3 particle control of species s on this rank (
 * readings R29-R31), between cycles.  Monitor: n = live count (synchronises);
 * n < target (1 - theta): splitting — each particle splits with probability
 * p = min(1, (target - n)/n) (Philox draw keyed by its id, seed and the cycle)
 * into two of half charge at x -/+ eps Delta e, e a random unit vector, unless
 * a child would leave the cell; n > target (1 + theta): coalescence — in each
 * cell with >= 2 particles (any number: cells of more than 512 particles or
 * with a velocity bin beyond +-2^20 take an unpacked global-memory sort)
 * sorted by (floor(v/dv) per component, id), neighbours with equal velocity
 * bins merge pair-wise (charge-weighted x and v; the smaller id survives)
 * until floor(frac n_c) merges, frac = (n - target)/n.  Uses the store's
 * second buffer as scratch.  *action: 0 none, 1 split, 2 coalesced.         */
PIC_API pic_status pic_control(pic_ctx *ctx, int32_t s, int64_t target, double theta, double eps, double dv,
                               uint64_t seed, int32_t *action);

/* NEXT-4 physics-aware compression (readings R32, R33) of
 * species s on this rank, between cycles: the velocity histogram with B bins
 * per axis over [-vmax, vmax) (weights |q|, out-of-range particles clipped to
 * the edge bins and counted in *clipped), then a Gaussian-mixture fit with M
 * components by n_em EM iterations on the bin centres (heaviest-bin +
 * farthest-point seeding, covariance floor 1e-6 (2 vmax / B)^2).  Outputs
 * (host or device, any may be NULL): alpha[M], mu[M][3], sigma[M][6] (xx xy xz
 * yy yz zz), hist[B][B][B] ([bz][by][bx]).  1 <= B <= 64, 1 <= M <= 8.
 * Synchronises.                                                              */
PIC_API pic_status pic_gmm(pic_ctx *ctx, int32_t s, int32_t B, double vmax, int32_t M, int32_t n_em, double *alpha,
                           double *mu, double *sigma, double *hist, int64_t *clipped);

/* Zero-copy access to the ghosted moment arrays of species s (device memory,
 * valid after pic_exchange until the next pic_moments): *ptr points at owned
 * node (0, 0, 0) of component comp (0..9: rho, Jx, Jy, Jz, Pxx, Pxy, Pxz,
 * Pyy, Pyz, Pzz), element (i, j, k) at ptr[i strides[0] + j strides[1] +
 * k strides[2]] for i, j, k < pic_moment_shape, global node origin + (i, j,
 * k).  Values are the raw sums sum q S {1, v, vv}; multiply by *scale = 1/V. */
PIC_API pic_status pic_moment_ptr(const pic_ctx *ctx, int32_t s, int32_t comp, const double **ptr,
                                  int64_t strides[3], int64_t origin[3], double *scale);

/* Make the context stream wait (on the device, no host block) for every copy
 * enqueued by pic_get_moments_async / pic_set_fields so far.                 */
PIC_API pic_status pic_join_copies(pic_ctx *ctx);

/* Transport in use: PIC_TRANSPORT_PEER, _NCCL or _LOOPBACK when nranks > 1
 * (AUTO resolved at pic_init), PIC_TRANSPORT_AUTO for a single rank.        */
PIC_API pic_status pic_get_transport(const pic_ctx *ctx, int32_t *out);

/* Number of libpic kernel launches enqueued on this context since pic_init
 * (the bench's gpu_launches evidence).                                       */
PIC_API pic_status pic_launch_count(const pic_ctx *ctx, int64_t *n);

/* Kernel timing with CUDA events recorded on the context stream around the
 * launches of each phase.  pic_profile(ctx, 1) resets and enables it (events
 * cost nothing measurable), 0 disables it.  pic_profile_read synchronises the
 * stream and returns accumulated milliseconds and launch counts:
 *   ms[0] mover kernels (Eq. 2), ms[1] order build (scan + perm scatter),
 *   ms[2] deposit kernels (Eq. 3), ms[3] pic_exchange (folds, ghost sums),
 *   ms[4] migration up to the count message (pack + NCCL counts),
 *   ms[5] migration after the host learnt the counts (payload + append);
 *   the host wait between ms[4] and ms[5] is in neither;
 *   ms[6] inflow injection (NEXT-3).
 *   launches[k] the number of timed intervals of each phase.                 */
#define PIC_PROF_PHASES 7
PIC_API pic_status pic_profile(pic_ctx *ctx, int32_t enable);
PIC_API pic_status pic_profile_read(pic_ctx *ctx, double ms[PIC_PROF_PHASES], int64_t launches[PIC_PROF_PHASES]);

/* Human-readable text of the last error on this context (never NULL).       */
PIC_API const char *pic_last_error(const pic_ctx *ctx);

/* Free the context (not the workspace).                                      */
PIC_API pic_status pic_destroy(pic_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* PIC_H */
