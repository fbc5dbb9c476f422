// pic_internal.cuh — context, store layout and shared device helpers of libpic.
//
// Internal representation:
//   * particle store, per species, SoA fp64 in two buffers (A = state, B =
//     mover destination): xi_x, xi_y, xi_z (positions in GLOBAL CELL UNITS,
//     xi_d = x_d / Delta_d), u, v, w (velocity, caller units), q (charge
//     q_s w_p, R14); int64 id.  The cell order is an indirection (perm) built
//     by a counting sort (order.cu, SpeciesStore below).
//   * key_new (uint32 per particle), written by the mover: the tile-major cell
//     key of x^{n+1} for live particles that stay, or one of the reserved tail
//     keys KEY_LEFT / KEY_RIGHT (slab leavers) / KEY_DEAD (removed, R21).
//   * field window: node-interleaved [kz][ky][kx][6] fp64, exactly the layout
//     of pic_set_fields (global nodes [slab_lo-G, slab_hi+G] x [-G, Ny+G] x
//     [-G, Nz+G]).
//   * moments, per species: 10 x [nzm][nym][nxm] fp64 raw sums
//     sum_p q {1, v, vv} S (the 1/V of R13 is applied when copying out);
//     x planes [slab_lo-G, slab_hi+G], y planes [0, Ny], z planes [0, Nz]
//     (the extra periodic plane is folded by pic_exchange, R18).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "pic.h"

namespace pic {

constexpr uint32_t KEY_DEAD = 0xFFFFFFFFu;
constexpr uint32_t KEY_RIGHT = 0xFFFFFFFEu;
constexpr uint32_t KEY_LEFT = 0xFFFFFFFDu;
constexpr uint32_t KEY_FIRST_RESERVED = 0xFFFFFFFDu;

// device counters (stats of pic_sync)
enum Stat {
  ST_REMOVED = 0, ST_SENT = 1, ST_RECEIVED = 2, ST_FAR = 3, ST_CLAMPED = 4,
  ST_NONFINITE = 5, ST_OVERFLOW = 6, ST_MULTIWRAP = 7,
  ST_CHECK = 8,     // failed device bounds checks (PIC_CHECKED builds only)
  ST_N = 9
};
constexpr int ST_PUBLIC = 8;   // counters returned by pic_sync

// Device bounds checks of the checked build (-DPIC_CHECKED; tools/checked_run.sh):
// every sub-array lives inside ONE workspace allocation, so an index past the
// end of an array would silently hit its neighbour (no fault, and
// compute-sanitizer's memcheck would not see it either).  The checked build
// counts every violated index invariant in stats[ST_CHECK], which pic_sync turns
// into PIC_ECUDA; the release build compiles the checks away.
#ifdef PIC_CHECKED
#define PIC_DCHECK(cond, stats)                                   \
  do {                                                            \
    if (!(cond)) atomicAdd(&(stats)[::pic::ST_CHECK], 1ull);      \
  } while (0)
#else
#define PIC_DCHECK(cond, stats) \
  do {                          \
  } while (0)
#endif

// Grid sizing of the grid-stride kernels: multiples of the B200's 148 SMs
// (the loops stay correct on any SM count).
constexpr int kSMs = 148;

// Slab migration records: x y z u v w q and the id bits, 8 words per particle.
constexpr int MIG_REC = 8;

// Control words of the peer transport (peer.cu), in the workspace of every rank
// and written by its neighbours over NVLink.
struct PeerCtl {
  unsigned long long flag[2];      // barrier epochs: [0] from the left neighbour, [1] from the right
  unsigned long long err;          // barrier timeouts
  unsigned long long epoch;        // own barrier epoch (advanced by the own barrier kernel only)
  unsigned long long cnt[2][PIC_MAX_SPECIES];   // arrivals reserved by [0] left / [1] right neighbour
  // forwarded far-flyers (R22, far_hops > 0): [hop parity][from side][species]
  unsigned long long fcnt[2][2][PIC_MAX_SPECIES];
};

// What a sender needs to write one species' leavers into its neighbours'
// receive buffers (side 0: left neighbour, 1: right; null = no peer link).
struct PeerOut {
  double *buf[2];
  unsigned long long *cnt[2];
  int64_t cap[2];
};

// Geometry passed by value to kernels.
struct Geom {
  int64_t ncell[3];       // global cells
  int32_t periodic[3];
  double delta[3];        // cell size
  double inv_delta[3];
  double dt, c;
  double planet_c[3];     // planet centre in CELL units
  double planet_r2;       // radius^2 in physical units (compared in physical units)
  int32_t has_planet;
  int64_t slab_lo, slab_hi;
  int32_t G;
  int32_t multi_rank;     // nranks > 1 (slab leavers migrate)
  int32_t far_hops;       // forwarding rounds for far-flyers (peer / loopback transports)
  // field window
  int64_t f_lo[3];        // global node index of window element 0
  int64_t f_n[3];         // window nodes per axis
  // moments
  int64_t m_lo[3];        // global node index of element 0 of the ghosted arrays
  int64_t m_n[3];         // ghosted node counts (x, y, z)
  int64_t m_plane;        // m_n[0]*m_n[1]*m_n[2] (stride between components)
  // local cell box used for the sort key
  int64_t k_n[3];         // local cells (slab_hi-slab_lo, Ny, Nz)
  int64_t nt[3];          // tiles per axis (ceil(k_n / TILE))
  int64_t ntiles;
  int64_t ncells;         // ntiles * TILE^3 (key range)
};

// Cell tiles of TILE^3 cells: the sort key is tile-major,
//   key = tile * TILE^3 + (lx % T) + T (ly % T) + T^2 (lz % T),
//   tile = tx + nt_x (ty + nt_y tz),  t_d = l_d / T,
// with l = local cell (x relative to slab_lo).
constexpr int TILE = 4;
constexpr int TILE3 = TILE * TILE * TILE;

__host__ __device__ __forceinline__ uint32_t tile_key(const Geom &g, int64_t lx, int64_t ly, int64_t lz) {
  const int64_t t = (lx / TILE) + g.nt[0] * ((ly / TILE) + g.nt[1] * (lz / TILE));
  return (uint32_t)(t * TILE3 + (lx % TILE) + TILE * (ly % TILE) + TILE * TILE * (lz % TILE));
}

// Particle store of one species.  Buffer A holds the state at
// positions [0, n_raw); the cell order of the live particles is an indirection:
// perm[q] = A-position of the q-th particle in tile-major cell order, key[q] its
// key, cell_off[c] the first q of cell c (exclusive scan of cell_count, built by
// a counting sort whose ranks the mover produces while it moves).  The movers
// gather A[perm[q]] and write B[q] (then A <-> B), so the store comes out of
// every cycle already in the order of the next one.  Dead particles and slab
// leavers are simply not counted, which drops them from the next order.
struct SpeciesStore {
  double *a[7] = {};      // A: xi_x xi_y xi_z u v w q
  int64_t *id = nullptr;
  double *b[7] = {};      // B: mover destination
  int64_t *id_b = nullptr;
  uint32_t *key_new = nullptr;    // [cap] key of the particle at A-position p
  uint32_t *rank = nullptr;       // [cap] rank of A-position p within its cell
  uint32_t *perm = nullptr;       // [cap] q -> A-position (cell order)
  uint32_t *cell_count = nullptr; // [2][ncells + 1]: stayers (kept their cell), arrivals
  uint32_t *cell_tot = nullptr;   // [ncells + 1] stayers + arrivals (scan input)
  uint32_t *cell_off = nullptr;   // [ncells + 1]; cell_off[ncells] = live count
  int64_t *d_nraw = nullptr;      // device scalar: number of A positions
  double *mom = nullptr;  // [10][m_plane]
  int64_t n_raw = 0;      // host upper bound of the A positions in use
  int64_t n = 0;          // host mirror of the live count (exact after pic_count / sync)
  int64_t cap = 0;
  double qom = 0;
  int32_t n_iter = 3;
  bool moved = false, deposited = false;
  bool order_valid = false;
  bool order_dirty = false;  // positions appended since the last order build (ensure_order)
  void swap_buffers() {
    for (int k = 0; k < 7; ++k) { double *t = a[k]; a[k] = b[k]; b[k] = t; }
    int64_t *t = id; id = id_b; id_b = t;
  }
};

// NEXT-3 inflow injection of one species (pic_set_injection).
struct InjectParams {
  int ppc = 0;             // ghost particles per face cell per cycle (0: off)
  double vth = 0.0, drift[3] = {0.0, 0.0, 0.0}, q = 0.0;
  uint64_t seed = 0;
};

struct Ctx {
  pic_config cfg;
  Geom geom;
  cudaStream_t stream = nullptr;
  SpeciesStore sp[PIC_MAX_SPECIES];
  // field window, double-buffered: pic_set_fields copies into the buffer the
  // next mover will use (on copy_stream) while the current one may still be read
  double *field_buf[2] = {};
  int field_cur = 0;                 // buffer of the last / next mover
  bool field_new = false;            // pic_set_fields since the last mover: switch
  cudaEvent_t field_ready[2] = {}, field_free[2] = {};
  double *field() const { return field_buf[field_cur]; }
  // asynchronous moment copy-out (pic_get_moments_async): 2 staging slots per species
  cudaStream_t copy_stream = nullptr;   // device -> host moment copies
  cudaStream_t h2d_stream = nullptr;    // field copies (separate: never queued behind a moment copy)
  double *pack_slot[2 * PIC_MAX_SPECIES] = {};
  cudaEvent_t slot_packed[2 * PIC_MAX_SPECIES] = {}, slot_free[2 * PIC_MAX_SPECIES] = {};
  bool slot_used[2 * PIC_MAX_SPECIES] = {};
  int slot_next[PIC_MAX_SPECIES] = {};
  cudaEvent_t copies_done = nullptr, fields_done = nullptr;
  bool copies_pending = false;
  int64_t field_elems = 0;
  bool fields_set = false;
  unsigned long long *stats = nullptr;  // ST_N device counters
  int64_t *dev_counts = nullptr;     // small device scratch for counts
  int64_t *host_counts = nullptr;    // pinned host [64] (migration counts)
  // exchange buffers
  double *ghost_send[2] = {};        // [0] to left, [1] to right
  double *ghost_recv[2] = {};
  int64_t ghost_elems = 0;           // per buffer
  double *mig_send[2] = {};          // [8][mig_cap] per side (7 fp64 + id as fp64 bits)
  double *mig_recv[2] = {};
  int64_t mig_cap = 0;
  double *pack = nullptr;            // moment copy-out staging
  double *src_buf = nullptr;         // NEXT-2 sources: chi [9], J-hat [3], rho-hat [1] per owned node
  double *gmm_buf = nullptr;         // NEXT-4: velocity histogram [64^3] + mixture parameters
  void *workspace = nullptr;         // caller's device workspace (pic_init)
  // peer transport (peer.cu): own control block and the mapped neighbours
  PeerCtl *peer_ctl = nullptr;
  struct PeerLink {
    char *mapped = nullptr;          // neighbour's workspace allocation (CUDA IPC)
    bool owns_mapping = false;
    unsigned long long *flag = nullptr, *cnt = nullptr;   // my slots in its PeerCtl
    double *recv = nullptr;          // its receive records from me
    int64_t mig_cap = 0;
    double *mom[PIC_MAX_SPECIES] = {};
    int64_t m_plane = 0, m_nx = 0, ghost_x = 0;
    double *src = nullptr;           // its NEXT-2 sources buffer
    int64_t owned_nx = 0;
    unsigned long long *fcnt[2] = {};  // my forward slots in its PeerCtl, per hop parity
    double *frecv[2] = {};           // its forward records from me, per hop parity
    int64_t fwd_cap = 0;
  } link[2];                         // [0] left, [1] right
  double *fwd_recv[2][2] = {};       // own forward regions [hop parity][from side] (in mig_send)
  int64_t fwd_cap = 0;               // records per region and species
  bool peer = false;
  Ctx *loop_nb[2] = {};              // loopback transport: the neighbour contexts (same process)
  struct LoopGroup *loop = nullptr;  // loopback transport: shared host-side barrier state (peer.cu)
  unsigned long long peer_epoch = 0;   // loopback transport: host-side barrier epochs
  // CUDA graphs of whole cycles (pic_set_graph): one per (field buffer, store
  // buffer parity), since the kernels' arguments differ only in those
  bool graph_on = false;
  struct CycleGraph {
    void *exec = nullptr;            // cudaGraphExec_t
    int field_cur = -1;
    const double *a0 = nullptr;      // species 0 buffer A at capture
    int64_t launches = 0;
  } graphs[4];
  InjectParams inj[PIC_MAX_SPECIES];
  void *cub_temp = nullptr;
  size_t cub_bytes = 0;
  void *nccl = nullptr;              // ncclComm_t
  int64_t hstat[8] = {};             // host-side counters (sent / received)
  int64_t launches = 0;              // libpic kernel launches (pic_launch_count)
  alignas(64) unsigned char tmap[2][128] = {};  // CUtensorMaps of the two field windows (tiled.cu)
  bool tmap_ok = false;
  int64_t cycle = 0;
  int64_t cap_max = 0;
  std::string err;
  // pic_profile: CUDA event pairs per phase (0 mover, 1 order, 2 deposit,
  // 3 ghost exchange, 4 migration before the count sync, 5 after it, 6 injection)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[PIC_PROF_PHASES];
  cudaEvent_t prof_event() {
    if (!prof_pool.empty()) {
      cudaEvent_t e = prof_pool.back();
      prof_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

// Records an event pair around a phase when profiling is on (RAII).
struct PhaseTimer {
  Ctx *ctx;
  int phase;
  cudaEvent_t start = nullptr;
  PhaseTimer(Ctx *c, int ph) : ctx(c), phase(ph) {
    if (ctx->prof_on) {
      start = ctx->prof_event();
      cudaEventRecord(start, ctx->stream);
    }
  }
  ~PhaseTimer() {
    if (start) {
      cudaEvent_t stop = ctx->prof_event();
      cudaEventRecord(stop, ctx->stream);
      ctx->prof_ev[phase].emplace_back(start, stop);
    }
  }
};

// ------------------------------------------------------------ error helpers --
#define PIC_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      return ::pic::fail(ctx, PIC_ECUDA, std::string(#call) + ": " +          \
                                             cudaGetErrorString(e_));         \
    }                                                                         \
  } while (0)

inline pic_status fail(Ctx *ctx, pic_status s, const std::string &m) {
  if (ctx) ctx->err = m;
  return s;
}

// -------------------------------------------------------------- launchers ----
// (implemented in the .cu files; all enqueue on ctx->stream)
pic_status launch_mover_basic(Ctx *ctx, int s);
pic_status launch_moments_basic(Ctx *ctx, int s);
pic_status launch_tiled_deposit(Ctx *ctx, int s0, int s1);
pic_status launch_tiled_step(Ctx *ctx, int s0, int s1);
size_t order_temp_bytes(int64_t ncells);
pic_status zero_cell_counts(Ctx *ctx, int s);
pic_status count_positions(Ctx *ctx, int s, int64_t from, int64_t to);
pic_status build_order(Ctx *ctx, int s);
// Rebuild the cell order if particles were appended since the last build
// (pic_add_particles defers it, so loading a store chunk by chunk builds it once).
pic_status ensure_order(Ctx *ctx, int s);
pic_status exchange(Ctx *ctx);
pic_status migrate(Ctx *ctx, int s0, int s1);
pic_status peer_setup(Ctx *ctx);
pic_status loopback_link(Ctx *const *ctxs, int n);
void peer_close(Ctx *ctx);
PeerOut peer_out(const Ctx *ctx, int s);
pic_status peer_migrate(Ctx *ctx, int s0, int s1);
pic_status peer_exchange(Ctx *ctx);
pic_status peer_barrier(Ctx *ctx);
pic_status recompute_keys(Ctx *ctx, int s, int64_t from, int64_t to);
pic_status zero_moments(Ctx *ctx, int s);
pic_status pack_moments(Ctx *ctx, int s, double *out);
pic_status pack_moments_async(Ctx *ctx, int s, double *out);
pic_status join_copies(Ctx *ctx);
pic_status implicit_sources(Ctx *ctx, double *chi, double *rho_hat, double *J_hat);
pic_status inject(Ctx *ctx, int s);
// After an append kernel whose slot counter may have run past the capacity
// (those appends were dropped and counted as overflow): d_nraw = min(d_nraw, cap).
pic_status clamp_nraw(Ctx *ctx, int s);
pic_status control(Ctx *ctx, int s, int64_t target, double theta, double eps, double dv, uint64_t seed,
                   int32_t *action);
pic_status live_count(Ctx *ctx, int s, int64_t *n);
pic_status append_particles(Ctx *ctx, int s, int64_t n, const double *const src[7], const int64_t *id);
pic_status load_particles(Ctx *ctx, int s, int64_t n, const double *const src[7], const int64_t *id);
pic_status unload_particles(Ctx *ctx, int s, double *const dst[7], int64_t *id);
pic_status gmm_fit(Ctx *ctx, int s, int B, double vmax, int M, int n_em, double *alpha, double *mu, double *sigma,
                   double *hist_out, int64_t *clipped);

// ---------------------------------------------------------- device helpers ---
// Periodic wrap of a cell-unit coordinate (R10): one wrap, then test.
__device__ __forceinline__ double wrap_cells(double xi, double n, bool *multi) {
  if (xi >= n) {
    xi = xi - n;
  } else if (xi < 0.0) {
    xi = xi + n;
    if (xi == n) xi = 0.0;
  }
  if (!(xi >= 0.0 && xi < n)) *multi = true;
  return xi;
}

// Trilinear sample of the 6 field components of the global window at a
// cell-unit position (R11 clamp to the window, R12 weights).  Returns true if
// the position was clamped.
__device__ __forceinline__ bool sample_window(const Geom &g, const double *__restrict__ F,
                                              const double xb[3], double out[6]) {
  int64_t idx[3];
  double f[3];
  bool clamped = false;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double u = xb[d] - (double)g.f_lo[d];
    double top = (double)(g.f_n[d] - 1);
    if (!(u >= 0.0)) { u = 0.0; clamped = true; }
    if (u > top) { u = top; clamped = true; }
    double fl = floor(u);
    if (fl > top - 1.0) fl = top - 1.0;
    idx[d] = (int64_t)fl;
    f[d] = u - fl;
  }
#pragma unroll
  for (int m = 0; m < 6; ++m) out[m] = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1;
    double S = (bx ? f[0] : 1.0 - f[0]) * (by ? f[1] : 1.0 - f[1]) * (bz ? f[2] : 1.0 - f[2]);
    const double *node = F + 6 * (((idx[2] + bz) * g.f_n[1] + (idx[1] + by)) * g.f_n[0] + (idx[0] + bx));
#pragma unroll
    for (int m = 0; m < 6; ++m) out[m] = fma(S, __ldg(node + m), out[m]);
  }
  return clamped;
}

// Tile-major key of a local cell (lx relative to slab_lo), 32-bit arithmetic
// (valid while the key range fits 32 bits, which pic_init checks; TILE == 4).
__device__ __forceinline__ uint32_t tile_key32(const Geom &g, uint32_t lx, uint32_t ly, uint32_t lz) {
  static_assert(TILE == 4, "tile_key32 assumes 4^3 tiles");
  const uint32_t t = (lx >> 2) + (uint32_t)g.nt[0] * ((ly >> 2) + (uint32_t)g.nt[1] * (lz >> 2));
  return t * TILE3 + (lx & 3u) + 4u * (ly & 3u) + 16u * (lz & 3u);
}

// Boundary conditions (R10, R11, R21) of a pushed particle and its destination
// key.  xnew: in = pre-wrap position (cell units), out = post-wrap position.
// Non-finite values fail the range tests, so the finiteness check only runs on
// the rare flagged path.  Fast path: the particle is still inside this rank's
// slab and the domain (no wrap, no leaver, no open face) and outside the planet,
// which is every particle but the few that cross a face this step.
// `old_cell` (optional): the particle's cell before the push and its key; a
// particle still in that cell keeps the key without recomputing it.
struct OldCell {
  int c[3];
  uint32_t key;
};
__device__ __forceinline__ uint32_t finish_particle(const Geom &g, double xnew[3], const double vnew[3],
                                                   bool clamped, unsigned long long *__restrict__ stats,
                                                   const OldCell *old_cell = nullptr) {
  if (xnew[0] >= (double)g.slab_lo && xnew[0] < (double)g.slab_hi && xnew[1] >= 0.0 &&
      xnew[1] < (double)g.ncell[1] && xnew[2] >= 0.0 && xnew[2] < (double)g.ncell[2]) {
    bool hit = false;
    if (g.has_planet) {
      double r2 = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double dx = (xnew[d] - g.planet_c[d]) * g.delta[d];
        r2 += dx * dx;
      }
      hit = r2 < g.planet_r2;
    }
    if (!hit) {
      if (clamped) atomicAdd(&stats[ST_CLAMPED], 1ull);
      const int cx = (int)xnew[0], cy = (int)xnew[1], cz = (int)xnew[2];
      if (old_cell && cx == old_cell->c[0] && cy == old_cell->c[1] && cz == old_cell->c[2]) return old_cell->key;
      return tile_key32(g, (uint32_t)(cx - (int)g.slab_lo), (uint32_t)cy, (uint32_t)cz);
    }
  }
  const double x_pre = xnew[0];
  bool bad = false, out = false;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double N = (double)g.ncell[d];
    const double x = xnew[d];
    if (g.periodic[d]) {
      // R10: x >= L -> x - L; x < 0 -> x + L (and L -> 0); more than one wrap is bad
      const bool neg = x < 0.0;
      double y = (x >= N) ? x - N : (neg ? x + N : x);
      y = (neg && y == N) ? 0.0 : y;
      bad |= !(y >= 0.0 && y < N);
      xnew[d] = y;
    } else {
      out |= !(x >= 0.0 && x < N);   // left through an open face (or non-finite)
    }
  }
  if (g.has_planet && !bad && !out) {
    double r2 = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double dx = (xnew[d] - g.planet_c[d]) * g.delta[d];
      r2 += dx * dx;
    }
    out = r2 < g.planet_r2;
  }
  uint32_t k;
  if (bad || out) {
    const bool finite = isfinite(vnew[0]) && isfinite(vnew[1]) && isfinite(vnew[2]) &&
                        isfinite(xnew[0]) && isfinite(xnew[1]) && isfinite(xnew[2]);
    atomicAdd(&stats[!finite ? ST_NONFINITE : (bad ? ST_MULTIWRAP : ST_REMOVED)], 1ull);
    k = KEY_DEAD;
  } else if (g.multi_rank && x_pre < (double)g.slab_lo) {
    k = KEY_LEFT;
    if (g.far_hops == 0 && x_pre < (double)(g.slab_lo - g.G)) atomicAdd(&stats[ST_FAR], 1ull);
  } else if (g.multi_rank && x_pre >= (double)g.slab_hi) {
    k = KEY_RIGHT;
    if (g.far_hops == 0 && x_pre >= (double)(g.slab_hi + g.G)) atomicAdd(&stats[ST_FAR], 1ull);
  } else {
    const int cx = (int)xnew[0], cy = (int)xnew[1], cz = (int)xnew[2];
    k = tile_key32(g, (uint32_t)(cx - (int)g.slab_lo), (uint32_t)cy, (uint32_t)cz);
  }
  if (clamped) atomicAdd(&stats[ST_CLAMPED], 1ull);
  return k;
}

// Rank of a live particle within its cell for the counting sort.  Particles
// that kept their cell ("stayers") and arrivals are counted separately so
// that, in the next order, every cell lists its stayers first, in their
// previous order (a contiguous run of the previous store: coalesced gathers),
// then its arrivals.  A stayer gets its rank among the cell's stayers here
// (the lanes of a warp holding the same key share one atomicAdd).  An arrival
// is only counted (a reduction without return, so no kernel waits for it) and
// gets the rank RANK_ARRIVAL; perm_kernel places it after the cell's stayers
// with an atomic cursor.  All 32 lanes must call it; `counted == false` lanes
// get no rank.
constexpr uint32_t RANK_ARRIVAL = 0x80000000u;
// a reduction without return (RED): atomicAdd with an unused result still
// compiles to an ATOMG that later instructions wait for
__device__ __forceinline__ void red_add_u32(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t count_rank(uint32_t *__restrict__ cell_count, int64_t ncells, uint32_t k,
                                               bool counted, bool arrival) {
  const unsigned kk = counted ? (k | (arrival ? RANK_ARRIVAL : 0u)) : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xffffffffu, kk);
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (counted && (int)lane == leader) {
    if (arrival)
      red_add_u32(cell_count + ncells + 1 + k, (unsigned)__popc(peers));
    else
      base = atomicAdd(cell_count + k, (unsigned)__popc(peers));
  }
  base = __shfl_sync(0xffffffffu, base, leader);
  return arrival ? RANK_ARRIVAL : base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
}

// The tiled mover's rank, in two halves: a stayer's cell belongs to the
// CTA's own tile, and no other CTA counts stayers of that tile, so stayers are
// counted in shared memory (`scnt`, the tile's 64 cells; the CTA stores the
// totals at its end) and the short shared atomic's latency is hidden behind
// the next round (count_rank_finish, called later by all 32 lanes).
// Arrivals are counted with a global reduction, as in count_rank.  (A global
// atomic with return here held every round: ptxas shares its scoreboard with
// the next round's loads.)
struct RankTicket {
  uint32_t base;      // shared atomic result (leader lanes), consumed in finish
  unsigned peers;
  int leader;
  bool counted, arrival;
};
__device__ __forceinline__ RankTicket count_rank_issue(uint32_t *__restrict__ scnt, uint32_t tile_key0,
                                                       uint32_t *__restrict__ cell_count, int64_t ncells,
                                                       uint32_t k, bool counted, bool arrival) {
  RankTicket t;
  const unsigned kk = counted ? (k | (arrival ? RANK_ARRIVAL : 0u)) : 0xFFFFFFFFu;
  t.peers = __match_any_sync(0xffffffffu, kk);
  t.leader = __ffs(t.peers) - 1;
  t.counted = counted;
  t.arrival = arrival;
  t.base = 0;
  if (counted && (int)(threadIdx.x & 31u) == t.leader) {
    if (arrival)
      red_add_u32(cell_count + ncells + 1 + k, (unsigned)__popc(t.peers));
    else
      t.base = atomicAdd(scnt + (k - tile_key0), (unsigned)__popc(t.peers));
  }
  return t;
}
__device__ __forceinline__ uint32_t count_rank_finish(const RankTicket &t) {
  const unsigned lane = threadIdx.x & 31u;
  const uint32_t base = __shfl_sync(0xffffffffu, t.base, t.leader);
  return t.arrival ? RANK_ARRIVAL : base + (uint32_t)__popc(t.peers & ((1u << lane) - 1u));
}

// Peer transport, warp-collective (all 32 lanes): lanes whose new key is
// KEY_LEFT / KEY_RIGHT copy their record (read back from the output slot p the
// mover just wrote) straight into the neighbour's receive buffer over NVLink.
// One remote atomic per warp and side reserves the slots; a slot beyond the
// neighbour's capacity is an overflow (pic_sync reports it).  Each writer
// fences its stores at system scope before the barrier publishes them.
__device__ __forceinline__ void send_leavers_peer(const PeerOut &po, uint32_t k, const double *const dst[7],
                                                  const int64_t *dst_id, int64_t p,
                                                  unsigned long long *stats) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const bool mine = k == (side == 0 ? KEY_LEFT : KEY_RIGHT);
    const unsigned mask = __ballot_sync(0xffffffffu, mine);
    if (!mask) continue;
    const int leader = __ffs(mask) - 1;
    unsigned long long slot0 = 0;
    if ((int)lane == leader) {
      slot0 = po.cnt[side] ? atomicAdd(po.cnt[side], (unsigned long long)__popc(mask)) : ~0ull >> 1;
      atomicAdd(&stats[ST_SENT], (unsigned long long)__popc(mask));
    }
    slot0 = __shfl_sync(0xffffffffu, slot0, leader);
    if (mine) {
      const int64_t slot = (int64_t)slot0 + __popc(mask & ((1u << lane) - 1u));
      if (slot < po.cap[side]) {
        double *rec = po.buf[side] + slot * MIG_REC;
#pragma unroll
        for (int c = 0; c < 7; ++c) rec[c] = dst[c][p];
        rec[7] = __longlong_as_double(dst_id[p]);
        __threadfence_system();
      } else {
        atomicAdd(&stats[ST_OVERFLOW], 1ull);
      }
    }
  }
}

// Eq. 3 deposit of one particle with global fp64 atomics (80 RED), at a
// cell-unit position relative to the ghosted moment arrays (basic family).
// Returns false if the stencil is outside.
__device__ __forceinline__ bool deposit_global(const Geom &g, double *__restrict__ mom, const double xi[3], double q,
                                               const double v[3]) {
  int64_t idx[3];
  double f[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double u = xi[d] - (double)g.m_lo[d];
    const double fl = floor(u);
    idx[d] = (int64_t)fl;
    f[d] = u - fl;
  }
  if (idx[0] < 0 || idx[0] > g.m_n[0] - 2 || idx[1] < 0 || idx[1] > g.m_n[1] - 2 || idx[2] < 0 ||
      idx[2] > g.m_n[2] - 2)
    return false;
  const double qu = q * v[0], qv = q * v[1], qw = q * v[2];
  const double val[10] = {q, qu, qv, qw, qu * v[0], qu * v[1], qu * v[2], qv * v[1], qv * v[2], qw * v[2]};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int bx = c & 1, by = (c >> 1) & 1, bz = c >> 2;
    const double S = (bx ? f[0] : 1.0 - f[0]) * (by ? f[1] : 1.0 - f[1]) * (bz ? f[2] : 1.0 - f[2]);
    const int64_t node = ((idx[2] + bz) * g.m_n[1] + (idx[1] + by)) * g.m_n[0] + (idx[0] + bx);
#pragma unroll
    for (int m = 0; m < 10; ++m) atomicAdd(mom + m * g.m_plane + node, S * val[m]);
  }
  return true;
}

// Map a global node index to the ghosted moment array (x: ghost planes; y, z:
// planes [0, N] with periodic images of -1 / N+1 wrapped).  -1 if outside.
__device__ __forceinline__ int64_t moment_node(const Geom &g, int64_t gx, int64_t gy, int64_t gz) {
  const int64_t ax = gx - g.m_lo[0];
  if (ax < 0 || ax >= g.m_n[0]) return -1;
  const int64_t Ny = g.ncell[1], Nz = g.ncell[2];
  if (g.periodic[1]) { if (gy < 0) gy += Ny; else if (gy > Ny) gy -= Ny; }
  if (g.periodic[2]) { if (gz < 0) gz += Nz; else if (gz > Nz) gz -= Nz; }
  if (gy < 0 || gy > Ny || gz < 0 || gz > Nz) return -1;
  return (gz * g.m_n[1] + gy) * g.m_n[0] + ax;
}

}  // namespace pic
