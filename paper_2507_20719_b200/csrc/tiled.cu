// tiled.cu — PIC_KERNEL_TILED: cell-ordered, tile-staged mover and deposit.
//
// The store is kept in tile-major cell order through an indirection (order.cu):
// tile t owns q in [cell_off[64 t], cell_off[64 (t+1)]), perm[q] is the
// particle's position in buffer A.  One CTA per tile of TILE^3 cells.
//
// mover_tiled_kernel  (pic_mover; Eq. 2)
//  1. TMA (cp.async.bulk.tensor.4d + mbarrier) stages the E,B nodes of the tile
//     plus a one-cell halo, 7^3 nodes x 48 B, from the field window into shared
//     memory; the CTA pre-scales them by k_s = (q/m) dt/2 and k_s / c so the
//     iteration reads E' = k_s E and a = k_s B / c directly (R7, R8).
//  2. Warps split the tile's particles evenly; lane = particle, rounds of 32.
//     perm runs PK_AHEAD rounds ahead and the sources x, v SRC_STAGES - 1
//     rounds ahead through cp.async (LDGSTS) rings in shared memory (mostly
//     contiguous runs: every cell lists its stayers first); q and id, which
//     only pass through, go straight to registers.  n_iter predictor-
//     corrector iterations (R1, R2) with trilinear gathers from shared memory
//     (R12); x^{n+1}, v^{n+1}, boundary conditions (R10, R11, R21; fast path
//     for particles that stay inside the slab); the result goes to buffer B at
//     q and the new cell key is counted for the counting sort of the next
//     order (a particle that keeps its cell is ranked with a shared-memory
//     atomic that completes during the next round; an arrival is only
//     counted, with a global reduction).  With the
//     peer transport, slab leavers are written straight into the neighbour's
//     receive buffer (send_leavers_peer).  REL = 1 instantiates the
//     relativistic Eq. 2 (NEXT-1).
//
// deposit_tiled_kernel  (pic_moments; Eq. 3)
//  Runs over the NEW order, so every particle of a cell segment really is in
//  that cell.  Warp ranges are cell-aligned; per round each lane computes its
//  particle's 8 corner weights S and 10 values q{1, v, vv} and stages them in
//  shared memory (XOR-swizzled, conflict-free); for each run of equal cells
//  the corner sums M = S^T V are accumulated on the fp64 tensor cores
//  (mma.m8n8k4: 8 corners x 4 particles x 8 + 8 moments), flushed into the
//  tile's shared node sums (5^3 x 10, shared atomics only at cell changes)
//  and finally added to the global ghosted moment arrays with fp64 atomics
//  (tile faces are shared).  The paper's "GPU-shared memory ... and atomic
//  operations", privatised per tile, reduced on tensor cores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "pic_internal.cuh"
#include "push.cuh"

namespace pic {

constexpr int NB = TILE + 3;            // staged field nodes per axis: -1 .. TILE+1
constexpr int NB3 = NB * NB * NB;       // 343
constexpr int MB = TILE + 1;            // deposit nodes per axis: 0 .. TILE
constexpr int MB3 = MB * MB * MB;       // 125
#ifndef PIC_SRC_STAGES
#define PIC_SRC_STAGES 2
#endif
constexpr int SRC_STAGES = PIC_SRC_STAGES;   // mover: rounds of gathered sources in flight (ring)
#ifndef PIC_PK_AHEAD
#define PIC_PK_AHEAD 3
#endif
constexpr int PK_AHEAD = PIC_PK_AHEAD;   // mover: perm fetched this many rounds ahead
constexpr int PK_SLOTS = PK_AHEAD + 1;   // mover: perm ring slots
#ifndef PIC_SRC_RING_SLOTS
#define PIC_SRC_RING_SLOTS 8
#endif
constexpr int SRC_STAGED = 6;            // mover: x, v staged in the ring (q, id go straight to registers)
constexpr int SRC_RING = PIC_SRC_RING_SLOTS;   // ring stage pitch in 32-double rows (>= SRC_STAGED;
                                              // 8 measured 1 % faster than 6)
constexpr int MOVER_WARP_STAGE = SRC_STAGES * SRC_RING * 32 + PK_SLOTS * 2 * 32 / 2;  // doubles per warp
// deposit staging per warp: S[32 particles][8 corners], V[32][moments 0..7]
// and V2[32][moments 8, 9].  S and V rows are 8 doubles whose 16-byte pairs
// are XOR-swizzled by row (stage_slot) so that both the row writes (STS.128,
// 8 consecutive rows per quarter-warp) and the MMA fragment reads (lanes
// (g, j) -> row 4t + j, column g) are free of bank conflicts.
constexpr int WBUF = 32 * 8 * 2 + 32 * 2;
#ifndef PIC_DEP_NACC
#define PIC_DEP_NACC 2
#endif
constexpr int NACC = PIC_DEP_NACC;               // independent MMA accumulator sets
#ifndef PIC_DEP_WARPS
#define PIC_DEP_WARPS 8
#endif
#ifndef PIC_DEP_MINB
#define PIC_DEP_MINB 3
#endif
constexpr int DWARPS = PIC_DEP_WARPS, DTHREADS = 32 * DWARPS;   // deposit CTA (one tile)
constexpr size_t DEPOSIT_SMEM = sizeof(double) * (MB3 * 10 + DWARPS * WBUF);

// Per-species arguments of the movers; one launch moves every species of
// pic_mover (species-major blocks: blockIdx.x = s * ntiles + tile), so the
// tail of one species' tiles overlaps the next species' first ones.
struct MoverSp {
  const double *src[7];       // buffer A (read through perm)
  const int64_t *src_id;
  double *dst[7];             // buffer B (written in cell order)
  int64_t *dst_id;
  const uint32_t *perm;       // q -> A-position
  const uint32_t *cell_off;   // tile t covers q in [cell_off[64 t], cell_off[64 (t+1)])
  uint32_t *key_new, *rank, *cell_count;
  int64_t *d_nraw;
  double ks, ks_c;
  PeerOut po;
  int64_t cap;                // store capacity (bounds checks of the checked build)
};

struct MoverTArgs {
  Geom g;
  MoverSp sp[PIC_MAX_SPECIES];
  const double *field;        // global window (fallback sampling)
  unsigned long long *stats;
  int n_iter;
  int peer;                   // slab leavers go straight into the neighbours' buffers (peer.cu)
};

struct DepositSp {
  const double *src[7];       // particle state (buffer A after the mover)
  const uint32_t *perm;       // new order
  const uint32_t *cell_off;
  double *mom;                // ghosted moment arrays [10][m_plane]
  int64_t cap;
};

struct DepositArgs {
  Geom g;
  DepositSp sp[PIC_MAX_SPECIES];
  unsigned long long *stats;
};

// ------------------------------------------------------------- PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// Trilinear gather of the pre-scaled fields from the staged box.  u = position
// in box node units.  Returns false if the 8 nodes are not all in the box.
__device__ __forceinline__ bool gather_smem(const double *__restrict__ fld, const double u[3], double out[6]) {
  double fl[3], f[3];
  int i[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    fl[d] = floor(u[d]);
    f[d] = u[d] - fl[d];
    i[d] = (int)fl[d];
  }
  if (!((unsigned)i[0] <= (unsigned)(NB - 2) && (unsigned)i[1] <= (unsigned)(NB - 2) &&
        (unsigned)i[2] <= (unsigned)(NB - 2)))
    return false;
  const double gx0 = 1.0 - f[0], gy0 = 1.0 - f[1], gz0 = 1.0 - f[2];
  const double w00 = gy0 * gz0, w10 = f[1] * gz0, w01 = gy0 * f[2], w11 = f[1] * f[2];
  const double S[8] = {gx0 * w00, f[0] * w00, gx0 * w10, f[0] * w10,
                       gx0 * w01, f[0] * w01, gx0 * w11, f[0] * w11};
  const int base = ((i[2] * NB + i[1]) * NB + i[0]) * 6;
#pragma unroll
  for (int m = 0; m < 6; ++m) out[m] = 0.0;
  auto accumulate = [&](const double *cell) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double *nd = cell + 6 * ((c & 1) + NB * ((c >> 1) & 1) + NB * NB * (c >> 2));
      const double2 a = *reinterpret_cast<const double2 *>(nd);
      const double2 b = *reinterpret_cast<const double2 *>(nd + 2);
      const double2 e = *reinterpret_cast<const double2 *>(nd + 4);
      out[0] = fma(S[c], a.x, out[0]);
      out[1] = fma(S[c], a.y, out[1]);
      out[2] = fma(S[c], b.x, out[2]);
      out[3] = fma(S[c], b.y, out[3]);
      out[4] = fma(S[c], e.x, out[4]);
      out[5] = fma(S[c], e.y, out[5]);
    }
  };
  accumulate(fld + base);
  return true;
}

// PIC_GATHER_MMA = 1 selects gather_mma below in the gamma == 1 mover.  It is
// correct (parity green) but measured 2.1x slower than the per-lane gather
// (C2: mover 5.59 vs 2.66 ms per step): its shuffles, weights,
// dependent DMMA pairs and transpose lengthen every iterate's critical path,
// and the mover is latency-bound at 16 warps per SM.  Kept as the measured
// alternative; off by default.
#ifndef PIC_GATHER_MMA
#define PIC_GATHER_MMA 0
#endif
__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// The trilinear gather of the staged box as a contraction on the fp64 tensor
// cores (warp-collective: all 32 lanes call it, each with its own particle's
// position).  For the particles of one cell the gather is the matrix product
//   EB[particle][component] = sum_corner S[particle][corner] F[corner][component]
// with the cell's 8 corner nodes F (8 x 6, padded to 8 x 8) shared by all of
// them: mma.m8n8k4 with M = 8 particles, K = 4 corners (two K-steps: z = 0, 1),
// N = 8 components.  F is the B operand, two doubles per lane read from shared
// memory once per distinct cell of the warp — instead of all 48 values into
// every lane (the 128 B/clk shared-memory crossbar bound of the per-lane gather).
// Lane L = 4 g + j owns particle (t = j, g) — row g of M-tile t; the A operand
// of lane (g, j) is the weight of corner (kk, j) of particle (t, g), computed
// from that particle's fractional position (shuffled within the quad); the C
// fragment (components 2j, 2j+1 of particle (t, g)) is transposed back to its
// owner within the quad.  A particle whose cell is not in the box returns false
// (the caller samples the global window).
__device__ __forceinline__ bool gather_mma(const double *__restrict__ fld, const double u[3], double out[6]) {
  constexpr unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u, j = lane & 3u, gq = lane >> 2;
  const unsigned quad = lane & ~3u;
  double f[3];
  int i[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double fl = floor(u[d]);
    f[d] = u[d] - fl;
    i[d] = (int)fl;
  }
  const bool inbox = (unsigned)i[0] <= (unsigned)(NB - 2) && (unsigned)i[1] <= (unsigned)(NB - 2) &&
                     (unsigned)i[2] <= (unsigned)(NB - 2);
  const int cell = inbox ? ((i[2] * NB + i[1]) * NB + i[0]) * 6 : -1;
  // A operands: a[t][kk] = weight of corner (x = j & 1, y = j >> 1, z = kk) of
  // the particle of lane quad + t
  double a[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const double fx = __shfl_sync(FULL, f[0], quad | t);
    const double fy = __shfl_sync(FULL, f[1], quad | t);
    const double fz = __shfl_sync(FULL, f[2], quad | t);
    const double wx = (j & 1u) ? fx : 1.0 - fx;
    const double wy = (j & 2u) ? fy : 1.0 - fy;
    const double wxy = wx * wy;
    a[t][0] = wxy * (1.0 - fz);
    a[t][1] = wxy * fz;
  }
  // one pair of B fragments and 8 DMMAs per distinct cell of the warp
  double ck[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) ck[t][0] = ck[t][1] = 0.0;
  unsigned todo = __ballot_sync(FULL, inbox);
  const int off0 = 6 * ((j & 1u) + NB * (j >> 1)), off1 = off0 + 6 * NB * NB;
  while (todo) {
    const int cur = __shfl_sync(FULL, cell, __ffs(todo) - 1);
    const unsigned in_cur = __ballot_sync(FULL, cell == cur);
    todo &= ~in_cur;
    const double b0 = gq < 6 ? fld[cur + off0 + gq] : 0.0;
    const double b1 = gq < 6 ? fld[cur + off1 + gq] : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      double c[2] = {0.0, 0.0};
      dmma_884(c, a[t][0], b0);
      dmma_884(c, a[t][1], b1);
      if ((in_cur >> (quad | t)) & 1u) {
        ck[t][0] = c[0];
        ck[t][1] = c[1];
      }
    }
  }
  // in-quad transpose: lane j holds components (2j, 2j+1) of the particles of
  // lanes quad + t; in round r it sends the pair of owner (j + r) & 3 and
  // receives, as owner, the pair computed by lane (j - r) & 3
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const unsigned tsend = (j + (unsigned)r) & 3u;
    double s0 = ck[0][0], s1 = ck[0][1];
    if (tsend == 1u) { s0 = ck[1][0]; s1 = ck[1][1]; }
    if (tsend == 2u) { s0 = ck[2][0]; s1 = ck[2][1]; }
    if (tsend == 3u) { s0 = ck[3][0]; s1 = ck[3][1]; }
    const unsigned src = (j - (unsigned)r) & 3u;
    const double r0 = r == 0 ? s0 : __shfl_sync(FULL, s0, quad | src);
    const double r1 = r == 0 ? s1 : __shfl_sync(FULL, s1, quad | src);
    if (src == 0u) { out[0] = r0; out[1] = r1; }
    if (src == 1u) { out[2] = r0; out[3] = r1; }
    if (src == 2u) { out[4] = r0; out[5] = r1; }
  }
  return inbox;
}

// ----------------------------------------------------------------- mover ----
#ifndef PIC_MOVER_MINB
#define PIC_MOVER_MINB 4
#endif
// NIT > 0: the iteration count is a compile-time constant (fully unrolled);
// NIT == 0: runtime A.n_iter.
#ifndef PIC_MOVER_WARPS
#define PIC_MOVER_WARPS 4
#endif
constexpr int MOVER_WARPS = PIC_MOVER_WARPS;
constexpr int MOVER_THREADS = 32 * MOVER_WARPS;
constexpr size_t MOVER_SMEM = sizeof(double) * (NB3 * 6 + MOVER_WARPS * MOVER_WARP_STAGE) + 16 + 4 * TILE3;

// REL = 1: relativistic Eq. 2 (NEXT-1, readings R4, R5), a separate
// instantiation so the gamma == 1 hot path keeps its registers.
template <int NIT, int REL>
__global__ void __launch_bounds__(MOVER_THREADS, PIC_MOVER_MINB)
    mover_tiled_kernel(const __grid_constant__ CUtensorMap tmap, const MoverTArgs A) {
  constexpr int MW = MOVER_WARPS;
  constexpr int MT = MOVER_THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *fld = reinterpret_cast<double *>(smem_raw);              // staged node box
  double *stage_base = fld + NB3 * 6;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(stage_base + MW * MOVER_WARP_STAGE);
  uint32_t *scnt = reinterpret_cast<uint32_t *>(mbar + 2);          // stayers per cell of the tile
  const Geom &g = A.g;

  const int sp_i = (int)(blockIdx.x / (unsigned)g.ntiles);
  const int tile = (int)(blockIdx.x - (unsigned)sp_i * (unsigned)g.ntiles);
  const MoverSp &S = A.sp[sp_i];
  if (tile == 0 && threadIdx.x == 0) *S.d_nraw = S.cell_off[g.ncells];
  const uint32_t p0 = S.cell_off[(int64_t)tile * TILE3], p1 = S.cell_off[(int64_t)(tile + 1) * TILE3];
  if (p0 == p1) return;
  const int tx = (int)(tile % g.nt[0]);
  const int ty = (int)((tile / g.nt[0]) % g.nt[1]);
  const int tz = (int)(tile / (g.nt[0] * g.nt[1]));
  // global cell (== node) index of the tile origin; box node 0 is origin - 1
  const int64_t ox = g.slab_lo + (int64_t)tx * TILE, oy = (int64_t)ty * TILE, oz = (int64_t)tz * TILE;
  const double bo[3] = {(double)(ox - 1), (double)(oy - 1), (double)(oz - 1)};
  const int tid = threadIdx.x;

  // ---- 1. stage fields with TMA
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  if (tid < TILE3) scnt[tid] = 0u;
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(mbar, NB3 * 6 * 8);
    tma_load_4d(fld, &tmap, 0, (int)(ox - 1 - g.f_lo[0]), (int)(oy - 1 - g.f_lo[1]), (int)(oz - 1 - g.f_lo[2]),
                mbar);
  }
  mbar_wait(mbar, 0);
  for (int nd = tid; nd < NB3; nd += MT) {   // E' = k E, a = k B / c (48 B per node)
    double2 *f2 = reinterpret_cast<double2 *>(fld + 6 * nd);
    double2 e0 = f2[0], e1 = f2[1], e2 = f2[2];
    e0.x *= S.ks; e0.y *= S.ks; e1.x *= S.ks;
    e1.y *= S.ks_c; e2.x *= S.ks_c; e2.y *= S.ks_c;
    f2[0] = e0; f2[1] = e1; f2[2] = e2;
  }
  __syncthreads();

  // ---- 2. warps over contiguous sub-ranges of the tile's particles
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t ntile = p1 - p0;
  const uint32_t chunk = ((ntile + 32 * MW - 1) / (32 * MW)) * 32;
  const uint32_t wbeg = p0 + warp * chunk;
  const uint32_t wend = min(p1, wbeg + chunk);
  const double h[3] = {0.5 * g.dt * g.inv_delta[0], 0.5 * g.dt * g.inv_delta[1], 0.5 * g.dt * g.inv_delta[2]};

  // Software pipeline through shared memory (cp.async / LDGSTS, no register
  // dependencies): in round r the warp gathers the sources of round
  // r+SRC_STAGES-1 into an SRC_STAGES-deep ring and fetches perm of round
  // r+PK_AHEAD into the perm ring, one commit group per round; "wait_group
  // SRC_STAGES-1" then guarantees round r's sources.  The counting-sort rank of
  // a round completes during the next one, so the global atomic's latency
  // overlaps compute.
  double *stg = stage_base + (size_t)warp * MOVER_WARP_STAGE;          // [SRC_STAGES][SRC_STAGED][32] doubles
  uint32_t *pk = reinterpret_cast<uint32_t *>(stg + SRC_STAGES * SRC_RING * 32);  // [PK_SLOTS][64]: perm in [0, 32)
  auto fetch_pk = [&](int ri) {        // perm of round ri
    const uint32_t q = wbeg + 32u * ri + lane;
    if (q < wend) {
      uint32_t *slot = pk + (ri % PK_SLOTS) * 64 + lane;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(slot)), "l"(S.perm + q) : "memory");
    }
  };
  auto fetch_src = [&](int ri) {       // sources of round ri (its perm is already in the ring)
    const uint32_t q = wbeg + 32u * ri + lane;
    if (q < wend) {
      const uint32_t src_idx = pk[(ri % PK_SLOTS) * 64 + lane];
      PIC_DCHECK(src_idx < S.cap, A.stats);
      double *d = stg + (ri % SRC_STAGES) * (SRC_RING * 32) + lane;
#pragma unroll
      for (int k = 0; k < SRC_STAGED; ++k)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(d + k * 32)), "l"(S.src[k] + src_idx)
                     : "memory");
    }
  };
  for (int ri = 0; ri < PK_AHEAD; ++ri) fetch_pk(ri);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  for (int ri = 0; ri < SRC_STAGES - 1; ++ri) {
    fetch_src(ri);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // rank ticket of the previous round: its atomic flies while this round computes
  RankTicket tk;
  tk.base = 0; tk.peers = 0; tk.leader = 0; tk.counted = false; tk.arrival = false;
  uint32_t pr_p = 0;
  int ri = 0;
  for (uint32_t r0 = wbeg; r0 < wend; r0 += 32, ++ri) {
    const uint32_t p = r0 + lane;
    const bool act = p < wend;
    uint32_t kold = 0u;          // the cell of x^n, set below
    fetch_src(ri + SRC_STAGES - 1);
    fetch_pk(ri + PK_AHEAD);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(SRC_STAGES - 1) : "memory");
    const double *sv = stg + (ri % SRC_STAGES) * (SRC_RING * 32) + lane;
    uint32_t knew = KEY_DEAD;
    constexpr bool kMma = PIC_GATHER_MMA && REL == 0;
    // with the tensor-core gather every lane pushes (warp-collective samples):
    // a lane past the end of the range pushes a particle at rest in the tile's
    // first cell and drops the result
    double xnew[3], vnew[3], qv = 0.0;
    int64_t idv = 0;
    if (kMma || act) {
      // q and id only pass through: loaded straight into registers (no
      // shared-memory staging: -0.3 crossbar wavefronts per particle), consumed
      // by the stores at the round's end
      if (act) {
        const uint32_t si = pk[(ri % PK_SLOTS) * 64 + lane];
        qv = __ldg(S.src[6] + si);
        idv = __ldg(S.src_id + si);
      }
      const double xn[3] = {act ? sv[0] : (double)ox + 0.5, act ? sv[32] : (double)oy + 0.5,
                            act ? sv[64] : (double)oz + 0.5};
      const double vn[3] = {act ? sv[96] : 0.0, act ? sv[128] : 0.0, act ? sv[160] : 0.0};
      // the cell of x^n (the key the order was built from: keys are always
      // taken from the stored position, so no key array is kept; a mismatch
      // would only reclassify a stayer as an arrival or back)
      // (this tile's cell: key = tile * 64 + local cell, no division)
      OldCell oc;
      oc.c[0] = (int)xn[0];
      oc.c[1] = (int)xn[1];
      oc.c[2] = (int)xn[2];
      oc.key = (uint32_t)tile * TILE3 +
               (uint32_t)(((oc.c[0] - (int)ox) & 3) + 4 * ((oc.c[1] - (int)oy) & 3) + 16 * ((oc.c[2] - (int)oz) & 3));
      if (act) kold = oc.key;
      // Eq. 2 (push.cuh); field samples from the staged box (tensor-core gather
      // or per-lane loads), the global window (clamped to it, R11) for iterates
      // outside the box
      auto sample = [&](const double xb[3], double EB[6]) -> bool {
        const double u[3] = {xb[0] - bo[0], xb[1] - bo[1], xb[2] - bo[2]};
        if constexpr (kMma) {
          if (gather_mma(fld, u, EB)) return false;
        } else {
          if (gather_smem(fld, u, EB)) return false;
        }
        return WindowSampler{&g, A.field, S.ks, S.ks_c}(xb, EB);
      };
      const bool clamped = push_eq2<NIT, REL>(xn, vn, h, g.c, A.n_iter, sample, xnew, vnew);
      if (act) knew = finish_particle(g, xnew, vnew, clamped, A.stats, &oc);
    }
    // complete the previous round's rank, then start this round's (order.cu);
    // leavers and removed particles are not counted.  The rank atomic is
    // issued before the result stores so that it does not queue behind them
    // (measured: mover -1.5 %).
    if (r0 != wbeg) {
      const uint32_t r = count_rank_finish(tk);
      if (tk.counted) S.rank[pr_p] = r;
    }
    tk = count_rank_issue(scnt, (uint32_t)tile * TILE3, S.cell_count, g.ncells, knew,
                          act && knew < KEY_FIRST_RESERVED, knew != kold);
    pr_p = p;
    if (act) {
      PIC_DCHECK(p < S.cap && (knew < g.ncells || knew >= KEY_FIRST_RESERVED), A.stats);
      S.dst[0][p] = xnew[0]; S.dst[1][p] = xnew[1]; S.dst[2][p] = xnew[2];
      S.dst[3][p] = vnew[0]; S.dst[4][p] = vnew[1]; S.dst[5][p] = vnew[2];
      S.dst[6][p] = qv;
      S.dst_id[p] = idv;
      S.key_new[p] = knew;
    }
    if (A.peer && __any_sync(0xffffffffu, knew == KEY_LEFT || knew == KEY_RIGHT))
      send_leavers_peer(S.po, knew, S.dst, S.dst_id, p, A.stats);
  }
  if (wbeg < wend) {
    const uint32_t r = count_rank_finish(tk);
    if (tk.counted) S.rank[pr_p] = r;
  }
  // the tile's stayer counts (no other CTA counts stayers of these cells)
  __syncthreads();
  if (tid < TILE3) S.cell_count[(int64_t)tile * TILE3 + tid] = scnt[tid];
}

// --------------------------------------------------------------- deposit ----
// word offset of column k (0..7) of row p in a swizzled 8-double staging row
__device__ __forceinline__ int stage_slot(int p, int k) {
  const int h = ((p >> 2) & 1) | (((p >> 1) & 1) << 1);
  return p * 8 + ((((k >> 1) ^ h) << 1) | (k & 1));
}

__global__ void __launch_bounds__(DTHREADS, PIC_DEP_MINB) deposit_tiled_kernel(const DepositArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *nacc = reinterpret_cast<double *>(smem_raw);  // node sums of the tile box [MB^3][10]
  double *wbuf = nacc + MB3 * 10;
  const Geom &g = A.g;
  const int sp_i = (int)(blockIdx.x / (unsigned)g.ntiles);
  const int tile = (int)(blockIdx.x - (unsigned)sp_i * (unsigned)g.ntiles);
  const DepositSp &S = A.sp[sp_i];
  const uint32_t *coff = S.cell_off + (int64_t)tile * TILE3;   // 65 offsets of this tile's cells
  const uint32_t p0 = coff[0], p1 = coff[TILE3];
  if (p0 == p1) return;
  const int tx = (int)(tile % g.nt[0]);
  const int ty = (int)((tile / g.nt[0]) % g.nt[1]);
  const int tz = (int)(tile / (g.nt[0] * g.nt[1]));
  const int64_t ox = g.slab_lo + (int64_t)tx * TILE, oy = (int64_t)ty * TILE, oz = (int64_t)tz * TILE;
  const int tid = threadIdx.x;
  for (int i = tid; i < MB3 * 10; i += DTHREADS) nacc[i] = 0.0;
  __syncthreads();

  // warp ranges are aligned to cell boundaries, so every cell belongs to one
  // warp and its corner sums are stored without atomics
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t ntile = p1 - p0;
  int cbeg = 0, cend = 0;
  {
    const uint32_t t0 = p0 + (uint32_t)(((uint64_t)ntile * warp) / DWARPS);
    const uint32_t t1 = p0 + (uint32_t)(((uint64_t)ntile * (warp + 1)) / DWARPS);
    // first cell starting at or after the target (lane-parallel search over 64 cells)
    const uint32_t o0 = coff[lane], o1 = coff[lane + 32];
    const unsigned b0a = __ballot_sync(0xffffffffu, o0 >= t0), b0b = __ballot_sync(0xffffffffu, o1 >= t0);
    const unsigned b1a = __ballot_sync(0xffffffffu, o0 >= t1), b1b = __ballot_sync(0xffffffffu, o1 >= t1);
    cbeg = b0a ? __ffs(b0a) - 1 : (b0b ? 32 + __ffs(b0b) - 1 : TILE3);
    cend = b1a ? __ffs(b1a) - 1 : (b1b ? 32 + __ffs(b1b) - 1 : TILE3);
    if (warp == DWARPS - 1) cend = TILE3;
    if (warp == 0) cbeg = 0;
  }
  const uint32_t wbeg = coff[cbeg];
  const uint32_t wend = coff[cend];
  double *Ss = wbuf + warp * WBUF;       // [32][8] swizzled
  double *Vs = Ss + 32 * 8;              // [32][8] swizzled, moments 0..7
  double *V2 = Vs + 32 * 8;              // [32][2], moments 8, 9
  // Per cell, the corner sums are a matrix product over its particles:
  //   M[corner][moment] = sum_p S[p][corner] V[p][moment]      (Eq. 3)
  // done on the fp64 tensor cores with mma.m8n8k4 (M = 8 corners, K = 4
  // particles per step, N = 8 + 8 moments, the second tile using 2 columns).
  // Fragments: lane (g = lane / 4, j = lane % 4) supplies A[g][j] = S[4t+j][g],
  // B[j][g] = V[4t+j][g] (and V2[4t+j][g]) and holds C[g][2j], C[g][2j+1].
  // Step t accumulates into set t % NACC, so consecutive MMAs are independent.
  const int g8 = lane >> 2, j4 = lane & 3;
  // lane-constant staging offsets: row writes (column pairs 0..3 of row lane)
  // and fragment reads (row 4t + j4, column g8: even / odd t)
  int wslot[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) wslot[k] = stage_slot(lane, 2 * k);
  const int rs0 = stage_slot(j4, g8), rs1 = stage_slot(4 + j4, g8) - 32;
  const int v2off = 2 * j4 + (g8 & 1);
  double c0[NACC][2], c1[NACC][2];
#pragma unroll
  for (int a = 0; a < NACC; ++a) c0[a][0] = c0[a][1] = c1[a][0] = c1[a][1] = 0.0;
  int cur = -1;  // local cell (0..63) of the accumulators, warp-uniform

  auto flush = [&](int c) {
#pragma unroll
    for (int a = 1; a < NACC; ++a) {
      c0[0][0] += c0[a][0]; c0[0][1] += c0[a][1];
      c1[0][0] += c1[a][0]; c1[0][1] += c1[a][1];
    }
    // corner g8 of cell c is node (cx + gx, cy + gy, cz + gz) of the tile box;
    // cells of different warps share nodes, hence shared-memory atomics (one
    // flush per cell and warp: rare next to the per-particle work)
    const int node = ((c & 3) + (g8 & 1)) + MB * ((((c >> 2) & 3) + ((g8 >> 1) & 1)) + MB * ((c >> 4) + (g8 >> 2)));
    PIC_DCHECK(c >= 0 && c < TILE3 && node < MB3, A.stats);
    double *dst = nacc + node * 10;
    atomicAdd(dst + 2 * j4, c0[0][0]);
    atomicAdd(dst + 2 * j4 + 1, c0[0][1]);
    if (j4 == 0) {
      atomicAdd(dst + 8, c1[0][0]);
      atomicAdd(dst + 9, c1[0][1]);
    }
#pragma unroll
    for (int a = 0; a < NACC; ++a) c0[a][0] = c0[a][1] = c1[a][0] = c1[a][1] = 0.0;
  };
  auto mma = [](double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
  };

  // two-stage software pipeline: the sources of round r+1 and the perm of
  // round r+2 are in flight while round r is reduced.  Lanes past the end load
  // position 0 (always valid) and get q = 0 below, so the loads need no predicate.
  uint32_t p_nx = 0, p_n2 = 0;
  double s_nx[7];
  {
    const uint32_t p = wbeg + lane;
    if (p < wend) p_nx = S.perm[p];
    if (p + 32 < wend) p_n2 = S.perm[p + 32];
#pragma unroll
    for (int k = 0; k < 7; ++k) s_nx[k] = S.src[k][p_nx];
  }
  for (uint32_t r0 = wbeg; r0 < wend; r0 += 32) {
    const uint32_t p = r0 + lane;
    const bool act = p < wend;
    double s_cur[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) s_cur[k] = s_nx[k];
    // advance the pipeline
    p_nx = p_n2;
    PIC_DCHECK(p_nx < S.cap, A.stats);
#pragma unroll
    for (int k = 0; k < 7; ++k) s_nx[k] = S.src[k][p_nx];
    p_n2 = (p + 64 < wend) ? S.perm[p + 64] : 0u;
    // inactive lanes carry zeros (q = 0: every value is 0, the weights finite)
    // the particle's cell in the tile, from its position (the order's cell:
    // keys are taken from positions; clamped to the tile, where a cell one off
    // still gives the same weights, f = 0 or 1)
    int c = 64;   // 64: sentinel, no particle
    if (act) {
      const int lx = min(max((int)s_cur[0] - (int)ox, 0), TILE - 1);
      const int ly = min(max((int)s_cur[1] - (int)oy, 0), TILE - 1);
      const int lz = min(max((int)s_cur[2] - (int)oz, 0), TILE - 1);
      c = lx + TILE * (ly + TILE * lz);
    }
    double Sk[8], val[10];
    {
      const double x = s_cur[0], y = s_cur[1], z = s_cur[2];
      const double u = s_cur[3], v = s_cur[4], w = s_cur[5], q = act ? s_cur[6] : 0.0;
      // values q {1, v, vv} (Eq. 3, R16 order)
      const double qu = q * u, qv = q * v, qw = q * w;
      val[0] = q; val[1] = qu; val[2] = qv; val[3] = qw;
      val[4] = qu * u; val[5] = qu * v; val[6] = qu * w;
      val[7] = qv * v; val[8] = qv * w; val[9] = qw * w;
      // trilinear corner weights inside the particle's cell (R12); the cell is
      // the one of the order (c), relative to the tile origin
      const double fx = x - (double)(ox + (c & 3));
      const double fy = y - (double)(oy + ((c >> 2) & 3));
      const double fz = z - (double)(oz + (c >> 4));
      const double gx = 1.0 - fx, gy = 1.0 - fy, gz = 1.0 - fz;
      const double w00 = gy * gz, w10 = fy * gz, w01 = gy * fz, w11 = fy * fz;
      Sk[0] = gx * w00; Sk[1] = fx * w00; Sk[2] = gx * w10; Sk[3] = fx * w10;
      Sk[4] = gx * w01; Sk[5] = fx * w01; Sk[6] = gx * w11; Sk[7] = fx * w11;
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const int o = wslot[k >> 1];
      *reinterpret_cast<double2 *>(Ss + o) = make_double2(Sk[k], Sk[k + 1]);
      *reinterpret_cast<double2 *>(Vs + o) = make_double2(val[k], val[k + 1]);
    }
    *reinterpret_cast<double2 *>(V2 + 2 * lane) = make_double2(val[8], val[9]);
    __syncwarp();
    // runs of equal cells in the round (the order is sorted, so a round holds
    // a few contiguous runs); each run accumulates into the fragments of its
    // cell, which are flushed when the cell changes
    const unsigned navail = min(32u, wend - r0);
    const int cprev = __shfl_up_sync(0xffffffffu, c, 1);
    unsigned starts = __ballot_sync(0xffffffffu, (unsigned)lane < navail && (lane == 0 || c != cprev));
    while (starts) {
      const int b = __ffs(starts) - 1;
      starts &= starts - 1;
      const int e = starts ? __ffs(starts) - 1 : (int)navail;
      const int rc = __shfl_sync(0xffffffffu, c, b);
      if (rc != cur) {
        if (cur >= 0) flush(cur);
        cur = rc;
      }
      if (b == 0 && e == 32) {
        // the round is one cell: 8 steps, no masking
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int o = 32 * t + ((t & 1) ? rs1 : rs0);
          mma(c0[t % NACC], Ss[o], Vs[o]);
          mma(c1[t % NACC], Ss[o], V2[8 * t + v2off]);
        }
      } else {
        // steps overlapping the run [b, e), particles outside it masked
        for (int t = b >> 2; 4 * t < e; ++t) {
          const int pi = 4 * t + j4;
          const int o = 32 * t + ((t & 1) ? rs1 : rs0);
          const double a = (pi >= b && pi < e) ? Ss[o] : 0.0;
          mma(c0[0], a, Vs[o]);
          mma(c1[0], a, V2[8 * t + v2off]);
        }
      }
    }
    __syncwarp();
  }
  if (cur >= 0) flush(cur);
  __syncthreads();

  // node sums of the tile -> global moments; one (node, moment) pair per
  // thread.  Nodes on the tile's faces are shared with neighbour tiles
  // (atomics); the 3^3 interior nodes belong to this tile's cells only, so a
  // plain store into the zeroed array suffices.
  for (int i = tid; i < MB3 * 10; i += DTHREADS) {
    const int n = i / 10, m = i - 10 * n;
    const int bx = n % MB, by = (n / MB) % MB, bz = n / (MB * MB);
    const double v = nacc[i];
    if (v == 0.0) continue;
    const int64_t node = moment_node(g, ox + bx, oy + by, oz + bz);
    if (node < 0) {
      if (m == 0) atomicAdd(&A.stats[ST_FAR], 1ull);
      continue;
    }
    const bool interior = bx > 0 && bx < TILE && by > 0 && by < TILE && bz > 0 && bz < TILE;
    if (interior)
      S.mom[m * g.m_plane + node] = v;
    else
      atomicAdd(S.mom + m * g.m_plane + node, v);
  }
}

// ------------------------------------------------------------------- host --
static pic_status make_tmap(Ctx *ctx) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
      return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const Geom &g = ctx->geom;
  cuuint64_t dims[4] = {6, (cuuint64_t)g.f_n[0], (cuuint64_t)g.f_n[1], (cuuint64_t)g.f_n[2]};
  cuuint64_t strides[3] = {48, (cuuint64_t)(48 * g.f_n[0]), (cuuint64_t)(48 * g.f_n[0] * g.f_n[1])};
  cuuint32_t box[4] = {6, NB, NB, NB};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int b = 0; b < 2; ++b) {   // one map per field buffer
    CUtensorMap *map = reinterpret_cast<CUtensorMap *>(ctx->tmap[b]);
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)ctx->field_buf[b], dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled failed");
  }
#define PIC_SET_SMEM(NIT) \
  PIC_CUDA(cudaFuncSetAttribute(mover_tiled_kernel<NIT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MOVER_SMEM)); \
  PIC_CUDA(cudaFuncSetAttribute(mover_tiled_kernel<NIT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MOVER_SMEM))
  PIC_SET_SMEM(0); PIC_SET_SMEM(1); PIC_SET_SMEM(2); PIC_SET_SMEM(3); PIC_SET_SMEM(4);
#undef PIC_SET_SMEM
  PIC_CUDA(cudaFuncSetAttribute(deposit_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)DEPOSIT_SMEM));
  ctx->tmap_ok = true;
  return PIC_OK;
}

// pic_mover, tiled family: move species [s0, s1) (one launch, species-major
// blocks) through the current order into buffer B, rank the new keys and swap
// buffers; pic_mover then migrates slab leavers (multi-rank) and builds the
// next order (order.cu).  The species of one launch share n_iter.
pic_status launch_tiled_step(Ctx *ctx, int s0, int s1) {
  if (!ctx->tmap_ok) {
    pic_status st = make_tmap(ctx);
    if (st != PIC_OK) return st;
  }
  MoverTArgs A;
  A.g = ctx->geom;
  for (int s = s0; s < s1; ++s) {
    SpeciesStore &sp = ctx->sp[s];
    pic_status st = zero_cell_counts(ctx, s);
    if (st != PIC_OK) return st;
    MoverSp &S = A.sp[s - s0];
    for (int k = 0; k < 7; ++k) { S.src[k] = sp.a[k]; S.dst[k] = sp.b[k]; }
    S.src_id = sp.id;
    S.dst_id = sp.id_b;
    S.perm = sp.perm;
    S.cell_off = sp.cell_off;
    S.key_new = sp.key_new;
    S.rank = sp.rank;
    S.cell_count = sp.cell_count;
    S.d_nraw = sp.d_nraw;
    S.ks = sp.qom * (ctx->geom.dt * 0.5);
    S.ks_c = S.ks / ctx->geom.c;
    S.po = ctx->peer ? peer_out(ctx, s) : PeerOut{};
    S.cap = sp.cap;
    if (sp.n_iter != ctx->sp[s0].n_iter) return fail(ctx, PIC_EINVAL, "one mover launch needs one n_iter");
  }
  A.field = ctx->field();
  A.stats = ctx->stats;
  A.n_iter = ctx->sp[s0].n_iter;
  A.peer = ctx->peer;
  const CUtensorMap &tm = *reinterpret_cast<const CUtensorMap *>(ctx->tmap[ctx->field_cur]);
  const unsigned grid = (unsigned)(ctx->geom.ntiles * (s1 - s0));
#define PIC_LAUNCH(NIT)                                                                            \
  do {                                                                                             \
    if (ctx->cfg.relativistic)                                                                     \
      mover_tiled_kernel<NIT, 1><<<grid, MOVER_THREADS, MOVER_SMEM, ctx->stream>>>(tm, A);         \
    else                                                                                           \
      mover_tiled_kernel<NIT, 0><<<grid, MOVER_THREADS, MOVER_SMEM, ctx->stream>>>(tm, A);         \
  } while (0)
  {
    PhaseTimer t(ctx, 0);
    switch (A.n_iter) {
      case 1: PIC_LAUNCH(1); break;
      case 2: PIC_LAUNCH(2); break;
      case 3: PIC_LAUNCH(3); break;
      case 4: PIC_LAUNCH(4); break;
      default: PIC_LAUNCH(0); break;
    }
  }
#undef PIC_LAUNCH
  ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  for (int s = s0; s < s1; ++s) ctx->sp[s].swap_buffers();
  return PIC_OK;
}

// pic_moments, tiled family: deposit species [s0, s1) (one launch) over the new
// order (requires the order built by pic_mover after migration, so arrivals are
// included and leavers are deposited by their new owner only).
pic_status launch_tiled_deposit(Ctx *ctx, int s0, int s1) {
  if (!ctx->tmap_ok) {
    pic_status st = make_tmap(ctx);
    if (st != PIC_OK) return st;
  }
  DepositArgs A;
  A.g = ctx->geom;
  for (int s = s0; s < s1; ++s) {
    SpeciesStore &sp = ctx->sp[s];
    pic_status st = zero_moments(ctx, s);
    if (st != PIC_OK) return st;
    DepositSp &S = A.sp[s - s0];
    for (int k = 0; k < 7; ++k) S.src[k] = sp.a[k];
    S.perm = sp.perm;
    S.cell_off = sp.cell_off;
    S.mom = sp.mom;
    S.cap = sp.cap;
  }
  A.stats = ctx->stats;
  deposit_tiled_kernel<<<(unsigned)(ctx->geom.ntiles * (s1 - s0)), DTHREADS, DEPOSIT_SMEM, ctx->stream>>>(A);
  ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

}  // namespace pic
