// tiled.cu — PIC_KERNEL_TILED: cell-sorted, tile-staged, fused mover + deposit.
//
// One CTA per tile of TILE^3 cells (the store is sorted tile-major, sort.cu):
//
//  1. TMA (cp.async.bulk.tensor.4d, mbarrier) stages the E,B nodes of the tile
//     plus a one-cell halo, 7^3 nodes x 48 B, from the field window into shared
//     memory; the CTA pre-scales them by k_s = (q/m) dt/2 and k_s / c so the
//     mover reads E' = k_s E and a = k_s B / c directly (Eq. 2, R7, R8).
//  2. Warps split the tile's particle range evenly.  Rounds of 32 consecutive
//     particles (lane = particle, coalesced SoA loads): n_iter predictor-
//     corrector iterations of Eq. 2 (R1, R2) with trilinear gathers from shared
//     memory (R12), then x^{n+1}, v^{n+1}, boundary conditions and the new
//     sort key (R10, R11, R21).
//  3. The deposit of the new state (Eq. 3, R13-R18) is fused: each lane turns
//     its particle into the 8 trilinear corner weights of its new cell c1 and
//     the 10 values q{1, v, vv}, written to a per-warp shared buffer; the warp
//     re-reads them as 8 corners x 4 particle slots.
//     Pass A (particles still in their sort-time cell c0, the vast majority):
//     each lane accumulates 10 register sums for one corner node of c0 across
//     rounds (no atomics inside a cell); when c0 changes the four slots are
//     reduced with shuffles and added to the tile's shared node accumulators
//     (7^3 nodes x 10).  Pass B (cell crossers, c1 != c0): 4 crossers per step,
//     one corner node per lane, added with shared-memory atomics.
//  4. The tile's shared accumulators are added to the global ghosted moment
//     arrays with fp64 atomics (tile faces are shared with neighbour tiles).
//
// Sample points or deposit nodes outside the staged 7^3 box fall back to the
// global field window / global atomics (counted in stats only when beyond the
// rank's ghost reach).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "pic_internal.cuh"

namespace pic {

constexpr int NB = TILE + 3;            // staged nodes per axis: -1 .. TILE+1
constexpr int NB3 = NB * NB * NB;       // 343
constexpr int WARPS = 8;
constexpr int THREADS = 32 * WARPS;
constexpr int SGRP = 36;                // doubles per 4-particle group in the S buffer (32 + pad)
constexpr int WBUF = 8 * SGRP + 32 * 10 + 16;  // doubles per warp: S[8][36] + V[32][10] + 32 ints
constexpr size_t SMEM_BYTES = sizeof(double) * (NB3 * 6 + 10 * NB3 + WARPS * WBUF) + 16;

struct TiledArgs {
  Geom g;
  const double *src[7];       // buffer A (read through perm)
  const int64_t *src_id;
  double *dst[7];             // buffer B (written in cell order)
  int64_t *dst_id;
  const uint32_t *perm;       // q -> A-position
  const uint32_t *key;        // key[q]: sort-time key (cell c0 of x^n)
  const uint32_t *cell_off;   // tile t covers q in [cell_off[64 t], cell_off[64 (t+1)])
  uint32_t *key_new, *rank, *cell_count;
  int64_t *d_nraw;
  const double *field;        // global window (fallback sampling)
  double *mom;                // ghosted moment arrays [10][m_plane]
  unsigned long long *stats;
  double ks, ks_c;
  int n_iter;
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

// 1/D for D >= 1 (D = 1 + |a|^2 of Eq. 2): MUFU.RCP64H seed + two Newton steps
// (error well below 1 ulp of the 1e-12 parity budget; no IEEE slow path).
__device__ __forceinline__ double rcp_ge1(double D) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(D));
  double e = fma(-D, r, 1.0);
  r = fma(r, e, r);
  e = fma(-D, r, 1.0);
  return fma(r, e, r);
}

// N independent fp64 additions into shared memory with compare-and-swap
// (sm_100 has no native shared fp64 add): the N CAS chains are issued together
// so their latencies overlap.  Bit i of `valid` enables entry i.
template <int N>
__device__ __forceinline__ void smem_add_batch(double *const *addr, const double *val, unsigned valid) {
  unsigned long long cur[N];
#pragma unroll
  for (int i = 0; i < N; ++i) cur[i] = ((valid >> i) & 1u) ? *reinterpret_cast<unsigned long long *>(addr[i]) : 0ull;
  while (valid) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((valid >> i) & 1u) {
        const unsigned long long want = __double_as_longlong(__longlong_as_double(cur[i]) + val[i]);
        const unsigned long long got = atomicCAS(reinterpret_cast<unsigned long long *>(addr[i]), cur[i], want);
        if (got == cur[i]) valid &= ~(1u << i);
        else cur[i] = got;
      }
    }
  }
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
  if (!(fl[0] >= 0.0 && fl[0] <= NB - 2 && fl[1] >= 0.0 && fl[1] <= NB - 2 && fl[2] >= 0.0 && fl[2] <= NB - 2))
    return false;
  const double gx0 = 1.0 - f[0], gy0 = 1.0 - f[1], gz0 = 1.0 - f[2];
  const double w00 = gy0 * gz0, w10 = f[1] * gz0, w01 = gy0 * f[2], w11 = f[1] * f[2];
  const double S[8] = {gx0 * w00, f[0] * w00, gx0 * w10, f[0] * w10,
                       gx0 * w01, f[0] * w01, gx0 * w11, f[0] * w11};
#pragma unroll
  for (int m = 0; m < 6; ++m) out[m] = 0.0;
  const int base = ((i[2] * NB + i[1]) * NB + i[0]) * 6;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int off = base + 6 * ((c & 1) + NB * ((c >> 1) & 1) + NB * NB * (c >> 2));
    const double2 a = *reinterpret_cast<const double2 *>(fld + off);
    const double2 b = *reinterpret_cast<const double2 *>(fld + off + 2);
    const double2 e = *reinterpret_cast<const double2 *>(fld + off + 4);
    out[0] = fma(S[c], a.x, out[0]);
    out[1] = fma(S[c], a.y, out[1]);
    out[2] = fma(S[c], b.x, out[2]);
    out[3] = fma(S[c], b.y, out[3]);
    out[4] = fma(S[c], e.x, out[4]);
    out[5] = fma(S[c], e.y, out[5]);
  }
  return true;
}

__global__ void __launch_bounds__(THREADS, 2) tiled_kernel(const __grid_constant__ CUtensorMap tmap,
                                                           const TiledArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *fld = reinterpret_cast<double *>(smem_raw);
  double *acc = fld + NB3 * 6;
  double *wbuf = acc + 10 * NB3;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(wbuf + WARPS * WBUF);
  const Geom &g = A.g;

  const int tile = blockIdx.x;
  if (tile == 0 && threadIdx.x == 0) *A.d_nraw = A.cell_off[g.ncells];
  const uint32_t p0 = A.cell_off[(int64_t)tile * TILE3], p1 = A.cell_off[(int64_t)(tile + 1) * TILE3];
  if (p0 == p1) return;
  const int tx = (int)(tile % g.nt[0]);
  const int ty = (int)((tile / g.nt[0]) % g.nt[1]);
  const int tz = (int)(tile / (g.nt[0] * g.nt[1]));
  // global cell (== node) index of the tile origin; box node 0 is origin - 1
  const int64_t ox = g.slab_lo + (int64_t)tx * TILE, oy = (int64_t)ty * TILE, oz = (int64_t)tz * TILE;
  const double bo[3] = {(double)(ox - 1), (double)(oy - 1), (double)(oz - 1)};
  const int tid = threadIdx.x;

  // ---- 1. stage fields with TMA, zero the accumulators meanwhile
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(mbar, NB3 * 6 * 8);
    tma_load_4d(fld, &tmap, 0, (int)(ox - 1 - g.f_lo[0]), (int)(oy - 1 - g.f_lo[1]), (int)(oz - 1 - g.f_lo[2]),
                mbar);
  }
  for (int i = tid; i < 10 * NB3; i += THREADS) acc[i] = 0.0;
  mbar_wait(mbar, 0);
  for (int i = tid; i < NB3 * 6; i += THREADS) fld[i] *= ((i % 6) < 3) ? A.ks : A.ks_c;
  __syncthreads();

  // ---- 2./3. warps over contiguous sub-ranges of the tile's particles
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t ntile = p1 - p0;
  const uint32_t chunk = ((ntile + 32 * WARPS - 1) / (32 * WARPS)) * 32;
  const uint32_t wbeg = p0 + warp * chunk;
  const uint32_t wend = min(p1, wbeg + chunk);
  double *Sb = wbuf + warp * WBUF;       // [8 groups][36]: S[k][j] at grp*36 + k*4 + j
  double *Vb = Sb + 8 * SGRP;            // [32][10]
  const int kc = lane & 7, js = lane >> 3;
  const int kbx = kc & 1, kby = (kc >> 1) & 1, kbz = kc >> 2;
  const double h[3] = {0.5 * g.dt * g.inv_delta[0], 0.5 * g.dt * g.inv_delta[1], 0.5 * g.dt * g.inv_delta[2]};
  double accr[10];
#pragma unroll
  for (int m = 0; m < 10; ++m) accr[m] = 0.0;
  int cur = -1;  // local cell (0..63) of the register accumulators, warp-uniform

  auto flush = [&](int c) {
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      accr[m] += __shfl_xor_sync(0xffffffffu, accr[m], 8);
      accr[m] += __shfl_xor_sync(0xffffffffu, accr[m], 16);
    }
    const int cx = c & 3, cy = (c >> 2) & 3, cz = c >> 4;
    const int node = ((cz + kbz + 1) * NB + (cy + kby + 1)) * NB + (cx + kbx + 1);
    double *ad[3];
    double vl[3];
    unsigned valid = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int m = js + 4 * i;
      ad[i] = acc + (m < 10 ? m : 0) * NB3 + node;
      double v = 0.0;
#pragma unroll
      for (int mm = 0; mm < 10; ++mm)
        if (mm == m) v = accr[mm];
      vl[i] = v;
      if (m < 10 && v != 0.0) valid |= 1u << i;
    }
    smem_add_batch<3>(ad, vl, valid);
#pragma unroll
    for (int m = 0; m < 10; ++m) accr[m] = 0.0;
  };

  int *cl = reinterpret_cast<int *>(Vb + 32 * 10);  // crosser -> lane table (32 ints)

  for (uint32_t r0 = wbeg; r0 < wend; r0 += 32) {
    const uint32_t p = r0 + lane;
    const bool act = p < wend;
    // prefetch the next round's gathered sources into L1 while this round computes
    if (p + 32 < wend) {
      const uint32_t pn = A.perm[p + 32];
#pragma unroll
      for (int k = 0; k < 7; ++k) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.src[k] + pn));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(A.src_id + pn));
    }
    int c0 = 0;          // sort-time local cell (0..63)
    int c1b = -1;        // new cell in box coordinates (bx + NB (by + NB bz)) of a crosser
    bool alive = false, crosser = false;
    double Sk[8], val[10];
#pragma unroll
    for (int k = 0; k < 8; ++k) Sk[k] = 0.0;
#pragma unroll
    for (int m = 0; m < 10; ++m) val[m] = 0.0;
    uint32_t knew_l = KEY_DEAD;
    if (act) {
      c0 = (int)(A.key[p] & (TILE3 - 1));
      const uint32_t sp_ = A.perm[p];
      const double xn[3] = {A.src[0][sp_], A.src[1][sp_], A.src[2][sp_]};
      const double vn[3] = {A.src[3][sp_], A.src[4][sp_], A.src[5][sp_]};
      const double q = A.src[6][sp_];
      A.dst[6][p] = q;
      A.dst_id[p] = A.src_id[sp_];
      double xb[3] = {xn[0], xn[1], xn[2]};
      double vb[3];
      bool clamped = false;
      for (int it = 0; it < A.n_iter; ++it) {
        double EB[6];
        const double u[3] = {xb[0] - bo[0], xb[1] - bo[1], xb[2] - bo[2]};
        if (!gather_smem(fld, u, EB)) {
          clamped |= sample_window(g, A.field, xb, EB);
#pragma unroll
          for (int m = 0; m < 6; ++m) EB[m] *= (m < 3) ? A.ks : A.ks_c;
        }
        // Eq. 2: vt = vn + k E ; a = k B / c ; vb = (vt + vt x a + (vt.a) a) / (1 + a.a)
        const double vt0 = vn[0] + EB[0], vt1 = vn[1] + EB[1], vt2 = vn[2] + EB[2];
        const double a0 = EB[3], a1 = EB[4], a2 = EB[5];
        const double dot = fma(vt0, a0, fma(vt1, a1, vt2 * a2));
        const double D = fma(a0, a0, fma(a1, a1, fma(a2, a2, 1.0)));
        const double invD = rcp_ge1(D);
        vb[0] = fma(dot, a0, fma(vt1, a2, fma(-vt2, a1, vt0))) * invD;
        vb[1] = fma(dot, a1, fma(vt2, a0, fma(-vt0, a2, vt1))) * invD;
        vb[2] = fma(dot, a2, fma(vt0, a1, fma(-vt1, a0, vt2))) * invD;
#pragma unroll
        for (int d = 0; d < 3; ++d) xb[d] = fma(vb[d], h[d], xn[d]);
      }
      double xnew[3], vnew[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        xnew[d] = fma(vb[d], 2.0 * h[d], xn[d]);
        vnew[d] = fma(2.0, vb[d], -vn[d]);
      }
      const double xdep[3] = {xnew[0], xnew[1], xnew[2]};  // pre-wrap: deposit position
      const uint32_t knew = finish_particle(g, xnew, vnew, clamped, A.stats);
      A.dst[0][p] = xnew[0]; A.dst[1][p] = xnew[1]; A.dst[2][p] = xnew[2];
      A.dst[3][p] = vnew[0]; A.dst[4][p] = vnew[1]; A.dst[5][p] = vnew[2];
      A.key_new[p] = knew;
      knew_l = knew;
      if (knew != KEY_DEAD) {
        alive = true;
        // values q {1, v, vv} (Eq. 3, R16 order)
        const double qu = q * vnew[0], qv = q * vnew[1], qw = q * vnew[2];
        val[0] = q; val[1] = qu; val[2] = qv; val[3] = qw;
        val[4] = qu * vnew[0]; val[5] = qu * vnew[1]; val[6] = qu * vnew[2];
        val[7] = qv * vnew[1]; val[8] = qv * vnew[2]; val[9] = qw * vnew[2];
        // trilinear weights of the 8 corners of the new cell c1 (R12)
        double f[3];
        int64_t c1g[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double fl = floor(xdep[d]);
          f[d] = xdep[d] - fl;
          c1g[d] = (int64_t)fl;
        }
        const double gx = 1.0 - f[0], gy = 1.0 - f[1], gz = 1.0 - f[2];
        const double w00 = gy * gz, w10 = f[1] * gz, w01 = gy * f[2], w11 = f[1] * f[2];
        Sk[0] = gx * w00; Sk[1] = f[0] * w00; Sk[2] = gx * w10; Sk[3] = f[0] * w10;
        Sk[4] = gx * w01; Sk[5] = f[0] * w01; Sk[6] = gx * w11; Sk[7] = f[0] * w11;
        crosser = (c1g[0] != ox + (c0 & 3)) || (c1g[1] != oy + ((c0 >> 2) & 3)) || (c1g[2] != oz + (c0 >> 4));
        if (crosser) {
          const int64_t bx = c1g[0] - ox + 1, by = c1g[1] - oy + 1, bz = c1g[2] - oz + 1;
          c1b = (bx >= 0 && bx <= NB - 2 && by >= 0 && by <= NB - 2 && bz >= 0 && bz <= NB - 2)
                    ? (int)((bz * NB + by) * NB + bx) : -2;   // -2: outside the box
        }
      }
    }
    // rank for the next cell order (order.cu); leavers and removed are not counted
    {
      const bool counted = act && knew_l < KEY_FIRST_RESERVED;
      const uint32_t r = count_rank(A.cell_count, g.ncells, knew_l, counted, !act || knew_l != A.key[p]);
      if (counted) A.rank[p] = r;
    }
    // stage S (corner-major per 4-particle group) and the 10 values, lane order
    {
      const int grp = lane >> 2, j = lane & 3;
#pragma unroll
      for (int k = 0; k < 8; ++k) Sb[grp * SGRP + k * 4 + j] = Sk[k];
#pragma unroll
      for (int m = 0; m < 10; m += 2)
        *reinterpret_cast<double2 *>(Vb + lane * 10 + m) = make_double2(val[m], val[m + 1]);
    }
    const unsigned xmask = __ballot_sync(0xffffffffu, crosser);
    if (crosser) cl[__popc(xmask & ((1u << lane) - 1u))] = lane;
    __syncwarp();

    // ---- pass B: cell crossers, one at a time; lane = (corner kc, value group
    // js) so the 32 lanes add distinct (node, component) pairs: the shared CAS
    // atomics never conflict inside the warp.
    const int ncross = __popc(xmask);
    // crossers outside the staged box (far movers, rare): global atomics
    if (__any_sync(0xffffffffu, crosser && c1b < 0)) {
      for (int r = 0; r < ncross; ++r) {
        const int src = cl[r];
        const int cb = __shfl_sync(0xffffffffu, c1b, src);
        if (cb >= 0) continue;
        // re-derive the (pre-wrap) cell of the crosser from what the mover stored
        const uint32_t qs = r0 + src;
        double xs = A.dst[0][qs];
        const uint32_t ks_ = A.key_new[qs];
        if (ks_ == KEY_LEFT && xs >= (double)g.slab_hi) xs -= (double)g.ncell[0];
        if (ks_ == KEY_RIGHT && xs < (double)g.slab_lo) xs += (double)g.ncell[0];
        if (g.periodic[0] && !g.multi_rank && xs < (double)(ox - 1)) xs += (double)g.ncell[0];
        if (g.periodic[0] && !g.multi_rank && xs >= (double)(ox + TILE + 1)) xs -= (double)g.ncell[0];
        const int64_t gx = (int64_t)floor(xs);
        const int64_t gy = (int64_t)floor(A.dst[1][qs]);
        const int64_t gz = (int64_t)floor(A.dst[2][qs]);
        const double s = Sb[(src >> 2) * SGRP + kc * 4 + (src & 3)];
        const double *vv = Vb + src * 10;
        const int64_t node = moment_node(g, gx + kbx, gy + kby, gz + kbz);
        if (node < 0) {
          if (js == 0 && s != 0.0) atomicAdd(&A.stats[ST_FAR], 1ull);
        } else {
          for (int m = js; m < 10; m += 4) atomicAdd(A.mom + m * g.m_plane + node, s * vv[m]);
        }
      }
    }
    // two crossers per step: up to 6 independent shared CAS chains per lane
    for (int r = 0; r < ncross; r += 2) {
      double *ad[6];
      double vl[6];
      unsigned valid = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (r + t < ncross) {
          const int src = cl[r + t];
          const int cb = __shfl_sync(0xffffffffu, c1b, src);
          const double s = Sb[(src >> 2) * SGRP + kc * 4 + (src & 3)];
          const double *vv = Vb + src * 10;
          const int node = cb + kbx + NB * (kby + NB * kbz);
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int m = js + 4 * i;
            ad[3 * t + i] = acc + m * NB3 + node;
            vl[3 * t + i] = (m < 10) ? s * vv[m] : 0.0;
            if (cb >= 0 && m < 10) valid |= 1u << (3 * t + i);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 3; ++i) { ad[3 * t + i] = acc; vl[3 * t + i] = 0.0; }
        }
      }
      smem_add_batch<6>(ad, vl, valid);
    }

    // ---- pass A: particles still in their sort-time cell, register accumulation
    const unsigned amask = __ballot_sync(0xffffffffu, alive && !crosser);
    if (amask) {
      const bool uniform = __all_sync(0xffffffffu, !(alive && !crosser) || c0 == cur);
      if (uniform) {
        // fast path: every pass-A particle of the round is in the current cell
        for (int grp = 0; grp < 8; ++grp) {
          if (((amask >> (grp * 4)) & 0xFu) == 0u) continue;
          const bool mine = (amask >> (grp * 4 + js)) & 1u;
          const double s = mine ? Sb[grp * SGRP + kc * 4 + js] : 0.0;
          const double *vv = Vb + (grp * 4 + js) * 10;
#pragma unroll
          for (int m = 0; m < 10; m += 2) {
            const double2 t = *reinterpret_cast<const double2 *>(vv + m);
            accr[m] = fma(s, t.x, accr[m]);
            accr[m + 1] = fma(s, t.y, accr[m + 1]);
          }
        }
      } else {
        const int ca = (alive && !crosser) ? c0 : 64;
        for (int grp = 0; grp < 8; ++grp) {
          if (((amask >> (grp * 4)) & 0xFu) == 0u) continue;
          const int cj = __shfl_sync(0xffffffffu, ca, grp * 4 + js);
          int v = (int)__reduce_min_sync(0xffffffffu, (unsigned)cj);
          const double s = Sb[grp * SGRP + kc * 4 + js];
          const double *vv = Vb + (grp * 4 + js) * 10;
          double vals[10];
#pragma unroll
          for (int m = 0; m < 10; m += 2) {
            const double2 t = *reinterpret_cast<const double2 *>(vv + m);
            vals[m] = t.x;
            vals[m + 1] = t.y;
          }
          while (v < 64) {
            if (v != cur) {
              if (cur >= 0) flush(cur);
              cur = v;
            }
            const double sw = (cj == v) ? s : 0.0;
#pragma unroll
            for (int m = 0; m < 10; ++m) accr[m] = fma(sw, vals[m], accr[m]);
            v = (int)__reduce_min_sync(0xffffffffu, (unsigned)(cj > v ? cj : 64));
          }
        }
      }
    }
    __syncwarp();
  }
  if (cur >= 0) flush(cur);
  __syncthreads();

  // ---- 4. tile accumulators -> global moments
  for (int i = tid; i < NB3; i += THREADS) {
    const int bx = i % NB, by = (i / NB) % NB, bz = i / (NB * NB);
    double vsum = 0.0;
#pragma unroll
    for (int m = 0; m < 10; ++m) vsum += fabs(acc[m * NB3 + i]);
    if (vsum == 0.0) continue;
    const int64_t node = moment_node(g, ox - 1 + bx, oy - 1 + by, oz - 1 + bz);
    if (node < 0) {
      atomicAdd(&A.stats[ST_FAR], 1ull);
      continue;
    }
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      const double a = acc[m * NB3 + i];
      if (a != 0.0) atomicAdd(A.mom + m * g.m_plane + node, a);
    }
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
  CUtensorMap *map = reinterpret_cast<CUtensorMap *>(ctx->tmap);
  cuuint64_t dims[4] = {6, (cuuint64_t)g.f_n[0], (cuuint64_t)g.f_n[1], (cuuint64_t)g.f_n[2]};
  cuuint64_t strides[3] = {48, (cuuint64_t)(48 * g.f_n[0]), (cuuint64_t)(48 * g.f_n[0] * g.f_n[1])};
  cuuint32_t box[4] = {6, NB, NB, NB};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)ctx->field, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, PIC_ECUDA, "cuTensorMapEncodeTiled failed");
  ctx->tmap_ok = true;
  return PIC_OK;
}

pic_status launch_tiled_step(Ctx *ctx, int s, bool *did_deposit) {
  *did_deposit = false;
  SpeciesStore &sp = ctx->sp[s];
  if (!ctx->tmap_ok) {
    pic_status st = make_tmap(ctx);
    if (st != PIC_OK) return st;
    PIC_CUDA(cudaFuncSetAttribute(tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
  }
  pic_status st = zero_moments(ctx, s);
  if (st != PIC_OK) return st;
  st = zero_cell_counts(ctx, s);
  if (st != PIC_OK) return st;
  TiledArgs A;
  A.g = ctx->geom;
  for (int k = 0; k < 7; ++k) { A.src[k] = sp.a[k]; A.dst[k] = sp.b[k]; }
  A.src_id = sp.id;
  A.dst_id = sp.id_b;
  A.perm = sp.perm;
  A.key = sp.key;
  A.cell_off = sp.cell_off;
  A.key_new = sp.key_new;
  A.rank = sp.rank;
  A.cell_count = sp.cell_count;
  A.d_nraw = sp.d_nraw;
  A.field = ctx->field;
  A.mom = sp.mom;
  A.stats = ctx->stats;
  A.ks = sp.qom * (ctx->geom.dt * 0.5);
  A.ks_c = A.ks / ctx->geom.c;
  A.n_iter = sp.n_iter;
  tiled_kernel<<<(unsigned)ctx->geom.ntiles, THREADS, SMEM_BYTES, ctx->stream>>>(
      *reinterpret_cast<const CUtensorMap *>(ctx->tmap), A); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  sp.swap_buffers();
  sp.order_valid = false;
  *did_deposit = true;
  return PIC_OK;
}

}  // namespace pic
