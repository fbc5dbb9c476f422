// inject.cu — NEXT-3: inflow injection at the open x = 0 face (PAPER.md:
// 232-233, "wind electrons and protons are injected with a prescribed bulk
// velocity"; reading R28).
//
// One thread per ghost particle: Philox4x32-10 draws (the counter-based
// generator the oracle implements too), a uniform position in ghost cell
// (-1, cy, cz), a drifting Maxwellian velocity (Box-Muller), one Eq. 2 push
// through the global field window, and — if the particle ended inside the
// domain — an append to the store with its cell ranked as an arrival, so the
// order built next by pic_mover includes it.  Ghost particles that did not
// cross the face are dropped (they were never part of the plasma).
#include "pic_internal.cuh"
#include "push.cuh"

namespace pic {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

struct InjectArgs {
  Geom g;
  double *dst[7];
  int64_t *dst_id;
  uint32_t *key_new, *rank, *cell_count;
  int64_t *d_nraw;
  int64_t cap;
  const double *F;
  unsigned long long *stats;
  double ks, ks_c;
  int n_iter, rel, species, ppc;
  uint32_t seed_lo, seed_hi, cycle;
  double vth, drift[3], q;
};

__global__ void __launch_bounds__(256) inject_kernel(const InjectArgs A) {
  const Geom &g = A.g;
  const int64_t total = g.ncell[1] * g.ncell[2] * (int64_t)A.ppc;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((int64_t)blockIdx.x * blockDim.x >= total) return;   // whole warps leave together
  const bool act = t < total;
  uint32_t k = KEY_DEAD;
  int64_t slot = -1;
  double xnew[3] = {0, 0, 0}, vnew[3] = {0, 0, 0};
  uint64_t idv = 0;
  if (act) {
    const uint32_t gc = (uint32_t)(t / A.ppc), kk = (uint32_t)(t % A.ppc);
    const int64_t cy = gc % g.ncell[1], cz = gc / g.ncell[1];
    double r[8];
#pragma unroll
    for (int call = 0; call < 4; ++call) {
      uint32_t c[4] = {gc, kk, A.cycle, ((uint32_t)A.species << 8) | (uint32_t)call};
      philox4x32_10(c, A.seed_lo, A.seed_hi);
      r[2 * call] = u53(c[0], c[1]);
      r[2 * call + 1] = u53(c[2], c[3]);
    }
    const double two_pi = 2.0 * 3.14159265358979323846;
    // positions in cell units (the store's units): ghost cell (-1, cy, cz)
    const double xn[3] = {-1.0 + r[0], (double)cy + r[1], (double)cz + r[2]};
    const double rad1 = sqrt(-2.0 * log(1.0 - r[3]));
    const double rad2 = sqrt(-2.0 * log(1.0 - r[5]));
    const double vn[3] = {A.drift[0] + A.vth * (rad1 * cos(two_pi * r[4])),
                          A.drift[1] + A.vth * (rad1 * sin(two_pi * r[4])),
                          A.drift[2] + A.vth * (rad2 * cos(two_pi * r[6]))};
    const double h[3] = {0.5 * g.dt * g.inv_delta[0], 0.5 * g.dt * g.inv_delta[1], 0.5 * g.dt * g.inv_delta[2]};
    // Eq. 2 (push.cuh) with samples from the global field window
    const WindowSampler sample{&g, A.F, A.ks, A.ks_c};
    const bool clamped = A.rel ? push_eq2<0, 1>(xn, vn, h, g.c, A.n_iter, sample, xnew, vnew)
                               : push_eq2<0, 0>(xn, vn, h, g.c, A.n_iter, sample, xnew, vnew);
    // only particles that crossed the face join the plasma; the others are
    // dropped without counting (R28).  NaN fails the test and is caught below.
    if (!(xnew[0] < 0.0)) {
      k = finish_particle(g, xnew, vnew, clamped, A.stats);
      if (k == KEY_LEFT || k == KEY_RIGHT) {   // crossed the whole first slab in one step
        atomicAdd(&A.stats[ST_FAR], 1ull);
        k = KEY_DEAD;
      }
      if (k < KEY_FIRST_RESERVED) {
        slot = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(A.d_nraw), 1ull);
        if (slot >= A.cap) {
          atomicAdd(&A.stats[ST_OVERFLOW], 1ull);
          slot = -1;
          k = KEY_DEAD;
        }
      }
    }
    idv = (1ull << 62) | ((uint64_t)A.cycle << 40) | ((uint64_t)A.species << 37) |
          ((uint64_t)gc * (uint64_t)A.ppc + kk);
  }
  if (slot >= 0) {
#pragma unroll
    for (int d = 0; d < 3; ++d) { A.dst[d][slot] = xnew[d]; A.dst[3 + d][slot] = vnew[d]; }
    A.dst[6][slot] = A.q;
    A.dst_id[slot] = (int64_t)idv;
    A.key_new[slot] = k;
  }
  const bool counted = slot >= 0 && k < KEY_FIRST_RESERVED;
  const uint32_t r = count_rank(A.cell_count, g.ncells, k, counted, true);
  if (counted) A.rank[slot] = r;
}

__global__ void clamp_nraw_kernel(int64_t *d_nraw, int64_t cap) {
  if (*d_nraw > cap) *d_nraw = cap;
}

pic_status clamp_nraw(Ctx *ctx, int s) {
  clamp_nraw_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sp[s].d_nraw, ctx->sp[s].cap); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

pic_status inject(Ctx *ctx, int s) {
  SpeciesStore &sp = ctx->sp[s];
  const InjectParams &ip = ctx->inj[s];
  const Geom &g = ctx->geom;
  if (ip.ppc <= 0 || g.periodic[0] || g.slab_lo != 0) return PIC_OK;
  InjectArgs A;
  A.g = g;
  for (int k = 0; k < 7; ++k) A.dst[k] = sp.a[k];
  A.dst_id = sp.id;
  A.key_new = sp.key_new;
  A.rank = sp.rank;
  A.cell_count = sp.cell_count;
  A.d_nraw = sp.d_nraw;
  A.cap = sp.cap;
  A.F = ctx->field();
  A.stats = ctx->stats;
  A.ks = sp.qom * (g.dt * 0.5);
  A.ks_c = A.ks / g.c;
  A.n_iter = sp.n_iter;
  A.rel = ctx->cfg.relativistic;
  A.species = s;
  A.ppc = ip.ppc;
  A.seed_lo = (uint32_t)ip.seed;
  A.seed_hi = (uint32_t)(ip.seed >> 32);
  A.cycle = (uint32_t)ctx->cycle;
  A.vth = ip.vth;
  for (int d = 0; d < 3; ++d) A.drift[d] = ip.drift[d];
  A.q = ip.q;
  const int64_t total = g.ncell[1] * g.ncell[2] * (int64_t)ip.ppc;
  inject_kernel<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(A); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  pic_status st = clamp_nraw(ctx, s);
  if (st != PIC_OK) return st;
  sp.n_raw = std::min<int64_t>(sp.cap, sp.n_raw + total);
  return PIC_OK;
}

}  // namespace pic
