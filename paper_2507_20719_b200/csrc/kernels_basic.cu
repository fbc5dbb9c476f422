// kernels_basic.cu — PIC_KERNEL_BASIC: one thread per particle.
//
//   mover_basic    Eq. 2, gamma = 1 (R3), first field
//                  sample at x^n (R1), fixed n_iter (R2), trilinear gather from
//                  the global field window (R12), boundary conditions (R10,
//                  R11, R21) and the destination key of the new position.
//                  Reads A[perm[q]], writes B[q] and ranks the particle for
//                  the next cell order (order.cu, built by pic_mover after
//                  the slab migration).
//   moments_basic  Eq. 3: 10 moments x 8 corners per
//                  particle, global fp64 atomics (RED.E.ADD.F64) into the
//                  ghosted node arrays.
//
// This family is the simple reference path on the GPU: correct for every
// config, but the deposit costs 80 global atomics per particle.
#include "pic_internal.cuh"
#include "push.cuh"

namespace pic {

struct MoverArgs {
  Geom g;
  const double *src[7];
  const int64_t *src_id;
  double *dst[7];
  int64_t *dst_id;
  const uint32_t *perm;
  const uint32_t *cell_off;   // cell_off[ncells] = number of particles to move
  uint32_t *key_new, *rank, *cell_count;
  int64_t *d_nraw;
  const double *F;
  unsigned long long *stats;
  double ks, ks_c;
  int n_iter;
  int rel;                    // relativistic Eq. 2 (NEXT-1)
  int peer;                   // slab leavers go straight into the neighbours' buffers (peer.cu)
  PeerOut po;
  int64_t cap;
};

__global__ void __launch_bounds__(256) mover_basic_kernel(const MoverArgs A) {
  const Geom &g = A.g;
  const int64_t n = A.cell_off[g.ncells];
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q == 0) *A.d_nraw = n;
  if ((int64_t)blockIdx.x * blockDim.x >= n) return;   // whole warps leave together
  const bool act = q < n;
  uint32_t k = KEY_DEAD, kold = KEY_DEAD;
  if (act) {
    const uint32_t p = A.perm[q];
    PIC_DCHECK(p < A.cap && q < A.cap, A.stats);
    const double xn[3] = {A.src[0][p], A.src[1][p], A.src[2][p]};
    // the cell of x^n (keys are always taken from the stored position)
    kold = tile_key32(g, (uint32_t)((int)xn[0] - (int)g.slab_lo), (uint32_t)(int)xn[1], (uint32_t)(int)xn[2]);
    const double vn[3] = {A.src[3][p], A.src[4][p], A.src[5][p]};
    const double h[3] = {0.5 * g.dt * g.inv_delta[0], 0.5 * g.dt * g.inv_delta[1], 0.5 * g.dt * g.inv_delta[2]};
    // Eq. 2 (push.cuh) with samples from the global field window
    const WindowSampler sample{&g, A.F, A.ks, A.ks_c};
    double xnew[3], vnew[3];
    const bool clamped = A.rel ? push_eq2<0, 1>(xn, vn, h, g.c, A.n_iter, sample, xnew, vnew)
                               : push_eq2<0, 0>(xn, vn, h, g.c, A.n_iter, sample, xnew, vnew);
    k = finish_particle(g, xnew, vnew, clamped, A.stats);
    A.dst[0][q] = xnew[0]; A.dst[1][q] = xnew[1]; A.dst[2][q] = xnew[2];
    A.dst[3][q] = vnew[0]; A.dst[4][q] = vnew[1]; A.dst[5][q] = vnew[2];
    A.dst[6][q] = A.src[6][p];
    A.dst_id[q] = A.src_id[p];
    A.key_new[q] = k;
  }
  const bool counted = act && k < KEY_FIRST_RESERVED;
  const uint32_t r = count_rank(A.cell_count, g.ncells, k, counted, !act || k != kold);
  if (counted) A.rank[q] = r;
  if (A.peer && __any_sync(0xffffffffu, k == KEY_LEFT || k == KEY_RIGHT))
    send_leavers_peer(A.po, k, A.dst, A.dst_id, q, A.stats);
}

__global__ void __launch_bounds__(256) moments_basic_kernel(
    Geom g, const double *__restrict__ X, const double *__restrict__ Y,
    const double *__restrict__ Z, const double *__restrict__ U, const double *__restrict__ V,
    const double *__restrict__ W, const double *__restrict__ Q, const uint32_t *__restrict__ key,
    const int64_t *__restrict__ d_nraw, double *__restrict__ mom, unsigned long long *__restrict__ stats) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= *d_nraw) return;
  // removed particles and slab leavers (deposited by their new owner) skip
  if (key[p] >= KEY_FIRST_RESERVED) return;
  const double xi[3] = {X[p], Y[p], Z[p]};
  const double v3[3] = {U[p], V[p], W[p]};
  if (!deposit_global(g, mom, xi, Q[p], v3)) atomicAdd(&stats[ST_FAR], 1ull);
}

pic_status launch_mover_basic(Ctx *ctx, int s) {
  SpeciesStore &S = ctx->sp[s];
  pic_status st = zero_cell_counts(ctx, s);
  if (st != PIC_OK) return st;
  MoverArgs A;
  A.g = ctx->geom;
  for (int k = 0; k < 7; ++k) { A.src[k] = S.a[k]; A.dst[k] = S.b[k]; }
  A.src_id = S.id;
  A.dst_id = S.id_b;
  A.perm = S.perm;
  A.cell_off = S.cell_off;
  A.key_new = S.key_new;
  A.rank = S.rank;
  A.cell_count = S.cell_count;
  A.d_nraw = S.d_nraw;
  A.F = ctx->field();
  A.stats = ctx->stats;
  A.ks = S.qom * (ctx->geom.dt * 0.5);
  A.ks_c = A.ks / ctx->geom.c;
  A.n_iter = S.n_iter;
  A.rel = ctx->cfg.relativistic;
  A.peer = ctx->peer;
  A.po = ctx->peer ? peer_out(ctx, s) : PeerOut{};
  A.cap = S.cap;
  const int threads = 256;
  const int64_t blocks = std::max<int64_t>(1, (S.n_raw + threads - 1) / threads);
  {
    PhaseTimer t(ctx, 0);
    mover_basic_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(A); ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  S.swap_buffers();
  return PIC_OK;
}

pic_status launch_moments_basic(Ctx *ctx, int s) {
  SpeciesStore &S = ctx->sp[s];
  if (S.n_raw == 0) return PIC_OK;
  const int threads = 256;
  const int64_t blocks = (S.n_raw + threads - 1) / threads;
  moments_basic_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(
      ctx->geom, S.a[0], S.a[1], S.a[2], S.a[3], S.a[4], S.a[5], S.a[6], S.key_new, S.d_nraw, S.mom,
      ctx->stats); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

}  // namespace pic
