// sources.cu — NEXT-2: the implicit field solver's particle sources from the
// gathered moments, Eq. 5 (susceptibility chi) and Eq. 6 (rho-hat, J-hat),
// PAPER.md:199-213, readings R24-R27.
//
// Node-local: chi = sum_s (1/2)(omega_ps dt)^2 R_s with omega_ps^2 =
// 4 pi rho_s q_s/m_s and R_s x = (x - a x x + (a.x) a)/(1 + a.a), a =
// q_s B dt/(2 m_s c); J-hat = sum_s R_s (J_s - (dt/2) div Pi_s).  Then
// rho-hat = sum_s rho_s - dt div J-hat.  Derivatives: second-order central
// differences over the owned nodes, periodic wrap, one-sided first order at
// the boundary nodes of an open axis (R27).  Two HBM-bound stencil passes over
// the owned nodes (one thread per node).
#include "pic_internal.cuh"

namespace pic {

struct SourcesArgs {
  Geom g;
  const double *mom[PIC_MAX_SPECIES];   // ghosted raw sums [10][m_plane] (after pic_exchange)
  double qom[PIC_MAX_SPECIES];
  int n_species;
  const double *field;                  // window [z][y][x][6]
  int64_t n[3];                         // owned nodes
  double invV;
  double inv_delta[3], inv_2delta[3];   // stencil factors (one-sided, central)
  double *chi, *rho_hat, *J_hat;        // [9][n], [n], [3][n] (owned-node layout)
  // x neighbours (multi-rank, peer transport): their moment arrays and J-hat
  int has_nb[2];                        // [0] left, [1] right
  const double *nb_mom[2][PIC_MAX_SPECIES];
  int64_t nb_plane[2], nb_nx[2], nb_xm[2];   // moment plane stride, x extent, x index of the adjacent plane
  const double *nb_jh[2];               // J-hat [3][nb_total]
  int64_t nb_total[2], nb_xj[2];        // their owned node count, x index of the adjacent owned plane
};

// owned node (i, j, k) -> element of the ghosted moment arrays
__device__ __forceinline__ int64_t src_node(const SourcesArgs &A, int64_t i, int64_t j, int64_t k) {
  return (k * A.g.m_n[1] + j) * A.g.m_n[0] + (A.g.G + i);
}

// d f / d x_axis at owned node c of a field given by a functor over owned nodes;
// along x a functor index of -1 / n[0] means the left / right neighbour's
// adjacent plane (multi-rank)
template <class F>
__device__ __forceinline__ double node_diff(const SourcesArgs &A, const int64_t c[3], int axis, F f) {
  const int64_t n = A.n[axis];
  int64_t lo[3] = {c[0], c[1], c[2]}, hi[3] = {c[0], c[1], c[2]};
  double ih = A.inv_2delta[axis];   // 1 / (2 delta), or 1 / delta one-sided
  if (axis == 0 && A.g.multi_rank) {
    const bool L = c[0] == 0, R = c[0] == n - 1;
    if ((!L || A.has_nb[0]) && (!R || A.has_nb[1])) {
      lo[0] = c[0] - 1;   // -1: left neighbour
      hi[0] = c[0] + 1;   // n: right neighbour
    } else if (L) {       // global open face: one-sided (R27)
      hi[0] = 1;          // (== n with one owned plane: the right neighbour)
      ih = A.inv_delta[axis];
    } else {
      lo[0] = n - 2;
      ih = A.inv_delta[axis];
    }
  } else if (A.g.periodic[axis]) {
    lo[axis] = c[axis] == 0 ? n - 1 : c[axis] - 1;
    hi[axis] = c[axis] == n - 1 ? 0 : c[axis] + 1;
  } else if (c[axis] == 0) {
    hi[axis] = 1;
    ih = A.inv_delta[axis];
  } else if (c[axis] == n - 1) {
    lo[axis] = n - 2;
    ih = A.inv_delta[axis];
  } else {
    lo[axis] = c[axis] - 1;
    hi[axis] = c[axis] + 1;
  }
  return (f(hi) - f(lo)) * ih;
}

__device__ __forceinline__ void apply_R(const double a[3], const double x[3], double out[3]) {
  const double cr0 = a[1] * x[2] - a[2] * x[1];
  const double cr1 = a[2] * x[0] - a[0] * x[2];
  const double cr2 = a[0] * x[1] - a[1] * x[0];
  const double dot = a[0] * x[0] + a[1] * x[1] + a[2] * x[2];
  const double inv = 1.0 / (1.0 + (a[0] * a[0] + a[1] * a[1] + a[2] * a[2]));
  out[0] = (x[0] - cr0 + dot * a[0]) * inv;
  out[1] = (x[1] - cr1 + dot * a[1]) * inv;
  out[2] = (x[2] - cr2 + dot * a[2]) * inv;
}

__global__ void chi_jhat_kernel(const SourcesArgs A) {
  const int64_t total = A.n[0] * A.n[1] * A.n[2];
  const double dt = A.g.dt;
  const double four_pi = 4.0 * 3.14159265358979323846;
  {
    // one thread per owned node: x from the block row, y and z from the grid
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n[0]) return;
    const int64_t c[3] = {i, (int64_t)blockIdx.y, (int64_t)blockIdx.z};
    const int64_t t = (c[2] * A.n[1] + c[1]) * A.n[0] + c[0];
    // B at the node from the field window (global node slab_lo + i, j, k)
    const double *fw = A.field + 6 * (((c[2] - A.g.f_lo[2]) * A.g.f_n[1] + (c[1] - A.g.f_lo[1])) * A.g.f_n[0] +
                                      (A.g.slab_lo + c[0] - A.g.f_lo[0]));
    const double B[3] = {fw[3], fw[4], fw[5]};
    double chi[9] = {}, jh[3] = {};
    const int64_t me = src_node(A, c[0], c[1], c[2]);
    for (int s = 0; s < A.n_species; ++s) {
      const double *m = A.mom[s];
      const double qom = A.qom[s];
      const int64_t P = A.g.m_plane;
      double a[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) a[d] = (qom * B[d] / A.g.c) * (dt / 2.0);
      const double w2 = four_pi * (m[me] * A.invV) * qom;     // R24: rho_s q_s/m_s >= 0
#pragma unroll
      for (int col = 0; col < 3; ++col) {
        double e[3] = {0.0, 0.0, 0.0}, r[3];
        e[col] = 1.0;
        apply_R(a, e, r);
#pragma unroll
        for (int row = 0; row < 3; ++row) chi[row * 3 + col] += 0.5 * w2 * dt * dt * r[row];
      }
      // (div Pi)_a = sum_b d Pi_ab / d x_b, Pi order xx xy xz yy yz zz (components 4..9)
      const int pidx[3][3] = {{4, 5, 6}, {5, 7, 8}, {6, 8, 9}};
      double x[3];
#pragma unroll
      for (int ra = 0; ra < 3; ++ra) {
        double div = 0.0;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int cm = pidx[ra][b];
          const double *comp = m + cm * P;
          div += node_diff(A, c, b, [&](const int64_t q[3]) {
            if (q[0] < 0 || q[0] >= A.n[0]) {   // neighbour's adjacent owned plane
              const int sd = q[0] < 0 ? 0 : 1;
              return A.nb_mom[sd][s][cm * A.nb_plane[sd] + (q[2] * A.g.m_n[1] + q[1]) * A.nb_nx[sd] + A.nb_xm[sd]] *
                     A.invV;
            }
            return comp[src_node(A, q[0], q[1], q[2])] * A.invV;
          });
        }
        x[ra] = m[(1 + ra) * P + me] * A.invV - (dt / 2.0) * div;
      }
      double r[3];
      apply_R(a, x, r);
#pragma unroll
      for (int d = 0; d < 3; ++d) jh[d] += r[d];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) A.chi[q * total + t] = chi[q];
#pragma unroll
    for (int d = 0; d < 3; ++d) A.J_hat[d * total + t] = jh[d];
  }
}

__global__ void rho_hat_kernel(const SourcesArgs A) {
  const int64_t total = A.n[0] * A.n[1] * A.n[2];
  {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n[0]) return;
    const int64_t c[3] = {i, (int64_t)blockIdx.y, (int64_t)blockIdx.z};
    const int64_t t = (c[2] * A.n[1] + c[1]) * A.n[0] + c[0];
    const int64_t me = src_node(A, c[0], c[1], c[2]);
    double rho = 0.0;
    for (int s = 0; s < A.n_species; ++s) rho += A.mom[s][me] * A.invV;
    double div = 0.0;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double *comp = A.J_hat + b * total;
      div += node_diff(A, c, b, [&](const int64_t q[3]) {
        if (q[0] < 0 || q[0] >= A.n[0]) {
          const int sd = q[0] < 0 ? 0 : 1;
          return A.nb_jh[sd][b * A.nb_total[sd] + (q[2] * A.n[1] + q[1]) * (A.nb_total[sd] / (A.n[1] * A.n[2])) +
                             A.nb_xj[sd]];
        }
        return comp[(q[2] * A.n[1] + q[1]) * A.n[0] + q[0]];
      });
    }
    A.rho_hat[t] = rho - A.g.dt * div;
  }
}

pic_status implicit_sources(Ctx *ctx, double *chi, double *rho_hat, double *J_hat) {
  if (ctx->cfg.nranks > 1 && !ctx->peer)
    return fail(ctx, PIC_EINVAL, "pic_implicit_sources with several ranks needs the peer transport");
  const Geom &g = ctx->geom;
  int64_t shape[3];
  pic_moment_shape((const pic_ctx *)ctx, shape);
  SourcesArgs A;
  A.g = g;
  A.n_species = ctx->cfg.n_species;
  for (int s = 0; s < A.n_species; ++s) {
    A.mom[s] = ctx->sp[s].mom;
    A.qom[s] = ctx->sp[s].qom;
  }
  // B of the most recent pic_set_fields
  const int b = ctx->field_new ? (ctx->field_cur ^ 1) : ctx->field_cur;
  if (ctx->field_new) PIC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->field_ready[b], 0));
  A.field = ctx->field_buf[b];
  for (int d = 0; d < 3; ++d) A.n[d] = shape[d];
  A.invV = 1.0 / (g.delta[0] * g.delta[1] * g.delta[2]);
  for (int d = 0; d < 3; ++d) {
    A.inv_delta[d] = 1.0 / g.delta[d];
    A.inv_2delta[d] = 1.0 / (2.0 * g.delta[d]);
  }
  const int64_t total = shape[0] * shape[1] * shape[2];
  // chi and rho-hat go straight into the caller's arrays when they are device
  // memory (no copy); J-hat always lands in the workspace first, where the
  // neighbours' rho-hat pass reads it over NVLink
  auto on_device = [](const void *p) {
    cudaPointerAttributes at;
    if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
  };
  const bool chi_dev = on_device(chi), rho_dev = on_device(rho_hat);
  A.chi = chi_dev ? chi : ctx->src_buf;
  A.J_hat = ctx->src_buf + 9 * total;
  A.rho_hat = rho_dev ? rho_hat : ctx->src_buf + 12 * total;
  for (int sd = 0; sd < 2; ++sd) {
    const Ctx::PeerLink &L = ctx->link[sd];
    A.has_nb[sd] = (g.multi_rank && L.mapped) ? 1 : 0;
    for (int s = 0; s < A.n_species; ++s) A.nb_mom[sd][s] = L.mom[s];
    A.nb_plane[sd] = L.m_plane;
    A.nb_nx[sd] = L.m_nx;
    // left: its last owned plane (array x index ghost_x - 1); right: its first (G)
    A.nb_xm[sd] = sd == 0 ? L.ghost_x - 1 : g.G;
    A.nb_total[sd] = L.owned_nx * shape[1] * shape[2];
    A.nb_jh[sd] = L.src ? L.src + 9 * A.nb_total[sd] : nullptr;
    A.nb_xj[sd] = sd == 0 ? L.owned_nx - 1 : 0;
  }
  const dim3 grid((unsigned)((shape[0] + 127) / 128), (unsigned)shape[1], (unsigned)shape[2]);
  if (shape[1] > 65535 || shape[2] > 65535) return fail(ctx, PIC_EINVAL, "sources: more than 65535 nodes in y or z");
  pic_status st;
  if (g.multi_rank) {   // the neighbours' moments are final (their pic_exchange)
    st = peer_barrier(ctx);
    if (st != PIC_OK) return st;
  }
  chi_jhat_kernel<<<grid, 128, 0, ctx->stream>>>(A); ++ctx->launches;
  if (g.multi_rank) {   // the neighbours' J-hat is complete
    st = peer_barrier(ctx);
    if (st != PIC_OK) return st;
  }
  rho_hat_kernel<<<grid, 128, 0, ctx->stream>>>(A); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  if (chi && !chi_dev)
    PIC_CUDA(cudaMemcpyAsync(chi, A.chi, 9 * sizeof(double) * total, cudaMemcpyDefault, ctx->stream));
  if (J_hat) PIC_CUDA(cudaMemcpyAsync(J_hat, A.J_hat, 3 * sizeof(double) * total, cudaMemcpyDefault, ctx->stream));
  if (rho_hat && !rho_dev)
    PIC_CUDA(cudaMemcpyAsync(rho_hat, A.rho_hat, sizeof(double) * total, cudaMemcpyDefault, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  return PIC_OK;
}

}  // namespace pic
