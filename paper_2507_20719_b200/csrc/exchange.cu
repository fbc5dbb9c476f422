// exchange.cu — slab migration (inside pic_mover), ghost-node moment sums and
// periodic folds (pic_exchange), plus particle / moment copy-in and copy-out.
//
// Paper mapping (Alg. 1 phase 2): "exiting particles are
// transferred using MPI".  Here slab leavers travel to the neighbouring slab
// right after the mover, before the order for the deposit is built, so every
// particle is deposited once, by its owner.  The x ghost planes (the stencil
// of the owner's last cell reaches node slab_hi) are then summed into their
// owners with NCCL point-to-point over NVLink (ring-periodic along x when x is
// periodic).  The ghost-node sum itself is implied, not stated, by the paper
// (north_star).
#include <nccl.h>

#include "pic_internal.cuh"

namespace pic {

#define PIC_NCCL(call)                                                       \
  do {                                                                       \
    ncclResult_t r_ = (call);                                                \
    if (r_ != ncclSuccess)                                                   \
      return fail(ctx, PIC_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// ------------------------------------------------------------- moment folds --
// Periodic y / z fold: plane N (the image of plane 0, R18) is added into 0.
// x planes [x0, x0 + nA) of arrays with nx planes.
__global__ void fold_axis_kernel(double *mom, int64_t nx, int64_t ny, int64_t nz, int axis,
                                 int64_t plane, int64_t x0, int64_t nA) {
  // iterate over the 2D face (other two axes) x 10 components
  int64_t nB = axis == 1 ? nz : ny;
  int64_t total = nA * nB * 10;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = x0 + t % nA, b = (t / nA) % nB, m = t / (nA * nB);
    int64_t src, dst;
    if (axis == 1) {  // y: a = x, b = z
      src = (b * ny + (ny - 1)) * nx + a;
      dst = (b * ny + 0) * nx + a;
    } else {          // z: a = x, b = y
      src = ((nz - 1) * ny + b) * nx + a;
      dst = (0 * ny + b) * nx + a;
    }
    mom[m * plane + dst] += mom[m * plane + src];
    mom[m * plane + src] = 0.0;
  }
}

// Copy (mode 0) or add (mode 1) `count` x-planes between a moment array and a
// contiguous plane buffer [10][count][nz][ny] (x-plane major per component).
__global__ void xplanes_kernel(double *mom, double *buf, int64_t x0, int64_t count, int64_t nx,
                               int64_t ny, int64_t nz, int64_t plane, int mode, int to_buf) {
  int64_t face = ny * nz;
  int64_t total = face * count * 10;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t yz = t % face, xi = (t / face) % count, m = t / (face * count);
    int64_t y = yz % ny, z = yz / ny;
    int64_t node = (z * ny + y) * nx + (x0 + xi);
    double *pm = mom + m * plane + node;
    if (to_buf) {
      buf[t] = *pm;
    } else {
      if (mode == 1) *pm += buf[t]; else *pm = buf[t];
    }
  }
}

// Local periodic fold along x (nranks == 1): ghost planes onto their images.
__global__ void fold_x_local_kernel(double *mom, int64_t N, int G, int64_t nx, int64_t ny,
                                    int64_t nz, int64_t plane) {
  // array x-index a holds global node a - G; images: a-G in [N, N+G] -> (a-G-N),
  // a-G in [-G, -1] -> a-G+N.
  int64_t face = ny * nz;
  int64_t nghost = 2 * G + 1;
  int64_t total = face * 10;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t yz = t % face, m = t / face;
    double *base = mom + m * plane + yz * nx;
    for (int64_t k = 0; k < nghost; ++k) {
      int64_t gidx = (k < G) ? (k - G) : (N + (k - G));  // global node of the ghost
      int64_t a_src = gidx + G;
      int64_t a_dst = ((gidx % N) + N) % N + G;
      base[a_dst] += base[a_src];
      base[a_src] = 0.0;
    }
  }
}

static unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > kSMs * 16) b = kSMs * 16;
  if (b < 1) b = 1;
  return (unsigned)b;
}

pic_status launch_fold_axis(Ctx *ctx, int s, int axis, int64_t x0, int64_t nxr) {
  const Geom &g = ctx->geom;
  const int64_t nx = g.m_n[0], ny = g.m_n[1], nz = g.m_n[2];
  const int64_t other = axis == 1 ? nz : ny;
  fold_axis_kernel<<<grid_for(nxr * other * 10), 256, 0, ctx->stream>>>(ctx->sp[s].mom, nx, ny, nz, axis, g.m_plane,
                                                                        x0, nxr); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

static pic_status fold_and_ghosts(Ctx *ctx) {
  const Geom &g = ctx->geom;
  const int64_t nx = g.m_n[0], ny = g.m_n[1], nz = g.m_n[2];
  const int S = ctx->cfg.n_species;
  for (int s = 0; s < S; ++s) {
    double *mom = ctx->sp[s].mom;
    if (g.periodic[1])
      fold_axis_kernel<<<grid_for(nx * nz * 10), 256, 0, ctx->stream>>>(mom, nx, ny, nz, 1, g.m_plane, 0, nx); ++ctx->launches;
    if (g.periodic[2])
      fold_axis_kernel<<<grid_for(nx * ny * 10), 256, 0, ctx->stream>>>(mom, nx, ny, nz, 2, g.m_plane, 0, nx); ++ctx->launches;
    if (ctx->cfg.nranks == 1 && g.periodic[0])
      fold_x_local_kernel<<<grid_for(ny * nz * 10), 256, 0, ctx->stream>>>(
          mom, g.ncell[0], g.G, nx, ny, nz, g.m_plane); ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  if (ctx->cfg.nranks == 1) return PIC_OK;

  // multi-rank: ghost planes along x to the neighbours.
  const int G = g.G;
  const int r = ctx->cfg.rank, P = ctx->cfg.nranks;
  const bool per = g.periodic[0];
  const int left = (r > 0) ? r - 1 : (per ? P - 1 : -1);
  const int right = (r < P - 1) ? r + 1 : (per ? 0 : -1);
  // array x-index of global node X is X - (slab_lo - G)
  const int64_t nloc = g.slab_hi - g.slab_lo;
  const int64_t a_right_ghost = G + nloc;   // planes [slab_hi, slab_hi+G] -> G+1 planes
  const int64_t a_left_ghost = 0;           // planes [slab_lo-G, slab_lo-1] -> G planes
  const int64_t face = ny * nz * 10;
  const int64_t nR = (int64_t)(G + 1) * face, nL = (int64_t)G * face;
  ncclComm_t comm = (ncclComm_t)ctx->nccl;
  const int64_t gs = ctx->ghost_elems;   // per-species stride in the ghost buffers
  for (int s = 0; s < S; ++s) {
    double *mom = ctx->sp[s].mom;
    if (right >= 0)
      xplanes_kernel<<<grid_for(nR), 256, 0, ctx->stream>>>(mom, ctx->ghost_send[1] + s * gs, a_right_ghost,
                                                             G + 1, nx, ny, nz, g.m_plane, 0, 1); ++ctx->launches;
    if (left >= 0)
      xplanes_kernel<<<grid_for(nL), 256, 0, ctx->stream>>>(mom, ctx->ghost_send[0] + s * gs, a_left_ghost,
                                                             G, nx, ny, nz, g.m_plane, 0, 1); ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  // one NCCL group for every species; per-peer order send-right, send-left,
  // recv-left, recv-right (matches when left == right, P == 2)
  PIC_NCCL(ncclGroupStart());
  for (int s = 0; s < S; ++s) {
    if (right >= 0) PIC_NCCL(ncclSend(ctx->ghost_send[1] + s * gs, nR, ncclDouble, right, comm, ctx->stream));
    if (left >= 0) PIC_NCCL(ncclSend(ctx->ghost_send[0] + s * gs, nL, ncclDouble, left, comm, ctx->stream));
    if (left >= 0) PIC_NCCL(ncclRecv(ctx->ghost_recv[0] + s * gs, nR, ncclDouble, left, comm, ctx->stream));
    if (right >= 0) PIC_NCCL(ncclRecv(ctx->ghost_recv[1] + s * gs, nL, ncclDouble, right, comm, ctx->stream));
  }
  PIC_NCCL(ncclGroupEnd());
  for (int s = 0; s < S; ++s) {
    double *mom = ctx->sp[s].mom;
    // from the left neighbour: its planes [its slab_hi, +G] == my [slab_lo, slab_lo+G]
    if (left >= 0)
      xplanes_kernel<<<grid_for(nR), 256, 0, ctx->stream>>>(mom, ctx->ghost_recv[0] + s * gs, G, G + 1, nx,
                                                             ny, nz, g.m_plane, 1, 0); ++ctx->launches;
    // from the right neighbour: its planes [its slab_lo-G, -1] == my [slab_hi-G, slab_hi-1]
    if (right >= 0)
      xplanes_kernel<<<grid_for(nL), 256, 0, ctx->stream>>>(mom, ctx->ghost_recv[1] + s * gs, nloc, G, nx,
                                                             ny, nz, g.m_plane, 1, 0); ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

// ---------------------------------------------------------------- migration --
// Slab leavers (keys LEFT / RIGHT written by the mover) are packed from the A
// positions into the send buffers as records of 8 words (x y z u v w q, id
// bits), so one message per neighbour and species carries them; slots come
// from warp-aggregated atomics.  No compaction of the stayers is needed: the
// next cell order (order.cu) only contains counted particles.
struct Arr7 { double *a[7]; };

__global__ void pack_leavers_kernel(Arr7 A, const int64_t *__restrict__ id, const uint32_t *__restrict__ key,
                                    const int64_t *__restrict__ d_nraw, double *__restrict__ sendL,
                                    double *__restrict__ sendR, int64_t mig_cap,
                                    unsigned long long *__restrict__ counts) {
  const int64_t n = *d_nraw;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t p = base + threadIdx.x;
    const uint32_t k = p < n ? key[p] : KEY_DEAD;
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const bool mine = k == (side == 0 ? KEY_LEFT : KEY_RIGHT);
      const unsigned mask = __ballot_sync(0xffffffffu, mine);
      if (!mask) continue;
      const int leader = __ffs(mask) - 1;
      unsigned long long slot0 = 0;
      if ((int)lane == leader) slot0 = atomicAdd(&counts[side], (unsigned long long)__popc(mask));
      slot0 = __shfl_sync(0xffffffffu, slot0, leader);
      if (mine) {
        const int64_t slot = (int64_t)slot0 + __popc(mask & ((1u << lane) - 1u));
        if (slot < mig_cap) {
          double *rec = (side == 0 ? sendL : sendR) + slot * MIG_REC;
#pragma unroll
          for (int c = 0; c < 7; ++c) rec[c] = A.a[c][p];
          rec[7] = __longlong_as_double(id[p]);
        }
      }
    }
  }
}

// Key of an in-slab particle from its position (cell units).
__device__ __forceinline__ uint32_t cell_key(const Geom &g, double x, double y, double z) {
  int64_t cx = (int64_t)floor(x) - g.slab_lo, cy = (int64_t)floor(y), cz = (int64_t)floor(z);
  return tile_key(g, cx, cy, cz);
}

// Append received records at `at` (component arrays, ids, keys).
__global__ void append_kernel(Geom g, Arr7 arrs, int64_t *__restrict__ id, uint32_t *__restrict__ key,
                              const double *__restrict__ buf, int64_t cnt, int64_t at,
                              unsigned long long *__restrict__ stats) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double *rec = buf + i * MIG_REC;
    double v[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      v[k] = rec[k];
      arrs.a[k][at + i] = v[k];
    }
    id[at + i] = __double_as_longlong(rec[7]);
    int64_t cx = (int64_t)floor(v[0]);
    if (cx < g.slab_lo || cx >= g.slab_hi) {
      atomicAdd(&stats[ST_FAR], 1ull);
      key[at + i] = KEY_DEAD;
    } else {
      key[at + i] = cell_key(g, v[0], v[1], v[2]);
    }
  }
}

__global__ void set_scalar_kernel(int64_t *dst, int64_t v) { *dst = v; }

// Migration of species [s0, s1) (collective): pack, one NCCL group with the
// counts of every species, one host synchronisation, one NCCL group with the
// payloads, append + rank the arrivals into the cell counts (order.cu).
pic_status migrate(Ctx *ctx, int s0, int s1) {
  const Geom &g = ctx->geom;
  const int S = ctx->cfg.n_species;   // count-scratch layout stride
  const int r = ctx->cfg.rank, P = ctx->cfg.nranks;
  const bool per = g.periodic[0];
  const int left = (r > 0) ? r - 1 : (per ? P - 1 : -1);
  const int right = (r < P - 1) ? r + 1 : (per ? 0 : -1);
  ncclComm_t comm = (ncclComm_t)ctx->nccl;
  const int64_t mc = ctx->mig_cap;
  const int64_t ms = MIG_REC * mc;           // per-species stride in the migration buffers
  // device scratch: [0, 2S) leaver counts L/R per species (unsigned long long),
  // [2S, 3S) A-positions per species, [3S, 5S) received counts from R, from L
  unsigned long long *cnt = (unsigned long long *)ctx->dev_counts;
  int64_t *drecv = ctx->dev_counts + 3 * S;
  int64_t *hc = ctx->host_counts;
  {
    PhaseTimer t(ctx, 4);
    PIC_CUDA(cudaMemsetAsync(cnt + 2 * s0, 0, sizeof(unsigned long long) * 2 * (s1 - s0), ctx->stream));
    for (int s = s0; s < s1; ++s) {
      SpeciesStore &sp = ctx->sp[s];
      if (sp.n_raw > 0) {
        Arr7 A;
        for (int k = 0; k < 7; ++k) A.a[k] = sp.a[k];
        pack_leavers_kernel<<<grid_for(sp.n_raw), 256, 0, ctx->stream>>>(
            A, sp.id, sp.key_new, sp.d_nraw, ctx->mig_send[0] + s * ms, ctx->mig_send[1] + s * ms, mc,
            cnt + 2 * s); ++ctx->launches;
      }
      PIC_CUDA(cudaMemcpyAsync((int64_t *)cnt + 2 * S + s, sp.d_nraw, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    }
    PIC_CUDA(cudaGetLastError());
    // per-peer order send-right, send-left, recv-left, recv-right (matches
    // when left == right, P == 2)
    PIC_NCCL(ncclGroupStart());
    for (int s = s0; s < s1; ++s) {
      if (right >= 0) PIC_NCCL(ncclSend((int64_t *)cnt + 2 * s + 1, 1, ncclInt64, right, comm, ctx->stream));
      if (left >= 0) PIC_NCCL(ncclSend((int64_t *)cnt + 2 * s + 0, 1, ncclInt64, left, comm, ctx->stream));
      if (left >= 0) PIC_NCCL(ncclRecv(drecv + 2 * s + 1, 1, ncclInt64, left, comm, ctx->stream));
      if (right >= 0) PIC_NCCL(ncclRecv(drecv + 2 * s + 0, 1, ncclInt64, right, comm, ctx->stream));
    }
    PIC_NCCL(ncclGroupEnd());
    PIC_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(int64_t) * 5 * S, cudaMemcpyDeviceToHost, ctx->stream));
  }
  // the one host synchronisation of the cycle
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  // Capacity limits are applied identically on both sides of every message
  // (no early return: a rank that stopped here would leave its neighbour's
  // matching ncclSend / ncclRecv blocked forever).  A side sends and receives
  // min(count, mig_cap) records (the pack kernel stored no more); what does
  // not fit is dropped, counted as overflow and reported by pic_sync
  // (PIC_ERANGE), like the peer transport does.
  int64_t nl[PIC_MAX_SPECIES], nr[PIC_MAX_SPECIES], nraw[PIC_MAX_SPECIES];
  int64_t recvL[PIC_MAX_SPECIES], recvR[PIC_MAX_SPECIES], keepL[PIC_MAX_SPECIES], keepR[PIC_MAX_SPECIES];
  for (int s = s0; s < s1; ++s) {
    const int64_t wl = hc[2 * s], wr = hc[2 * s + 1];
    nraw[s] = hc[2 * S + s];
    nl[s] = left >= 0 ? std::min(wl, mc) : 0;     // no neighbour: cannot happen (open faces remove first)
    nr[s] = right >= 0 ? std::min(wr, mc) : 0;
    ctx->hstat[ST_OVERFLOW] += (wl - nl[s]) + (wr - nr[s]);
    recvR[s] = (right >= 0) ? std::min(hc[3 * S + 2 * s + 0], mc) : 0;
    recvL[s] = (left >= 0) ? std::min(hc[3 * S + 2 * s + 1], mc) : 0;
    // appended arrivals that fit the store (the rest were received but are dropped)
    const int64_t room = std::max<int64_t>(0, ctx->sp[s].cap - nraw[s]);
    keepL[s] = std::min(recvL[s], room);
    keepR[s] = std::min(recvR[s], room - keepL[s]);
    ctx->hstat[ST_OVERFLOW] += (recvL[s] - keepL[s]) + (recvR[s] - keepR[s]);
  }
  PhaseTimer t(ctx, 5);
  // payloads of every species in one NCCL group, one message per neighbour
  PIC_NCCL(ncclGroupStart());
  for (int s = s0; s < s1; ++s) {
    const int64_t o = s * ms;
    if (right >= 0 && nr[s]) PIC_NCCL(ncclSend(ctx->mig_send[1] + o, MIG_REC * nr[s], ncclDouble, right, comm, ctx->stream));
    if (left >= 0 && nl[s]) PIC_NCCL(ncclSend(ctx->mig_send[0] + o, MIG_REC * nl[s], ncclDouble, left, comm, ctx->stream));
    if (left >= 0 && recvL[s]) PIC_NCCL(ncclRecv(ctx->mig_recv[0] + o, MIG_REC * recvL[s], ncclDouble, left, comm, ctx->stream));
    if (right >= 0 && recvR[s]) PIC_NCCL(ncclRecv(ctx->mig_recv[1] + o, MIG_REC * recvR[s], ncclDouble, right, comm, ctx->stream));
  }
  PIC_NCCL(ncclGroupEnd());
  for (int s = s0; s < s1; ++s) {
    SpeciesStore &sp = ctx->sp[s];
    Arr7 arrs;
    for (int k = 0; k < 7; ++k) arrs.a[k] = sp.a[k];
    if (keepL[s])
      append_kernel<<<grid_for(keepL[s]), 256, 0, ctx->stream>>>(g, arrs, sp.id, sp.key_new, ctx->mig_recv[0] + s * ms,
                                                                  keepL[s], nraw[s], ctx->stats); ++ctx->launches;
    if (keepR[s])
      append_kernel<<<grid_for(keepR[s]), 256, 0, ctx->stream>>>(g, arrs, sp.id, sp.key_new, ctx->mig_recv[1] + s * ms,
                                                                  keepR[s], nraw[s] + keepL[s], ctx->stats); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
    const int64_t nnew = nraw[s] + keepL[s] + keepR[s];
    set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(sp.d_nraw, nnew); ++ctx->launches;
    pic_status st = count_positions(ctx, s, nraw[s], nnew);
    if (st != PIC_OK) return st;
    sp.n_raw = std::max(sp.n_raw, nnew);
    ctx->hstat[ST_SENT] += nl[s] + nr[s];
    ctx->hstat[ST_RECEIVED] += keepL[s] + keepR[s];
  }
  return PIC_OK;
}

__global__ void keys_from_positions_kernel(Geom g, const double *__restrict__ X, const double *__restrict__ Y,
                                           const double *__restrict__ Z, uint32_t *__restrict__ key, int64_t from,
                                           int64_t to, unsigned long long *__restrict__ stats) {
  for (int64_t p = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < to;
       p += (int64_t)gridDim.x * blockDim.x) {
    double x = X[p], y = Y[p], z = Z[p];
    int64_t cx = (int64_t)floor(x), cy = (int64_t)floor(y), cz = (int64_t)floor(z);
    if (!(cx >= g.slab_lo && cx < g.slab_hi && cy >= 0 && cy < g.ncell[1] && cz >= 0 && cz < g.ncell[2])) {
      atomicAdd(&stats[ST_FAR], 1ull);
      key[p] = KEY_DEAD;
    } else {
      key[p] = cell_key(g, x, y, z);
    }
  }
}

pic_status recompute_keys(Ctx *ctx, int s, int64_t from, int64_t to) {
  SpeciesStore &sp = ctx->sp[s];
  if (to <= from) return PIC_OK;
  keys_from_positions_kernel<<<grid_for(to - from), 256, 0, ctx->stream>>>(ctx->geom, sp.a[0], sp.a[1], sp.a[2],
                                                                           sp.key_new, from, to, ctx->stats); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

pic_status exchange(Ctx *ctx) { return fold_and_ghosts(ctx); }

pic_status zero_moments(Ctx *ctx, int s) {
  PIC_CUDA(cudaMemsetAsync(ctx->sp[s].mom, 0, sizeof(double) * 10 * ctx->geom.m_plane, ctx->stream));
  return PIC_OK;
}

// ------------------------------------------------------------- copy in / out --
__global__ void pack_moments_kernel(const double *__restrict__ mom, double *__restrict__ out,
                                    int64_t ox, int64_t nx, int64_t ny, int64_t nz, int64_t mnx,
                                    int64_t mny, int64_t plane, double invV) {
  int64_t total = nx * ny * nz * 10;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = t % nx, y = (t / nx) % ny, z = (t / (nx * ny)) % nz, m = t / (nx * ny * nz);
    out[t] = mom[m * plane + (z * mny + y) * mnx + (ox + x)] * invV;
  }
}

// Asynchronous copy-out: pack into one of the species' two staging slots on
// the context stream, copy to `out` on the copy stream; the slot is reused
// two calls later, after its copy completed.  `out` is valid after
// pic_join_copies + a stream synchronisation, or pic_sync.
pic_status pack_moments_async(Ctx *ctx, int s, double *out) {
  const Geom &g = ctx->geom;
  int64_t shape[3];
  pic_moment_shape((const pic_ctx *)ctx, shape);
  const double invV = 1.0 / (g.delta[0] * g.delta[1] * g.delta[2]);
  const int64_t total = shape[0] * shape[1] * shape[2] * 10;
  const int k = 2 * s + ctx->slot_next[s];
  ctx->slot_next[s] ^= 1;
  if (ctx->slot_used[k]) PIC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slot_free[k], 0));
  pack_moments_kernel<<<grid_for(total), 256, 0, ctx->stream>>>(
      ctx->sp[s].mom, ctx->pack_slot[k], g.G, shape[0], shape[1], shape[2], g.m_n[0], g.m_n[1], g.m_plane, invV); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  PIC_CUDA(cudaEventRecord(ctx->slot_packed[k], ctx->stream));
  PIC_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->slot_packed[k], 0));
  PIC_CUDA(cudaMemcpyAsync(out, ctx->pack_slot[k], sizeof(double) * total, cudaMemcpyDefault, ctx->copy_stream));
  PIC_CUDA(cudaEventRecord(ctx->slot_free[k], ctx->copy_stream));
  ctx->slot_used[k] = true;
  ctx->copies_pending = true;
  return PIC_OK;
}

// The context stream waits for every copy enqueued so far (no host block).
pic_status join_copies(Ctx *ctx) {
  PIC_CUDA(cudaEventRecord(ctx->fields_done, ctx->h2d_stream));
  PIC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->fields_done, 0));
  if (!ctx->copies_pending) return PIC_OK;
  PIC_CUDA(cudaEventRecord(ctx->copies_done, ctx->copy_stream));
  PIC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->copies_done, 0));
  ctx->copies_pending = false;
  return PIC_OK;
}

pic_status pack_moments(Ctx *ctx, int s, double *out) {
  const Geom &g = ctx->geom;
  int64_t shape[3];
  pic_moment_shape((const pic_ctx *)ctx, shape);
  const double invV = 1.0 / (g.delta[0] * g.delta[1] * g.delta[2]);
  const int64_t total = shape[0] * shape[1] * shape[2] * 10;
  pack_moments_kernel<<<grid_for(total), 256, 0, ctx->stream>>>(
      ctx->sp[s].mom, ctx->pack, g.G, shape[0], shape[1], shape[2], g.m_n[0], g.m_n[1], g.m_plane, invV); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  PIC_CUDA(cudaMemcpyAsync(out, ctx->pack, sizeof(double) * total, cudaMemcpyDefault, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  return PIC_OK;
}

__global__ void divide_kernel(double *a, int64_t n, double d) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    a[p] = a[p] / d;
}
__global__ void iota_kernel(int64_t *a, int64_t n, int64_t first = 0) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    a[p] = first + p;
}
// out[q] = src[perm[q]] * scale  (q < live count)
__global__ void gather_scaled_kernel(const double *__restrict__ src, const uint32_t *__restrict__ perm,
                                     const uint32_t *__restrict__ nlive, double *__restrict__ out, double scale) {
  const int64_t n = *nlive;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = src[perm[q]] * scale;
}
__global__ void gather_i64_kernel(const int64_t *__restrict__ src, const uint32_t *__restrict__ perm,
                                  const uint32_t *__restrict__ nlive, int64_t *__restrict__ out) {
  const int64_t n = *nlive;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = src[perm[q]];
}

pic_status load_particles(Ctx *ctx, int s, int64_t n, const double *const src[7], const int64_t *id) {
  SpeciesStore &sp = ctx->sp[s];
  for (int k = 0; k < 7; ++k) {
    if (n) PIC_CUDA(cudaMemcpyAsync(sp.a[k], src[k], sizeof(double) * n, cudaMemcpyDefault, ctx->stream));
    if (k < 3 && n) {
      divide_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.a[k], n, ctx->geom.delta[k]); ++ctx->launches;
    }
  }
  if (id) {
    if (n) PIC_CUDA(cudaMemcpyAsync(sp.id, id, sizeof(int64_t) * n, cudaMemcpyDefault, ctx->stream));
  } else if (n) {
    iota_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.id, n); ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  sp.n_raw = n;
  set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(sp.d_nraw, n); ++ctx->launches;
  pic_status st = recompute_keys(ctx, s, 0, n);
  if (st != PIC_OK) return st;
  st = zero_cell_counts(ctx, s);
  if (st != PIC_OK) return st;
  st = count_positions(ctx, s, 0, n);
  if (st != PIC_OK) return st;
  st = build_order(ctx, s);
  if (st != PIC_OK) return st;
  uint32_t nlive = 0;
  PIC_CUDA(cudaMemcpyAsync(&nlive, sp.cell_off + ctx->geom.ncells, 4, cudaMemcpyDeviceToHost, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));  // caller buffers may be pageable
  sp.n = nlive;
  return PIC_OK;
}

// Append n particles behind the store's positions [0, d_nraw) and add them to
// the cell order as arrivals (the counts and ranks of the particles already
// there stay valid: they are those the order was built from).
pic_status append_particles(Ctx *ctx, int s, int64_t n, const double *const src[7], const int64_t *id) {
  SpeciesStore &sp = ctx->sp[s];
  if (!sp.order_valid) {
    const double *none[7] = {};
    pic_status st = load_particles(ctx, s, 0, none, nullptr);
    if (st != PIC_OK) return st;
  }
  int64_t old = 0;
  PIC_CUDA(cudaMemcpyAsync(&old, sp.d_nraw, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (old + n > sp.cap) return fail(ctx, PIC_ERANGE, "pic_add_particles: capacity exceeded");
  if (n == 0) return PIC_OK;
  for (int k = 0; k < 7; ++k) {
    PIC_CUDA(cudaMemcpyAsync(sp.a[k] + old, src[k], sizeof(double) * n, cudaMemcpyDefault, ctx->stream));
    if (k < 3) {
      divide_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.a[k] + old, n, ctx->geom.delta[k]); ++ctx->launches;
    }
  }
  if (id) {
    PIC_CUDA(cudaMemcpyAsync(sp.id + old, id, sizeof(int64_t) * n, cudaMemcpyDefault, ctx->stream));
  } else {
    iota_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.id + old, n, old); ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  sp.n_raw = std::max(sp.n_raw, old + n);
  set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(sp.d_nraw, old + n); ++ctx->launches;
  pic_status st = recompute_keys(ctx, s, old, old + n);
  if (st != PIC_OK) return st;
  st = count_positions(ctx, s, old, old + n);
  if (st != PIC_OK) return st;
  sp.order_dirty = true;   // built once, by the next call that needs the order
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));  // caller buffers may be pageable
  return PIC_OK;
}

pic_status live_count(Ctx *ctx, int s, int64_t *n) {
  SpeciesStore &sp = ctx->sp[s];
  pic_status st = ensure_order(ctx, s);
  if (st != PIC_OK) return st;
  uint32_t nlive = 0;
  PIC_CUDA(cudaMemcpyAsync(&nlive, sp.cell_off + ctx->geom.ncells, 4, cudaMemcpyDeviceToHost, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  sp.n = nlive;
  *n = nlive;
  return PIC_OK;
}

pic_status unload_particles(Ctx *ctx, int s, double *const dst[7], int64_t *id) {
  SpeciesStore &sp = ctx->sp[s];
  int64_t n = 0;
  pic_status st = live_count(ctx, s, &n);
  if (st != PIC_OK) return st;
  const uint32_t *nl = sp.cell_off + ctx->geom.ncells;
  // buffer B is free between cycles: gather into it, then copy out
  for (int k = 0; k < 7; ++k) {
    if (!dst[k] || !n) continue;
    gather_scaled_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.a[k], sp.perm, nl, sp.b[k],
                                                               k < 3 ? ctx->geom.delta[k] : 1.0); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
    PIC_CUDA(cudaMemcpyAsync(dst[k], sp.b[k], sizeof(double) * n, cudaMemcpyDefault, ctx->stream));
  }
  if (id && n) {
    gather_i64_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.id, sp.perm, nl, sp.id_b); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
    PIC_CUDA(cudaMemcpyAsync(id, sp.id_b, sizeof(int64_t) * n, cudaMemcpyDefault, ctx->stream));
  }
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  return PIC_OK;
}

}  // namespace pic
