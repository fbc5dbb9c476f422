// api.cu — the C ABI of include/pic.h: validation, workspace layout, call-order
// state machine, stream handling and dispatch to the kernel families.
#include <nccl.h>

#include <algorithm>
#include <new>

#include "pic_internal.cuh"

using namespace pic;

namespace {

constexpr int64_t ALIGN = 256;

inline int64_t align_up(int64_t v) { return (v + ALIGN - 1) / ALIGN * ALIGN; }

struct Layout {
  int64_t total = 0;
  int64_t take(int64_t bytes) {
    int64_t off = total;
    total += align_up(bytes);
    return off;
  }
};

pic_status validate(const pic_config *c, std::string *why) {
  if (!c) { *why = "null config"; return PIC_EINVAL; }
  for (int d = 0; d < 3; ++d) {
    if (c->ncell[d] < 2) { *why = "ncell must be >= 2 per axis"; return PIC_EINVAL; }
    if (!(c->len[d] > 0)) { *why = "len must be > 0"; return PIC_EINVAL; }
    if (c->bc[d] != PIC_BC_PERIODIC && c->bc[d] != PIC_BC_OPEN) { *why = "bad bc"; return PIC_EINVAL; }
  }
  if (!(c->dt > 0) || !(c->c > 0)) { *why = "dt and c must be > 0"; return PIC_EINVAL; }
  if (c->n_species < 1 || c->n_species > PIC_MAX_SPECIES) { *why = "n_species out of range"; return PIC_EINVAL; }
  for (int s = 0; s < c->n_species; ++s) {
    if (c->n_iter[s] < 1 || c->n_iter[s] > 64) { *why = "n_iter must be in [1, 64]"; return PIC_EINVAL; }
    if (c->capacity[s] < 0 || c->capacity[s] > (int64_t(1) << 30)) {
      *why = "capacity must be in [0, 2^30] per species per rank"; return PIC_EINVAL;
    }
  }
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) { *why = "bad rank/nranks"; return PIC_EINVAL; }
  if (c->slab_lo < 0 || c->slab_hi > c->ncell[0] || c->slab_hi - c->slab_lo < 1) {
    *why = "bad slab"; return PIC_EINVAL;
  }
  if (c->nranks == 1 && (c->slab_lo != 0 || c->slab_hi != c->ncell[0])) {
    *why = "single rank must own all x cells"; return PIC_EINVAL;
  }
  if (c->ghost < 1 || c->ghost > 8) { *why = "ghost must be in [1, 8]"; return PIC_EINVAL; }
  if (c->nranks > 1 && c->slab_hi - c->slab_lo < c->ghost + 1) {
    *why = "slab narrower than ghost + 1 cells"; return PIC_EINVAL;
  }
  const int64_t tcells = ((c->slab_hi - c->slab_lo + TILE - 1) / TILE) * ((c->ncell[1] + TILE - 1) / TILE) *
                         ((c->ncell[2] + TILE - 1) / TILE) * TILE3;
  if (tcells >= (int64_t)KEY_FIRST_RESERVED) { *why = "too many local cells for 32-bit keys"; return PIC_EINVAL; }
  if (c->planet_radius < 0) { *why = "planet_radius < 0"; return PIC_EINVAL; }
  if (c->transport < PIC_TRANSPORT_AUTO || c->transport > PIC_TRANSPORT_LOOPBACK) { *why = "bad transport"; return PIC_EINVAL; }
  if (c->kernel < 0 || c->kernel > 2) { *why = "bad kernel"; return PIC_EINVAL; }
  if (c->relativistic != 0 && c->relativistic != 1) { *why = "relativistic must be 0 or 1"; return PIC_EINVAL; }
  if (c->barrier_timeout_ms < 0) { *why = "barrier_timeout_ms must be >= 0"; return PIC_EINVAL; }
  if (c->far_hops < 0 || (c->far_hops > 0 && c->far_hops >= c->nranks)) {
    *why = "far_hops must be in [0, nranks)"; return PIC_EINVAL;
  }
  return PIC_OK;
}

void make_geom(const pic_config *c, Geom *g) {
  memset(g, 0, sizeof(*g));
  for (int d = 0; d < 3; ++d) {
    g->ncell[d] = c->ncell[d];
    g->periodic[d] = c->bc[d] == PIC_BC_PERIODIC;
    g->delta[d] = c->len[d] / (double)c->ncell[d];
    g->inv_delta[d] = 1.0 / g->delta[d];
    g->planet_c[d] = c->planet_center[d] / g->delta[d];
  }
  g->dt = c->dt;
  g->c = c->c;
  g->planet_r2 = c->planet_radius * c->planet_radius;
  g->has_planet = c->planet_radius > 0;
  g->slab_lo = c->slab_lo;
  g->slab_hi = c->slab_hi;
  g->G = c->ghost;
  g->multi_rank = c->nranks > 1;
  g->far_hops = c->far_hops;
  const int64_t G = c->ghost;
  g->f_lo[0] = c->slab_lo - G; g->f_lo[1] = -G; g->f_lo[2] = -G;
  g->f_n[0] = c->slab_hi - c->slab_lo + 1 + 2 * G;
  g->f_n[1] = c->ncell[1] + 1 + 2 * G;
  g->f_n[2] = c->ncell[2] + 1 + 2 * G;
  g->m_lo[0] = c->slab_lo - G; g->m_lo[1] = 0; g->m_lo[2] = 0;
  g->m_n[0] = c->slab_hi - c->slab_lo + 1 + 2 * G;
  g->m_n[1] = c->ncell[1] + 1;
  g->m_n[2] = c->ncell[2] + 1;
  g->m_plane = g->m_n[0] * g->m_n[1] * g->m_n[2];
  g->k_n[0] = c->slab_hi - c->slab_lo;
  g->k_n[1] = c->ncell[1];
  g->k_n[2] = c->ncell[2];
  for (int d = 0; d < 3; ++d) g->nt[d] = (g->k_n[d] + TILE - 1) / TILE;
  g->ntiles = g->nt[0] * g->nt[1] * g->nt[2];
  g->ncells = g->ntiles * TILE3;
}

// Workspace plan; if base != nullptr, assigns pointers into ctx.
int64_t plan(const pic_config *c, const Geom &g, Ctx *ctx, char *base, size_t cub_bytes) {
  Layout L;
  int64_t cap_max = 0;
  for (int s = 0; s < c->n_species; ++s) cap_max = std::max<int64_t>(cap_max, c->capacity[s]);
  cap_max = std::max<int64_t>(cap_max, 1);
  const int64_t mig_cap = std::max<int64_t>(cap_max / 64, 65536);   // slab leavers per side per species
  for (int s = 0; s < c->n_species; ++s) {
    // two buffers of the SoA store (the mover gathers A[perm[q]] into B[q]),
    // plus the order metadata of the counting sort (order.cu)
    const int64_t cap = std::max<int64_t>(c->capacity[s], 1);
    int64_t oa[7], ob[7];
    for (int k = 0; k < 7; ++k) oa[k] = L.take(8 * cap);
    for (int k = 0; k < 7; ++k) ob[k] = L.take(8 * cap);
    int64_t oid = L.take(8 * cap), oidb = L.take(8 * cap);
    int64_t okn = L.take(4 * cap), ork = L.take(4 * cap), opm = L.take(4 * cap);
    int64_t occ = L.take(8 * (g.ncells + 1)), oco = L.take(4 * (g.ncells + 1)), oct = L.take(4 * (g.ncells + 1));
    int64_t onraw = L.take(8);
    int64_t omom = L.take(8 * 10 * g.m_plane);
    if (base) {
      SpeciesStore &sp = ctx->sp[s];
      for (int k = 0; k < 7; ++k) {
        sp.a[k] = (double *)(base + oa[k]);
        sp.b[k] = (double *)(base + ob[k]);
      }
      sp.id = (int64_t *)(base + oid);
      sp.id_b = (int64_t *)(base + oidb);
      sp.key_new = (uint32_t *)(base + okn);
      sp.rank = (uint32_t *)(base + ork);
      sp.perm = (uint32_t *)(base + opm);
      sp.cell_count = (uint32_t *)(base + occ);
      sp.cell_off = (uint32_t *)(base + oco);
      sp.cell_tot = (uint32_t *)(base + oct);
      sp.d_nraw = (int64_t *)(base + onraw);
      sp.mom = (double *)(base + omom);
      sp.cap = c->capacity[s];
      sp.qom = c->qom[s];
      sp.n_iter = c->n_iter[s];
    }
  }
  int64_t field_elems = g.f_n[0] * g.f_n[1] * g.f_n[2] * 6;
  int64_t ofield[2] = {L.take(8 * field_elems), L.take(8 * field_elems)};
  int64_t ostats = L.take(8 * ST_N);
  int64_t ocounts = L.take(8 * 64);
  int64_t opeer = L.take(sizeof(PeerCtl));
  const int64_t face = g.m_n[1] * g.m_n[2] * 10;
  const int64_t ghost_elems = (int64_t)(c->ghost + 1) * face;
  int64_t og[4];
  const bool multi = c->nranks > 1;
  for (int k = 0; k < 4; ++k) og[k] = L.take(multi ? 8 * ghost_elems * c->n_species : 8);
  int64_t om[4];
  for (int k = 0; k < 4; ++k) om[k] = L.take(multi ? 8 * 8 * mig_cap * c->n_species : 8);
  const int64_t pack_elems = (g.k_n[0] + 1) * g.m_n[1] * g.m_n[2] * 10;
  int64_t opack = L.take(8 * pack_elems);
  int64_t osrc = L.take(8 * 13 * (pack_elems / 10));
  int64_t ogmm = L.take(8 * (64 * 64 * 64 + 128));
  int64_t oslot[2 * PIC_MAX_SPECIES];
  for (int k = 0; k < 2 * c->n_species; ++k) oslot[k] = L.take(8 * pack_elems);
  int64_t ocub = L.take((int64_t)cub_bytes);
  if (base) {
    ctx->field_buf[0] = (double *)(base + ofield[0]);
    ctx->field_buf[1] = (double *)(base + ofield[1]);
    for (int k = 0; k < 2 * c->n_species; ++k) ctx->pack_slot[k] = (double *)(base + oslot[k]);
    ctx->field_elems = field_elems;
    ctx->stats = (unsigned long long *)(base + ostats);
    ctx->dev_counts = (int64_t *)(base + ocounts);
    ctx->peer_ctl = (PeerCtl *)(base + opeer);
    ctx->ghost_send[0] = (double *)(base + og[0]);
    ctx->ghost_send[1] = (double *)(base + og[1]);
    ctx->ghost_recv[0] = (double *)(base + og[2]);
    ctx->ghost_recv[1] = (double *)(base + og[3]);
    ctx->ghost_elems = ghost_elems;
    ctx->mig_send[0] = (double *)(base + om[0]);
    ctx->mig_send[1] = (double *)(base + om[1]);
    ctx->mig_recv[0] = (double *)(base + om[2]);
    ctx->mig_recv[1] = (double *)(base + om[3]);
    ctx->mig_cap = mig_cap;
    // the peer transports never use the send buffers: they hold the forwarded
    // far-flyers, [hop parity] halves of mig_send[from side]
    ctx->fwd_cap = mig_cap / 2;
    for (int par = 0; par < 2; ++par)
      for (int side = 0; side < 2; ++side)
        ctx->fwd_recv[par][side] = ctx->mig_send[side] + (int64_t)par * MIG_REC * (mig_cap / 2) * c->n_species;
    ctx->pack = (double *)(base + opack);
    ctx->src_buf = (double *)(base + osrc);
    ctx->gmm_buf = (double *)(base + ogmm);
    ctx->cub_temp = base + ocub;
    ctx->cub_bytes = cub_bytes;
    ctx->cap_max = cap_max;
  }
  return L.total + ALIGN;
}

inline Ctx *C(pic_ctx *p) { return reinterpret_cast<Ctx *>(p); }
inline const Ctx *C(const pic_ctx *p) { return reinterpret_cast<const Ctx *>(p); }

pic_status check_species(Ctx *ctx, int32_t s, bool allow_all) {
  if (allow_all && s == -1) return PIC_OK;
  if (s < 0 || s >= ctx->cfg.n_species) return fail(ctx, PIC_EINVAL, "species index out of range");
  return PIC_OK;
}

bool use_tiled(const Ctx *ctx) {
  return ctx->cfg.kernel == PIC_KERNEL_TILED || ctx->cfg.kernel == PIC_KERNEL_AUTO;
}

}  // namespace

extern "C" {

int32_t pic_abi_version(void) { return PIC_ABI_VERSION; }

pic_status pic_nccl_id(void *out) {
  if (!out) return PIC_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PIC_ENCCL;
  static_assert(sizeof(ncclUniqueId) == PIC_NCCL_ID_BYTES, "nccl id size");
  memcpy(out, &id, sizeof(id));
  return PIC_OK;
}

pic_status pic_workspace_bytes(const pic_config *cfg, int64_t *bytes) {
  std::string why;
  pic_status st = validate(cfg, &why);
  if (st != PIC_OK) return st;
  if (!bytes) return PIC_EINVAL;
  Geom g;
  make_geom(cfg, &g);
  *bytes = plan(cfg, g, nullptr, nullptr, order_temp_bytes(g.ncells));
  return PIC_OK;
}

pic_status pic_init(const pic_config *cfg, const void *nccl_id, void *workspace, int64_t bytes,
                    pic_ctx **out) {
  if (!out) return PIC_EINVAL;
  *out = nullptr;
  std::string why;
  pic_status st = validate(cfg, &why);
  if (st != PIC_OK) return st;
  if (!workspace || ((uintptr_t)workspace % ALIGN) != 0) return PIC_EINVAL;
  Ctx *ctx = new (std::nothrow) Ctx();
  if (!ctx) return PIC_ENOMEM;
  ctx->cfg = *cfg;
  make_geom(cfg, &ctx->geom);
  const size_t cub_bytes = order_temp_bytes(ctx->geom.ncells);
  const int64_t need = plan(cfg, ctx->geom, nullptr, nullptr, cub_bytes);
  if (bytes < need) {
    delete ctx;
    return PIC_ENOMEM;
  }
  plan(cfg, ctx->geom, ctx, (char *)workspace, cub_bytes);
  ctx->workspace = workspace;
  cudaError_t e = cudaHostAlloc((void **)&ctx->host_counts, 64 * sizeof(int64_t), cudaHostAllocDefault);
  if (e != cudaSuccess) { delete ctx; return PIC_ECUDA; }
  e = cudaMemset(ctx->stats, 0, 8 * ST_N);
  if (e != cudaSuccess) { cudaFreeHost(ctx->host_counts); delete ctx; return PIC_ECUDA; }
  e = cudaMemset(ctx->field_buf[0], 0, 8 * ctx->field_elems);
  if (e == cudaSuccess) e = cudaMemset(ctx->field_buf[1], 0, 8 * ctx->field_elems);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&ctx->field_ready[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->field_free[k], cudaEventDisableTiming);
  }
  for (int k = 0; k < 2 * cfg->n_species && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&ctx->slot_packed[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->slot_free[k], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->copies_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->fields_done, cudaEventDisableTiming);
  if (e != cudaSuccess) { cudaFreeHost(ctx->host_counts); delete ctx; return PIC_ECUDA; }
  if (cfg->nranks > 1 && cfg->transport == PIC_TRANSPORT_LOOPBACK) {
    // no communicator: pic_loopback_link joins the contexts of this process
    e = cudaMemset(ctx->peer_ctl, 0, sizeof(PeerCtl));
    if (e != cudaSuccess) { cudaFreeHost(ctx->host_counts); delete ctx; return PIC_ECUDA; }
  } else if (cfg->nranks > 1) {
    if (!nccl_id) { cudaFreeHost(ctx->host_counts); delete ctx; return PIC_EINVAL; }
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclComm_t comm;
    if (ncclCommInitRank(&comm, cfg->nranks, id, cfg->rank) != ncclSuccess) {
      cudaFreeHost(ctx->host_counts);
      delete ctx;
      return PIC_ENCCL;
    }
    ctx->nccl = comm;
    if (peer_setup(ctx) != PIC_OK) {
      ncclCommDestroy(comm);
      cudaFreeHost(ctx->host_counts);
      delete ctx;
      return PIC_ECUDA;
    }
  }
  for (int s = 0; s < cfg->n_species; ++s) {
    if (zero_moments(ctx, s) != PIC_OK) { cudaFreeHost(ctx->host_counts); delete ctx; return PIC_ECUDA; }
  }
  *out = reinterpret_cast<pic_ctx *>(ctx);
  return PIC_OK;
}

pic_status pic_loopback_link(pic_ctx *const *ctxs, int32_t n) {
  if (!ctxs || n < 2 || n > 64) return PIC_EINVAL;
  int dev0 = -1;
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r]) return PIC_EINVAL;
    Ctx *ctx = C(ctxs[r]);
    const pic_config &c = ctx->cfg;
    if (c.transport != PIC_TRANSPORT_LOOPBACK || c.nranks != n || c.rank != r)
      return fail(ctx, PIC_EINVAL, "pic_loopback_link: ctxs[r] must be rank r of a loopback config with nranks == n");
    if (ctx->peer) return fail(ctx, PIC_ESTATE, "pic_loopback_link: already linked");
    if (r > 0) {
      const pic_config &c0 = C(ctxs[0])->cfg;
      bool same = c.n_species == c0.n_species && c.ghost == c0.ghost && c.slab_lo == C(ctxs[r - 1])->cfg.slab_hi;
      for (int d = 0; d < 3; ++d) same = same && c.ncell[d] == c0.ncell[d] && c.bc[d] == c0.bc[d];
      if (!same) return fail(ctx, PIC_EINVAL, "pic_loopback_link: slabs must tile one grid in rank order");
    }
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ctx->workspace) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, PIC_ECUDA, "pic_loopback_link: workspace is not device memory");
    }
    if (dev0 < 0) dev0 = at.device;
    if (at.device != dev0) return fail(ctx, PIC_EINVAL, "pic_loopback_link: contexts on different devices");
  }
  if (C(ctxs[0])->cfg.slab_lo != 0 || C(ctxs[n - 1])->cfg.slab_hi != C(ctxs[0])->cfg.ncell[0])
    return fail(C(ctxs[0]), PIC_EINVAL, "pic_loopback_link: slabs must cover the x axis");
  std::vector<Ctx *> v(n);
  for (int r = 0; r < n; ++r) v[r] = C(ctxs[r]);
  return loopback_link(v.data(), n);
}

pic_status pic_set_stream(pic_ctx *p, void *stream) {
  if (!p) return PIC_EINVAL;
  C(p)->stream = (cudaStream_t)stream;
  return PIC_OK;
}

pic_status pic_set_particles(pic_ctx *p, int32_t s, int64_t n, const double *const xyzuvwq[7],
                             const int64_t *id) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (n < 0) return fail(ctx, PIC_EINVAL, "n < 0");
  if (n > ctx->sp[s].cap) return fail(ctx, PIC_ERANGE, "n exceeds capacity");
  if (n > 0) {
    if (!xyzuvwq) return fail(ctx, PIC_EINVAL, "null particle arrays");
    for (int k = 0; k < 7; ++k)
      if (!xyzuvwq[k]) return fail(ctx, PIC_EINVAL, "null particle array");
  }
  st = load_particles(ctx, s, n, xyzuvwq, id);
  if (st != PIC_OK) return st;
  ctx->sp[s].moved = ctx->sp[s].deposited = false;
  return PIC_OK;
}

pic_status pic_add_particles(pic_ctx *p, int32_t s, int64_t n, const double *const xyzuvwq[7], const int64_t *id) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (n < 0) return fail(ctx, PIC_EINVAL, "n < 0");
  if (ctx->sp[s].moved) return fail(ctx, PIC_ESTATE, "pic_add_particles between pic_mover and pic_exchange");
  if (n > 0) {
    if (!xyzuvwq) return fail(ctx, PIC_EINVAL, "null particle arrays");
    for (int k = 0; k < 7; ++k)
      if (!xyzuvwq[k]) return fail(ctx, PIC_EINVAL, "null particle array");
  }
  st = append_particles(ctx, s, n, xyzuvwq, id);
  if (st != PIC_OK) return st;
  ctx->sp[s].deposited = false;
  return PIC_OK;
}

pic_status pic_count(pic_ctx *p, int32_t s, int64_t *n) {
  if (!p || !n) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (ctx->sp[s].moved) return fail(ctx, PIC_ESTATE, "pic_count between pic_mover and pic_exchange");
  return live_count(ctx, s, n);
}

pic_status pic_get_particles(pic_ctx *p, int32_t s, double *const xyzuvwq[7], int64_t *id) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (ctx->sp[s].moved)
    return fail(ctx, PIC_ESTATE, "pic_get_particles between pic_mover and pic_exchange");
  double *none[7] = {};
  return unload_particles(ctx, s, xyzuvwq ? xyzuvwq : none, id);
}

pic_status pic_set_fields(pic_ctx *p, const double *EB) {
  if (!p || !EB) return PIC_EINVAL;
  Ctx *ctx = C(p);
  // into the buffer the next mover will read, on the copy stream, once the
  // mover that last read that buffer is done (double buffering: the copy of
  // the next cycle's fields overlaps the current cycle)
  const int b = ctx->field_cur ^ 1;
  PIC_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, ctx->field_free[b], 0));
  // a device source may be produced by work on the caller's stream: order the
  // copy after it (host sources need no ordering and overlap the cycle)
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, EB) == cudaSuccess && at.type == cudaMemoryTypeDevice) {
    PIC_CUDA(cudaEventRecord(ctx->field_ready[b], ctx->stream));
    PIC_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, ctx->field_ready[b], 0));
  }
  cudaGetLastError();
  PIC_CUDA(cudaMemcpyAsync(ctx->field_buf[b], EB, 8 * ctx->field_elems, cudaMemcpyDefault, ctx->h2d_stream));
  PIC_CUDA(cudaEventRecord(ctx->field_ready[b], ctx->h2d_stream));
  ctx->field_new = true;
  ctx->fields_set = true;
  return PIC_OK;
}

pic_status pic_mover(pic_ctx *p, int32_t s) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, true);
  if (st != PIC_OK) return st;
  if (!ctx->fields_set) return fail(ctx, PIC_ESTATE, "pic_set_fields must precede pic_mover");
  if (ctx->cfg.nranks > 1 && ctx->cfg.transport == PIC_TRANSPORT_LOOPBACK) {
    if (!ctx->peer) return fail(ctx, PIC_ESTATE, "loopback contexts need pic_loopback_link before pic_mover");
    // the flag barriers spin on the device: every context needs its own stream
    for (Ctx *nb : ctx->loop_nb)
      if (!ctx->stream || (nb && nb->stream == ctx->stream))
        return fail(ctx, PIC_EINVAL, "loopback contexts need distinct non-default streams (pic_set_stream)");
  }
  const int s0 = s < 0 ? 0 : s, s1 = s < 0 ? ctx->cfg.n_species : s + 1;
  for (int k = s0; k < s1; ++k)
    if (ctx->sp[k].moved || !ctx->sp[k].order_valid)
      return fail(ctx, PIC_ESTATE, "pic_mover called twice without pic_exchange");
  for (int k = s0; k < s1; ++k) {
    st = ensure_order(ctx, k);
    if (st != PIC_OK) return st;
  }
  if (ctx->field_new) {
    ctx->field_cur ^= 1;
    ctx->field_new = false;
    PIC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->field_ready[ctx->field_cur], 0));
  }
  if (use_tiled(ctx)) {
    // one launch for the species that share n_iter (species-major tiles)
    for (int a = s0; a < s1;) {
      int b = a + 1;
      while (b < s1 && ctx->sp[b].n_iter == ctx->sp[a].n_iter) ++b;
      st = launch_tiled_step(ctx, a, b);
      if (st != PIC_OK) return st;
      a = b;
    }
  } else {
    for (int k = s0; k < s1; ++k) {
      st = launch_mover_basic(ctx, k);
      if (st != PIC_OK) return st;
    }
  }
  for (int k = s0; k < s1; ++k) {
    ctx->sp[k].moved = true;
    ctx->sp[k].deposited = false;
  }
  // inflow injection (NEXT-3) appends the wind particles that entered this cycle
  for (int k = s0; k < s1; ++k) {
    PhaseTimer t(ctx, 6);
    st = inject(ctx, k);
    if (st != PIC_OK) return st;
  }
  // the field buffer may be refilled once these movers are done (a cycle being
  // captured into a graph records this after the graph launch instead)
  cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
  PIC_CUDA(cudaStreamIsCapturing(ctx->stream, &cap_st));
  if (cap_st == cudaStreamCaptureStatusNone)
    PIC_CUDA(cudaEventRecord(ctx->field_free[ctx->field_cur], ctx->stream));
  // slab leavers go to their neighbour right after the mover (Alg. 1: the
  // particle communication follows the push), every species in one NCCL group
  // per message; the receiver deposits them like its own particles
  if (ctx->cfg.nranks > 1) {
    st = ctx->peer ? peer_migrate(ctx, s0, s1) : migrate(ctx, s0, s1);
    if (st != PIC_OK) return st;
  }
  // the next cell order (stayers, in-slab arrivals, migrated arrivals)
  for (int k = s0; k < s1; ++k) {
    PhaseTimer t(ctx, 1);
    st = build_order(ctx, k);
    if (st != PIC_OK) return st;
  }
  return PIC_OK;
}

pic_status pic_moments(pic_ctx *p, int32_t s) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, true);
  if (st != PIC_OK) return st;
  const int s0 = s < 0 ? 0 : s, s1 = s < 0 ? ctx->cfg.n_species : s + 1;
  for (int k = s0; k < s1; ++k)
    if (ctx->sp[k].deposited) return fail(ctx, PIC_ESTATE, "pic_moments called twice without pic_exchange");
  for (int k = s0; k < s1; ++k) {
    st = ensure_order(ctx, k);
    if (st != PIC_OK) return st;
  }
  {
    PhaseTimer t(ctx, 2);
    if (use_tiled(ctx)) {
      st = launch_tiled_deposit(ctx, s0, s1);   // one launch, species-major tiles
    } else {
      for (int k = s0; k < s1 && st == PIC_OK; ++k) {
        st = zero_moments(ctx, k);
        if (st == PIC_OK) st = launch_moments_basic(ctx, k);
      }
    }
  }
  if (st != PIC_OK) return st;
  for (int k = s0; k < s1; ++k) ctx->sp[k].deposited = true;
  return PIC_OK;
}

pic_status pic_exchange(pic_ctx *p) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  for (int k = 0; k < ctx->cfg.n_species; ++k)
    if (!ctx->sp[k].deposited) return fail(ctx, PIC_ESTATE, "pic_exchange before pic_moments of every species");
  pic_status st;
  {
    PhaseTimer t(ctx, 3);
    st = ctx->peer ? peer_exchange(ctx) : exchange(ctx);
  }
  if (st != PIC_OK) return st;
  for (int k = 0; k < ctx->cfg.n_species; ++k) ctx->sp[k].moved = ctx->sp[k].deposited = false;
  ctx->cycle++;
  return PIC_OK;
}

static pic_status cycle_plain(pic_ctx *p) {
  pic_status st = pic_mover(p, -1);
  if (st != PIC_OK) return st;
  st = pic_moments(p, -1);
  if (st != PIC_OK) return st;
  return pic_exchange(p);
}

// A cycle can be replayed from a CUDA graph when every kernel argument is fixed
// by (field buffer, store buffer parity) and no host decision sits inside it:
// one rank or the peer transport (the NCCL transport learns the migration
// counts on the host; the loopback barrier is a host handshake), no inflow
// injection (its draws are keyed by the host's cycle counter), no profiling
// events, and every species in one state.
static bool graph_ok(const Ctx *ctx) {
  if (ctx->prof_on) return false;
  // stream capture needs a stream of its own (not the legacy default stream)
  if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy || ctx->stream == cudaStreamPerThread) return false;
  if (ctx->cfg.nranks > 1 && (!ctx->peer || ctx->loop)) return false;
  for (int s = 0; s < ctx->cfg.n_species; ++s) {
    const SpeciesStore &sp = ctx->sp[s];
    if (ctx->inj[s].ppc > 0 || sp.moved || sp.deposited || !sp.order_valid || sp.order_dirty) return false;
  }
  return ctx->fields_set;
}

static pic_status cycle_graph(pic_ctx *p) {
  Ctx *ctx = C(p);
  if (ctx->field_new) {            // as pic_mover: switch to the freshly copied field buffer
    ctx->field_cur ^= 1;
    ctx->field_new = false;
    PIC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->field_ready[ctx->field_cur], 0));
  }
  Ctx::CycleGraph *G = nullptr;
  for (auto &g : ctx->graphs)
    if (g.exec && g.field_cur == ctx->field_cur && g.a0 == ctx->sp[0].a[0]) G = &g;
  if (G) {
    PIC_CUDA(cudaGraphLaunch((cudaGraphExec_t)G->exec, ctx->stream));
    PIC_CUDA(cudaEventRecord(ctx->field_free[ctx->field_cur], ctx->stream));
    // the host-side effects of the replayed cycle
    for (int s = 0; s < ctx->cfg.n_species; ++s) ctx->sp[s].swap_buffers();
    ctx->launches += G->launches;
    ctx->cycle++;
    return PIC_OK;
  }
  for (auto &g : ctx->graphs)
    if (!g.exec) G = &g;
  if (!G) return cycle_plain(p);   // (cannot happen: at most 2 x 2 keys)
  // grid sizes of the grid-stride kernels from the capacity (the host's
  // running upper bound of the store is not advanced by replays)
  for (int s = 0; s < ctx->cfg.n_species; ++s) ctx->sp[s].n_raw = ctx->sp[s].cap;
  const int field_cur = ctx->field_cur;
  const double *a0 = ctx->sp[0].a[0];
  const int64_t l0 = ctx->launches;
  PIC_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  pic_status st = cycle_plain(p);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (st != PIC_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return fail(ctx, PIC_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(ctx, PIC_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  G->exec = exec;
  G->field_cur = field_cur;
  G->a0 = a0;
  G->launches = ctx->launches - l0;
  // the capture enqueued nothing: run the captured cycle (host state already advanced)
  PIC_CUDA(cudaGraphLaunch(exec, ctx->stream));
  PIC_CUDA(cudaEventRecord(ctx->field_free[field_cur], ctx->stream));
  return PIC_OK;
}

pic_status pic_cycle(pic_ctx *p) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  if (ctx->graph_on && graph_ok(ctx)) return cycle_graph(p);
  return cycle_plain(p);
}

pic_status pic_set_graph(pic_ctx *p, int32_t enable) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  ctx->graph_on = enable != 0;
  return PIC_OK;
}

pic_status pic_moment_shape(const pic_ctx *p, int64_t out[3]) {
  if (!p || !out) return PIC_EINVAL;
  const Ctx *ctx = C(p);
  const pic_config &c = ctx->cfg;
  out[0] = c.slab_hi - c.slab_lo + ((c.bc[0] == PIC_BC_OPEN && c.slab_hi == c.ncell[0]) ? 1 : 0);
  out[1] = c.ncell[1] + (c.bc[1] == PIC_BC_OPEN ? 1 : 0);
  out[2] = c.ncell[2] + (c.bc[2] == PIC_BC_OPEN ? 1 : 0);
  return PIC_OK;
}

pic_status pic_get_moments(pic_ctx *p, int32_t s, double *out) {
  if (!p || !out) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  return pack_moments(ctx, s, out);
}

pic_status pic_sync(pic_ctx *p, int64_t stats[8]) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->copy_stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->h2d_stream));
  unsigned long long h[ST_N];
  PIC_CUDA(cudaMemcpy(h, ctx->stats, sizeof(h), cudaMemcpyDeviceToHost));
  int64_t all[ST_N];
  for (int k = 0; k < ST_N; ++k) all[k] = (int64_t)h[k] + (k < 8 ? ctx->hstat[k] : 0);
  if (stats)
    for (int k = 0; k < ST_PUBLIC; ++k) stats[k] = all[k];
  if (all[ST_CHECK]) return fail(ctx, PIC_ECUDA, "checked build: " + std::to_string(all[ST_CHECK]) +
                                                   " device bounds checks failed");
  if (ctx->peer) {
    unsigned long long perr = 0;
    PIC_CUDA(cudaMemcpy(&perr, &ctx->peer_ctl->err, sizeof(perr), cudaMemcpyDeviceToHost));
    if (perr) return fail(ctx, PIC_ENCCL, "peer barrier timed out (a neighbour rank stopped)");
  }
  if (all[ST_NONFINITE]) return fail(ctx, PIC_ENONFINITE, "non-finite particle update");
  if (all[ST_FAR] || all[ST_OVERFLOW] || all[ST_MULTIWRAP])
    return fail(ctx, PIC_ERANGE, "particle beyond ghost reach, capacity overflow or multiple wrap");
  return PIC_OK;
}

pic_status pic_get_moments_async(pic_ctx *p, int32_t s, double *out) {
  if (!p || !out) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  return pack_moments_async(ctx, s, out);
}

pic_status pic_implicit_sources(pic_ctx *p, double *chi, double *rho_hat, double *J_hat) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  for (int k = 0; k < ctx->cfg.n_species; ++k)
    if (ctx->sp[k].moved || ctx->sp[k].deposited)
      return fail(ctx, PIC_ESTATE, "pic_implicit_sources needs the moments after pic_exchange");
  if (!ctx->fields_set) return fail(ctx, PIC_ESTATE, "pic_implicit_sources needs pic_set_fields (B)");
  return implicit_sources(ctx, chi, rho_hat, J_hat);
}

pic_status pic_set_injection(pic_ctx *p, int32_t s, int32_t ppc, double vth, const double drift[3], double q,
                             uint64_t seed) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (ppc < 0 || !(vth >= 0.0) || !drift) return fail(ctx, PIC_EINVAL, "bad injection parameters");
  if (ppc > 0 && ctx->cfg.bc[0] != PIC_BC_OPEN) return fail(ctx, PIC_EINVAL, "injection needs an open x axis");
  InjectParams &ip = ctx->inj[s];
  ip.ppc = ppc;
  ip.vth = vth;
  for (int d = 0; d < 3; ++d) ip.drift[d] = drift[d];
  ip.q = q;
  ip.seed = seed;
  return PIC_OK;
}

pic_status pic_control(pic_ctx *p, int32_t s, int64_t target, double theta, double eps, double dv, uint64_t seed,
                       int32_t *action) {
  if (!p || !action) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (ctx->sp[s].moved || !ctx->sp[s].order_valid)
    return fail(ctx, PIC_ESTATE, "pic_control runs between cycles (after pic_exchange)");
  if (!(theta >= 0.0) || !(eps > 0.0 && eps < 0.5) || !(dv > 0.0))
    return fail(ctx, PIC_EINVAL, "pic_control: theta >= 0, 0 < eps < 0.5, dv > 0");
  return control(ctx, s, target, theta, eps, dv, seed, action);
}

pic_status pic_gmm(pic_ctx *p, int32_t s, int32_t B, double vmax, int32_t M, int32_t n_em, double *alpha, double *mu,
                   double *sigma, double *hist, int64_t *clipped) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  pic_status st = check_species(ctx, s, false);
  if (st != PIC_OK) return st;
  if (ctx->sp[s].moved || !ctx->sp[s].order_valid)
    return fail(ctx, PIC_ESTATE, "pic_gmm runs between cycles (after pic_exchange)");
  st = ensure_order(ctx, s);
  if (st != PIC_OK) return st;
  return gmm_fit(ctx, s, B, vmax, M, n_em, alpha, mu, sigma, hist, clipped);
}

pic_status pic_moment_ptr(const pic_ctx *p, int32_t s, int32_t comp, const double **ptr, int64_t strides[3],
                          int64_t origin[3], double *scale) {
  if (!p || !ptr || !strides || !origin || !scale) return PIC_EINVAL;
  const Ctx *ctx = C(p);
  if (s < 0 || s >= ctx->cfg.n_species || comp < 0 || comp >= 10) return PIC_EINVAL;
  const Geom &g = ctx->geom;
  *ptr = ctx->sp[s].mom + comp * g.m_plane + g.G;
  strides[0] = 1;
  strides[1] = g.m_n[0];
  strides[2] = g.m_n[0] * g.m_n[1];
  origin[0] = g.slab_lo;
  origin[1] = 0;
  origin[2] = 0;
  *scale = 1.0 / (g.delta[0] * g.delta[1] * g.delta[2]);
  return PIC_OK;
}

pic_status pic_join_copies(pic_ctx *p) {
  if (!p) return PIC_EINVAL;
  return join_copies(C(p));
}

pic_status pic_get_transport(const pic_ctx *p, int32_t *out) {
  if (!p || !out) return PIC_EINVAL;
  const Ctx *ctx = C(p);
  *out = ctx->cfg.nranks < 2 ? PIC_TRANSPORT_AUTO
        : ctx->cfg.transport == PIC_TRANSPORT_LOOPBACK ? PIC_TRANSPORT_LOOPBACK
        : (ctx->peer ? PIC_TRANSPORT_PEER : PIC_TRANSPORT_NCCL);
  return PIC_OK;
}

pic_status pic_launch_count(const pic_ctx *p, int64_t *n) {
  if (!p || !n) return PIC_EINVAL;
  *n = C(p)->launches;
  return PIC_OK;
}

pic_status pic_profile(pic_ctx *p, int32_t enable) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto &v : ctx->prof_ev)
    for (auto &e : v) {
      ctx->prof_pool.push_back(e.first);
      ctx->prof_pool.push_back(e.second);
    }
  for (auto &v : ctx->prof_ev) v.clear();
  ctx->prof_on = enable != 0;
  return PIC_OK;
}

pic_status pic_profile_read(pic_ctx *p, double ms[PIC_PROF_PHASES], int64_t launches[PIC_PROF_PHASES]) {
  if (!p || !ms || !launches) return PIC_EINVAL;
  Ctx *ctx = C(p);
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < PIC_PROF_PHASES; ++k) {
    double t = 0.0;
    for (auto &e : ctx->prof_ev[k]) {
      float f = 0.f;
      PIC_CUDA(cudaEventElapsedTime(&f, e.first, e.second));
      t += f;
    }
    ms[k] = t;
    launches[k] = (int64_t)ctx->prof_ev[k].size();
  }
  return PIC_OK;
}

const char *pic_last_error(const pic_ctx *p) {
  if (!p) return "null context";
  return C(p)->err.c_str();
}

pic_status pic_destroy(pic_ctx *p) {
  if (!p) return PIC_EINVAL;
  Ctx *ctx = C(p);
  cudaStreamSynchronize(ctx->stream);
  for (cudaStream_t cs : {ctx->copy_stream, ctx->h2d_stream})
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
    }
  for (int k = 0; k < 2; ++k) {
    if (ctx->field_ready[k]) cudaEventDestroy(ctx->field_ready[k]);
    if (ctx->field_free[k]) cudaEventDestroy(ctx->field_free[k]);
  }
  for (int k = 0; k < 2 * PIC_MAX_SPECIES; ++k) {
    if (ctx->slot_packed[k]) cudaEventDestroy(ctx->slot_packed[k]);
    if (ctx->slot_free[k]) cudaEventDestroy(ctx->slot_free[k]);
  }
  if (ctx->copies_done) cudaEventDestroy(ctx->copies_done);
  if (ctx->fields_done) cudaEventDestroy(ctx->fields_done);
  for (auto &g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy((cudaGraphExec_t)g.exec);
  peer_close(ctx);
  if (ctx->nccl) ncclCommDestroy((ncclComm_t)ctx->nccl);
  for (auto &v : ctx->prof_ev)
    for (auto &e : v) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
  cudaFreeHost(ctx->host_counts);
  delete ctx;
  return PIC_OK;
}

}  // extern "C"
