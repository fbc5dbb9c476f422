// peer.cu — multi-rank transport over NVLink peer memory (PIC_TRANSPORT_PEER).
//
// The paper moves exiting particles with MPI after the push and sums the
// moments of shared nodes (Alg. 1 phase 2).  On one
// B200 node every rank can map its slab neighbours' workspaces (CUDA IPC over
// NVLink / NVSwitch), so both exchanges become stores into peer memory issued
// by the kernels that produce the data:
//
//   migration   the mover itself writes every slab leaver's record into the
//               neighbour's receive buffer (send_leavers_peer, pic_internal.cuh;
//               one remote atomic per warp and side reserves the slots).  A
//               flag barrier (release / acquire at system scope) then tells the
//               receiver that its buffer is complete; arrive_kernel appends and
//               ranks the arrivals into the cell counts of the next order, with
//               no host round trip for the counts.
//   ghost sums  after the deposit and a second flag barrier, each rank reads
//               its left neighbour's ghost node plane x = slab_hi (== my
//               slab_lo) from peer memory and adds it into its own plane
//               (ghost_pull_kernel); the periodic y / z folds then run over the
//               owned planes only, so the plane a neighbour reads is never
//               modified concurrently.
//
// Ordering: every barrier is a release store of a monotonically increasing
// epoch into both neighbours' flag words after a system-scope fence, and an
// acquire spin on the own flags (bounded: a neighbour that never arrives sets
// the peer error word instead of hanging the GPU; pic_sync reports it).
// Reuse safety: a receive buffer is refilled only by the neighbour's next
// mover, which starts after the second barrier of this cycle, i.e. after the
// arrivals were consumed; a ghost plane is re-zeroed only after the first
// barrier of the next cycle, i.e. after the neighbour pulled it.
#include <nccl.h>

#include <cuda.h>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>

#include "pic_internal.cuh"

namespace pic {

#define PIC_NCCL(call)                                                       \
  do {                                                                       \
    ncclResult_t r_ = (call);                                                \
    if (r_ != ncclSuccess)                                                   \
      return fail(ctx, PIC_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// What a rank tells its neighbours about its workspace (offsets from the base
// of the CUDA allocation that holds it).
struct PeerDesc {
  cudaIpcMemHandle_t handle;
  int64_t ok;                  // this rank could export its workspace
  int64_t ctl_off;             // PeerCtl
  int64_t recv_off[2];         // receive records: [0] from the left, [1] from the right
  int64_t mom_off[PIC_MAX_SPECIES];
  int64_t mig_cap;             // records per side and species
  int64_t m_plane, m_nx;       // moment array plane stride and x extent
  int64_t ghost_x;             // array x index of node slab_hi (the plane the right neighbour pulls)
  int64_t src_off;             // NEXT-2 sources buffer (J-hat at 9 x owned nodes)
  int64_t owned_nx;            // owned x node planes (pic_moment_shape x)
  int64_t fwd_off[2][2];       // forwarded far-flyers: [hop parity][from side]
  int64_t fwd_cap;
};

static unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > kSMs * 16) b = kSMs * 16;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// ----------------------------------------------------------------- setup ----
// Descriptor of this rank's workspace relative to `base` (the start of the
// allocation that holds it: the CUDA-IPC mapping for the peer transport, the
// workspace itself for the loopback transport).
static PeerDesc describe(Ctx *ctx, char *b) {
  const pic_config &c = ctx->cfg;
  const Geom &g = ctx->geom;
  PeerDesc d;
  memset(&d, 0, sizeof(d));
  d.ctl_off = reinterpret_cast<char *>(ctx->peer_ctl) - b;
  d.recv_off[0] = reinterpret_cast<char *>(ctx->mig_recv[0]) - b;
  d.recv_off[1] = reinterpret_cast<char *>(ctx->mig_recv[1]) - b;
  for (int s = 0; s < c.n_species; ++s) d.mom_off[s] = reinterpret_cast<char *>(ctx->sp[s].mom) - b;
  d.mig_cap = ctx->mig_cap;
  d.m_plane = g.m_plane;
  d.m_nx = g.m_n[0];
  d.ghost_x = g.G + (g.slab_hi - g.slab_lo);
  d.src_off = reinterpret_cast<char *>(ctx->src_buf) - b;
  int64_t shape[3];
  pic_moment_shape((const pic_ctx *)ctx, shape);
  d.owned_nx = shape[0];
  for (int par = 0; par < 2; ++par)
    for (int side = 0; side < 2; ++side) d.fwd_off[par][side] = reinterpret_cast<char *>(ctx->fwd_recv[par][side]) - b;
  d.fwd_cap = ctx->fwd_cap;
  return d;
}

// My link to the neighbour on `side` (0 left, 1 right) whose workspace
// allocation is visible at `mapped` and described by `d`.
static void fill_link(Ctx *ctx, int side, char *mapped, const PeerDesc &d, bool owns) {
  Ctx::PeerLink &L = ctx->link[side];
  L.mapped = mapped;
  L.owns_mapping = owns;
  // I am the neighbour's right (side 0) or left (side 1) neighbour
  const int from = side == 0 ? 1 : 0;
  PeerCtl *pc = reinterpret_cast<PeerCtl *>(mapped + d.ctl_off);
  L.flag = &pc->flag[from];
  L.cnt = &pc->cnt[from][0];
  L.recv = reinterpret_cast<double *>(mapped + d.recv_off[from]);
  L.mig_cap = d.mig_cap;
  for (int s = 0; s < ctx->cfg.n_species; ++s) L.mom[s] = reinterpret_cast<double *>(mapped + d.mom_off[s]);
  L.m_plane = d.m_plane;
  L.m_nx = d.m_nx;
  L.ghost_x = d.ghost_x;
  L.src = reinterpret_cast<double *>(mapped + d.src_off);
  L.owned_nx = d.owned_nx;
  for (int par = 0; par < 2; ++par) {
    L.fcnt[par] = &pc->fcnt[par][from][0];
    L.frecv[par] = reinterpret_cast<double *>(mapped + d.fwd_off[par][from]);
  }
  L.fwd_cap = d.fwd_cap;
}

pic_status peer_setup(Ctx *ctx) {
  const pic_config &c = ctx->cfg;
  const Geom &g = ctx->geom;
  if (c.nranks < 2 || c.transport == PIC_TRANSPORT_NCCL) return PIC_OK;
  const int r = c.rank, P = c.nranks;
  const bool per = g.periodic[0];
  const int left = (r > 0) ? r - 1 : (per ? P - 1 : -1);
  const int right = (r < P - 1) ? r + 1 : (per ? 0 : -1);

  // Clear the own control block BEFORE any neighbour can learn where it is:
  // a neighbour writes into it (arrival counts, barrier epochs) only after it
  // has received this rank's descriptor below, so the clear cannot erase a
  // remote write (a late clear could drop a count or a barrier epoch).
  PIC_CUDA(cudaMemset(ctx->peer_ctl, 0, sizeof(PeerCtl)));
  PIC_CUDA(cudaDeviceSynchronize());
  PeerDesc mine;
  memset(&mine, 0, sizeof(mine));
  // base of the allocation holding the workspace (driver API through the runtime)
  using GetRange = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  char *ws = reinterpret_cast<char *>(ctx->workspace);
  if (get_range && get_range(&base, &size, (CUdeviceptr)ws) == CUDA_SUCCESS &&
      cudaIpcGetMemHandle(&mine.handle, (void *)base) == cudaSuccess) {
    mine.ok = 1;
  }
  cudaGetLastError();
  {
    const cudaIpcMemHandle_t h = mine.handle;
    const int64_t ok = mine.ok;
    mine = describe(ctx, reinterpret_cast<char *>(base));
    mine.handle = h;
    mine.ok = ok;
  }

  // neighbours' descriptors: NCCL point-to-point through a device staging area
  char *stage = reinterpret_cast<char *>(ctx->pack);
  const size_t D = sizeof(PeerDesc);
  PIC_CUDA(cudaMemcpy(stage, &mine, D, cudaMemcpyHostToDevice));
  ncclComm_t comm = (ncclComm_t)ctx->nccl;
  PIC_NCCL(ncclGroupStart());
  if (right >= 0) PIC_NCCL(ncclSend(stage, D, ncclChar, right, comm, ctx->stream));
  if (left >= 0) PIC_NCCL(ncclSend(stage, D, ncclChar, left, comm, ctx->stream));
  if (left >= 0) PIC_NCCL(ncclRecv(stage + D, D, ncclChar, left, comm, ctx->stream));
  if (right >= 0) PIC_NCCL(ncclRecv(stage + 2 * D, D, ncclChar, right, comm, ctx->stream));
  PIC_NCCL(ncclGroupEnd());
  PeerDesc nb[2];
  memset(nb, 0, sizeof(nb));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (left >= 0) PIC_CUDA(cudaMemcpy(&nb[0], stage + D, D, cudaMemcpyDeviceToHost));
  if (right >= 0) PIC_CUDA(cudaMemcpy(&nb[1], stage + 2 * D, D, cudaMemcpyDeviceToHost));

  // map them (once when left == right)
  int ok = mine.ok ? 1 : 0;
  char *mapped[2] = {nullptr, nullptr};
  for (int side = 0; side < 2 && ok; ++side) {
    const int peer = side == 0 ? left : right;
    if (peer < 0) continue;
    if (!nb[side].ok) { ok = 0; break; }
    if (side == 1 && right == left) { mapped[1] = mapped[0]; nb[1] = nb[0]; continue; }
    void *ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, nb[side].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    mapped[side] = reinterpret_cast<char *>(ptr);
  }
  // every rank must agree on the transport
  int *dok = reinterpret_cast<int *>(stage);
  PIC_CUDA(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
  PIC_NCCL(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  int all_ok = 0;
  PIC_CUDA(cudaMemcpy(&all_ok, dok, sizeof(int), cudaMemcpyDeviceToHost));
  if (!all_ok) {
    for (int side = 0; side < 2; ++side)
      if (mapped[side] && !(side == 1 && mapped[1] == mapped[0])) cudaIpcCloseMemHandle(mapped[side]);
    if (c.transport == PIC_TRANSPORT_PEER)
      return fail(ctx, PIC_ECUDA, "peer transport requested but a neighbour workspace cannot be mapped");
    return PIC_OK;   // AUTO: NCCL transport
  }
  for (int side = 0; side < 2; ++side)
    if (mapped[side]) fill_link(ctx, side, mapped[side], nb[side], !(side == 1 && mapped[1] == mapped[0]));
  ctx->peer = true;
  return PIC_OK;
}

// Loopback transport: the P slab contexts of one process on one device link
// to each other directly (the neighbour's workspace needs no mapping).  Every
// data-path kernel of the peer transport runs unchanged (send_leavers_peer in
// the movers, arrive_kernel, ghost_pull_kernel, the sources' neighbour reads);
// only the barrier differs.  A spinning device barrier between streams of ONE
// device can deadlock when two contexts' streams share a hardware queue (the
// spinner blocks the work it waits for), so a loopback barrier is an event
// handshake instead: each context records an event on its stream, its host
// thread waits until both neighbours have recorded theirs for the same epoch,
// and its stream waits on those events.  Each context is driven by its own
// host thread, as a rank would be.
static int barrier_timeout_ms(const Ctx *ctx) {
  return ctx->cfg.barrier_timeout_ms > 0 ? ctx->cfg.barrier_timeout_ms : 20000;
}

struct LoopGroup {
  std::mutex mu;
  std::condition_variable cv;
  int n = 0, refs = 0;
  std::vector<unsigned long long> arrived;      // last barrier epoch recorded per rank
  std::vector<cudaEvent_t> ev;                  // [rank][2]: events of even / odd epochs
};

pic_status loopback_barrier(Ctx *ctx) {
  LoopGroup *G = ctx->loop;
  const int r = ctx->cfg.rank;
  const unsigned long long e = ++ctx->peer_epoch;
  cudaEvent_t mine = G->ev[2 * r + (e & 1)];
  PIC_CUDA(cudaEventRecord(mine, ctx->stream));
  std::unique_lock<std::mutex> lk(G->mu);
  G->arrived[r] = e;
  G->cv.notify_all();
  for (Ctx *nb : ctx->loop_nb) {
    if (!nb) continue;
    const int q = nb->cfg.rank;
    // like the device barrier: a neighbour that never arrives is an error, not a hang
    if (!G->cv.wait_for(lk, std::chrono::milliseconds(barrier_timeout_ms(ctx)), [&] { return G->arrived[q] >= e; }))
      return fail(ctx, PIC_ENCCL, "loopback barrier timed out (a neighbour context stopped)");
    // the neighbour cannot re-record this event (epoch e + 2) before it passed
    // barrier e + 1, which needs this context's arrival there
    PIC_CUDA(cudaStreamWaitEvent(ctx->stream, G->ev[2 * q + (e & 1)], 0));
  }
  return PIC_OK;
}

void loopback_release(Ctx *ctx) {
  LoopGroup *G = ctx->loop;
  if (!G) return;
  ctx->loop = nullptr;
  bool last = false;
  {
    std::lock_guard<std::mutex> lk(G->mu);
    last = --G->refs == 0;
  }
  if (last) {
    for (cudaEvent_t e : G->ev)
      if (e) cudaEventDestroy(e);
    delete G;
  }
}

pic_status loopback_link(Ctx *const *ctxs, int n) {
  for (int r = 0; r < n; ++r) {
    Ctx *ctx = ctxs[r];
    PIC_CUDA(cudaMemset(ctx->peer_ctl, 0, sizeof(PeerCtl)));
  }
  {
    Ctx *ctx = ctxs[0];
    PIC_CUDA(cudaDeviceSynchronize());
  }
  LoopGroup *G = new (std::nothrow) LoopGroup();
  if (!G) return fail(ctxs[0], PIC_ENOMEM, "loopback group");
  G->n = n;
  G->refs = n;
  G->arrived.assign(n, 0ull);
  G->ev.assign(2 * n, nullptr);
  for (int k = 0; k < 2 * n; ++k) {
    Ctx *ctx = ctxs[k / 2];
    if (cudaEventCreateWithFlags(&G->ev[k], cudaEventDisableTiming) != cudaSuccess) {
      for (cudaEvent_t e : G->ev)
        if (e) cudaEventDestroy(e);
      delete G;
      return fail(ctx, PIC_ECUDA, "loopback events");
    }
  }
  for (int r = 0; r < n; ++r) {
    Ctx *ctx = ctxs[r];
    ctx->loop = G;
    const bool per = ctx->geom.periodic[0];
    const int left = (r > 0) ? r - 1 : (per ? n - 1 : -1);
    const int right = (r < n - 1) ? r + 1 : (per ? 0 : -1);
    for (int side = 0; side < 2; ++side) {
      const int nb = side == 0 ? left : right;
      ctx->loop_nb[side] = nb >= 0 ? ctxs[nb] : nullptr;
      if (nb < 0) continue;
      char *base = reinterpret_cast<char *>(ctxs[nb]->workspace);
      fill_link(ctx, side, base, describe(ctxs[nb], base), false);
    }
    ctx->peer = true;
  }
  return PIC_OK;
}

void peer_close(Ctx *ctx) {
  loopback_release(ctx);
  for (int side = 0; side < 2; ++side)
    if (ctx->link[side].mapped && ctx->link[side].owns_mapping) cudaIpcCloseMemHandle(ctx->link[side].mapped);
}

PeerOut peer_out(const Ctx *ctx, int s) {
  PeerOut po;
  for (int side = 0; side < 2; ++side) {
    const Ctx::PeerLink &L = ctx->link[side];
    po.buf[side] = L.mapped ? L.recv + (int64_t)s * MIG_REC * L.mig_cap : nullptr;
    po.cnt[side] = L.mapped ? L.cnt + s : nullptr;
    po.cap[side] = L.mapped ? L.mig_cap : 0;
  }
  return po;
}

// --------------------------------------------------------------- barrier ----
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The epoch lives in device memory (PeerCtl::epoch, advanced by this kernel
// only): every rank runs the same sequence of barriers, and a barrier captured
// in a CUDA graph (pic_set_graph) advances it on every replay.
__global__ void peer_barrier_kernel(unsigned long long *own_flag, unsigned long long *left_flag,
                                    unsigned long long *right_flag, unsigned long long *own_epoch,
                                    unsigned long long *err, unsigned long long timeout_ns) {
  const unsigned long long epoch = ++*own_epoch;
  __threadfence_system();
  if (left_flag) st_release_sys(left_flag, epoch);
  if (right_flag) st_release_sys(right_flag, epoch);
  const unsigned long long t0 = global_ns();
  // own_flag[0] is written by the left neighbour, own_flag[1] by the right one
  while ((left_flag && ld_acquire_sys(own_flag) < epoch) || (right_flag && ld_acquire_sys(own_flag + 1) < epoch)) {
    if (global_ns() - t0 > timeout_ns) {   // a neighbour is gone
      atomicAdd(err, 1ull);
      break;
    }
    __nanosleep(64);
  }
}

pic_status peer_barrier(Ctx *ctx) {
  if (ctx->loop) return loopback_barrier(ctx);
  peer_barrier_kernel<<<1, 1, 0, ctx->stream>>>(ctx->peer_ctl->flag, ctx->link[0].flag, ctx->link[1].flag,
                                                &ctx->peer_ctl->epoch, &ctx->peer_ctl->err,
                                                1000000ull * (unsigned long long)barrier_timeout_ms(ctx)); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

// -------------------------------------------------------------- arrivals ----
struct ArriveArgs {
  Geom g;
  double *a[PIC_MAX_SPECIES][7];
  int64_t *id[PIC_MAX_SPECIES];
  uint32_t *key_new[PIC_MAX_SPECIES], *rank[PIC_MAX_SPECIES], *cell_count[PIC_MAX_SPECIES];
  int64_t *d_nraw[PIC_MAX_SPECIES];
  int64_t cap[PIC_MAX_SPECIES];
  const double *recv[2];           // own receive records, [from][species][MIG_REC * rcap]
  int64_t rcap;
  unsigned long long *rcnt[2];     // their counts, [from][species]
  // far-flyers not owned here go on (hop < far_hops) into the neighbour's
  // forward region of this hop's parity; after the last hop they are dropped
  int forward;
  double *fwd[2];                  // neighbour's region from me, [side][species][MIG_REC * fcap]
  unsigned long long *fcnt[2];     // its counts, [side][species]
  int64_t fcap;
  unsigned long long *stats;
  int s0;
};

// blockIdx.y = species - s0.  Arrival i < n_from_left comes from the left
// buffer, the rest from the right one; appended at d_nraw + i and ranked into
// the cell counts as an arrival (order.cu).  Records whose position is not in
// this slab (they crossed more than one slab) are forwarded in their direction
// or counted as far-flyers (R22).
__global__ void arrive_kernel(const ArriveArgs A) {
  const int s = A.s0 + blockIdx.y;
  const int64_t c0 = min((int64_t)A.rcnt[0][s], A.rcap), c1 = min((int64_t)A.rcnt[1][s], A.rcap);
  const int64_t n = c0 + c1, base = *A.d_nraw[s];
  const Geom &g = A.g;
  const unsigned lane = threadIdx.x & 31u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w0 = (int64_t)blockIdx.x * blockDim.x; w0 < n; w0 += stride) {
    const int64_t i = w0 + threadIdx.x;
    uint32_t k = KEY_DEAD;
    const int64_t at = base + i;
    const bool act = i < n;
    int fwd_side = -1;
    double v[7];
    int64_t idv = 0;
    if (act) {
      const double *rec = i < c0 ? A.recv[0] + ((int64_t)s * A.rcap + i) * MIG_REC
                                 : A.recv[1] + ((int64_t)s * A.rcap + (i - c0)) * MIG_REC;
#pragma unroll
      for (int c = 0; c < 7; ++c) v[c] = rec[c];
      idv = __double_as_longlong(rec[7]);
      const int64_t cx = (int64_t)floor(v[0]), cy = (int64_t)floor(v[1]), cz = (int64_t)floor(v[2]);
      const bool mine = cx >= g.slab_lo && cx < g.slab_hi && cy >= 0 && cy < g.ncell[1] && cz >= 0 && cz < g.ncell[2];
      if (at >= A.cap[s]) {
        atomicAdd(&A.stats[ST_OVERFLOW], 1ull);
      } else {
        if (mine) {
          k = tile_key(g, cx - g.slab_lo, cy, cz);
        } else if (A.forward && A.fwd[i < c0 ? 1 : 0]) {
          // onward in the direction of motion: a record from the left neighbour
          // moves right (and vice versa), also across the periodic seam
          fwd_side = i < c0 ? 1 : 0;
        } else {
          atomicAdd(&A.stats[ST_FAR], 1ull);
        }
#pragma unroll
        for (int c = 0; c < 7; ++c) A.a[s][c][at] = v[c];
        A.id[s][at] = idv;
        A.key_new[s][at] = k;
      }
    }
    // forwarding: one remote atomic per warp and side reserves the slots
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const unsigned mask = __ballot_sync(0xffffffffu, fwd_side == side);
      if (!mask) continue;
      const int leader = __ffs(mask) - 1;
      unsigned long long slot0 = 0;
      if ((int)lane == leader) slot0 = atomicAdd(A.fcnt[side] + s, (unsigned long long)__popc(mask));
      slot0 = __shfl_sync(0xffffffffu, slot0, leader);
      if (fwd_side == side) {
        const int64_t slot = (int64_t)slot0 + __popc(mask & ((1u << lane) - 1u));
        if (slot < A.fcap) {
          double *rec = A.fwd[side] + ((int64_t)s * A.fcap + slot) * MIG_REC;
#pragma unroll
          for (int c = 0; c < 7; ++c) rec[c] = v[c];
          rec[7] = __longlong_as_double(idv);
          __threadfence_system();
        } else {
          atomicAdd(&A.stats[ST_OVERFLOW], 1ull);
        }
      }
    }
    const bool counted = act && k < KEY_FIRST_RESERVED;
    const unsigned nrecv = __popc(__ballot_sync(0xffffffffu, counted));
    if (lane == 0 && nrecv) atomicAdd(&A.stats[ST_RECEIVED], (unsigned long long)nrecv);
    const uint32_t r = count_rank(A.cell_count[s], g.ncells, k, counted, true);
    if (counted) A.rank[s][at] = r;
  }
}

__global__ void arrive_finish_kernel(const ArriveArgs A, int S) {
  const int s = A.s0 + threadIdx.x;
  if (threadIdx.x >= S) return;
  const int64_t c0 = min((int64_t)A.rcnt[0][s], A.rcap), c1 = min((int64_t)A.rcnt[1][s], A.rcap);
  const int64_t n = c0 + c1;
  *A.d_nraw[s] = min(*A.d_nraw[s] + n, A.cap[s]);
  A.rcnt[0][s] = 0;
  A.rcnt[1][s] = 0;
}

// After the movers of species [s0, s1): barrier, append + rank the arrivals;
// with far_hops > 0 as many more rounds (barrier, then the forwarded records)
// for particles that crossed more than one slab.
pic_status peer_migrate(Ctx *ctx, int s0, int s1) {
  const int hops = ctx->cfg.far_hops;
  for (int hop = 0; hop <= hops; ++hop) {
    {
      PhaseTimer t(ctx, 4);
      pic_status st = peer_barrier(ctx);
      if (st != PIC_OK) return st;
    }
    PhaseTimer t(ctx, 5);
    ArriveArgs A;
    A.g = ctx->geom;
    for (int s = s0; s < s1; ++s) {
      SpeciesStore &sp = ctx->sp[s];
      for (int k = 0; k < 7; ++k) A.a[s][k] = sp.a[k];
      A.id[s] = sp.id;
      A.key_new[s] = sp.key_new;
      A.rank[s] = sp.rank;
      A.cell_count[s] = sp.cell_count;
      A.d_nraw[s] = sp.d_nraw;
      A.cap[s] = sp.cap;
      // the host no longer knows the live count exactly: keep an upper bound for grid sizes
      sp.n_raw = std::min<int64_t>(sp.cap, sp.n_raw + 2 * (hop == 0 ? ctx->mig_cap : ctx->fwd_cap));
    }
    if (hop == 0) {
      A.recv[0] = ctx->mig_recv[0];
      A.recv[1] = ctx->mig_recv[1];
      A.rcap = ctx->mig_cap;
      A.rcnt[0] = ctx->peer_ctl->cnt[0];
      A.rcnt[1] = ctx->peer_ctl->cnt[1];
    } else {
      const int par = (hop - 1) & 1;
      A.recv[0] = ctx->fwd_recv[par][0];
      A.recv[1] = ctx->fwd_recv[par][1];
      A.rcap = ctx->fwd_cap;
      A.rcnt[0] = ctx->peer_ctl->fcnt[par][0];
      A.rcnt[1] = ctx->peer_ctl->fcnt[par][1];
    }
    A.forward = hop < hops;
    for (int side = 0; side < 2; ++side) {
      const Ctx::PeerLink &L = ctx->link[side];
      A.fwd[side] = (A.forward && L.mapped) ? L.frecv[hop & 1] : nullptr;
      A.fcnt[side] = (A.forward && L.mapped) ? L.fcnt[hop & 1] : nullptr;
    }
    A.fcap = ctx->fwd_cap;
    A.stats = ctx->stats;
    A.s0 = s0;
    dim3 grid(kSMs, s1 - s0);
    arrive_kernel<<<grid, 256, 0, ctx->stream>>>(A); ++ctx->launches;
    arrive_finish_kernel<<<1, 32, 0, ctx->stream>>>(A, s1 - s0); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
  }
  return PIC_OK;
}

// ------------------------------------------------------------ ghost sums ----
struct PullArgs {
  double *mine[PIC_MAX_SPECIES];
  const double *theirs[PIC_MAX_SPECIES];
  int64_t face_yz, my_plane, my_nx, my_x, their_plane, their_nx, their_x;
};

// my plane x = slab_lo (array index G) += left neighbour's plane x = its slab_hi
__global__ void ghost_pull_kernel(const PullArgs A) {
  const int s = blockIdx.y;
  const int64_t total = A.face_yz * 10;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t yz = t % A.face_yz, m = t / A.face_yz;
    A.mine[s][m * A.my_plane + yz * A.my_nx + A.my_x] += A.theirs[s][m * A.their_plane + yz * A.their_nx + A.their_x];
  }
}

pic_status launch_fold_axis(Ctx *ctx, int s, int axis, int64_t x0, int64_t nxr);

pic_status peer_exchange(Ctx *ctx) {
  const Geom &g = ctx->geom;
  const int S = ctx->cfg.n_species;
  pic_status st = peer_barrier(ctx);
  if (st != PIC_OK) return st;
  const Ctx::PeerLink &L = ctx->link[0];
  if (L.mapped) {
    PullArgs A;
    for (int s = 0; s < S; ++s) {
      A.mine[s] = ctx->sp[s].mom;
      A.theirs[s] = L.mom[s];
    }
    A.face_yz = g.m_n[1] * g.m_n[2];
    A.my_plane = g.m_plane;
    A.my_nx = g.m_n[0];
    A.my_x = g.G;
    A.their_plane = L.m_plane;
    A.their_nx = L.m_nx;
    A.their_x = L.ghost_x;
    ghost_pull_kernel<<<dim3(grid_for(A.face_yz * 10), S), 256, 0, ctx->stream>>>(A); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
  }
  // periodic y / z folds over the owned x planes only
  const int64_t nloc = g.slab_hi - g.slab_lo;
  const bool last_open = !g.periodic[0] && g.slab_hi == g.ncell[0];
  for (int s = 0; s < S; ++s) {
    for (int axis = 1; axis <= 2; ++axis)
      if (g.periodic[axis]) {
        st = launch_fold_axis(ctx, s, axis, g.G, nloc + (last_open ? 1 : 0));
        if (st != PIC_OK) return st;
      }
  }
  return PIC_OK;
}

}  // namespace pic
