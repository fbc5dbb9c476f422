// order.cu — cell order of the particle store by a counting sort through an
// indirection (not a step of the paper, which sorts only
// for coalescence).
//
// The mover counts every particle that stays on this rank in its new cell
// and ranks those that kept their cell (count_rank); the exchange counts
// received particles the same way.  build_order then turns the counts into
// cell offsets (exclusive scan) and scatters perm[cell_off[k] + rank] =
// position, arrivals after each cell's stayers.  The next mover gathers its
// inputs through perm and writes them in that order, so no separate
// permutation pass over the particle data is ever needed (≈ 12 B / particle of
// order metadata instead of a radix sort + gather of all arrays).  No key array is kept: a particle's cell always
// follows from its stored position.  Removed particles and slab leavers are
// not counted and so drop out of the next order.
#include <cub/device/device_scan.cuh>

#include "pic_internal.cuh"

namespace pic {

static unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > kSMs * 32) b = kSMs * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

size_t order_temp_bytes(int64_t ncells) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                (int)(ncells + 1));
  return bytes + 1024;
}

__global__ void count_kernel(const uint32_t *__restrict__ key_new, uint32_t *__restrict__ rank,
                             uint32_t *__restrict__ cell_count, int64_t ncells, int64_t from, int64_t to) {
  // grid-stride loop with whole warps (count_rank is warp-collective)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = from + (int64_t)blockIdx.x * blockDim.x; base < to; base += stride) {
    const int64_t p = base + threadIdx.x;
    const bool act = p < to;
    const uint32_t k = act ? key_new[p] : KEY_DEAD;
    const bool counted = act && k < KEY_FIRST_RESERVED;
    const uint32_t r = count_rank(cell_count, ncells, k, counted, true);
    if (counted) rank[p] = r;
  }
}

__global__ void total_kernel(const uint32_t *__restrict__ cell_count, uint32_t *__restrict__ tot, int64_t ncells) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= ncells; c += (int64_t)gridDim.x * blockDim.x)
    tot[c] = cell_count[c] + cell_count[ncells + 1 + c];
}

#ifndef PIC_PERM_UNROLL
#define PIC_PERM_UNROLL 8
#endif
constexpr int PERM_UNROLL = PIC_PERM_UNROLL;

// Stayers go to cell_off[k] + rank; arrivals after the cell's stayers, in the
// order of an atomic cursor per cell (`cursor`, zeroed after the scan).  (A
// warp-aggregated cursor atomic measured slower: its warp-collective match
// serialises the unrolled gathers.)
__global__ void perm_kernel(const uint32_t *__restrict__ key_new, const uint32_t *__restrict__ rank,
                            const uint32_t *__restrict__ cell_off, const uint32_t *__restrict__ cell_count,
                            uint32_t *__restrict__ cursor, const int64_t *__restrict__ d_nraw,
                            uint32_t *__restrict__ perm, int64_t ncells, unsigned long long *__restrict__ stats) {
  // PERM_UNROLL independent elements per thread and iteration (memory-level
  // parallelism for the dependent cell_off gather)
  const int64_t n = *d_nraw;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p0 < n; p0 += PERM_UNROLL * stride) {
    uint32_t k[PERM_UNROLL], r[PERM_UNROLL];
#pragma unroll
    for (int u = 0; u < PERM_UNROLL; ++u) {
      const int64_t p = p0 + u * stride;
      k[u] = p < n ? key_new[p] : KEY_DEAD;
      r[u] = p < n ? rank[p] : 0u;
    }
#pragma unroll
    for (int u = 0; u < PERM_UNROLL; ++u) {
      if (k[u] >= KEY_FIRST_RESERVED) continue;
      const uint32_t q =
          cell_off[k[u]] + ((r[u] & RANK_ARRIVAL) ? cell_count[k[u]] + atomicAdd(cursor + k[u], 1u) : r[u]);
      PIC_DCHECK(k[u] < ncells && q < cell_off[k[u] + 1], stats);
      perm[q] = (uint32_t)(p0 + u * stride);
    }
  }
}

pic_status zero_cell_counts(Ctx *ctx, int s) {
  PIC_CUDA(cudaMemsetAsync(ctx->sp[s].cell_count, 0, sizeof(uint32_t) * 2 * (ctx->geom.ncells + 1), ctx->stream));
  return PIC_OK;
}

pic_status count_positions(Ctx *ctx, int s, int64_t from, int64_t to) {
  SpeciesStore &sp = ctx->sp[s];
  if (to <= from) return PIC_OK;
  count_kernel<<<grid_for(to - from), 256, 0, ctx->stream>>>(sp.key_new, sp.rank, sp.cell_count,
                                                              ctx->geom.ncells, from, to); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  return PIC_OK;
}

// Exclusive scan of the counts and the perm scatter (positions [0, d_nraw)).
pic_status build_order(Ctx *ctx, int s) {
  SpeciesStore &sp = ctx->sp[s];
  const int64_t nc = ctx->geom.ncells;
  total_kernel<<<grid_for(nc + 1), 256, 0, ctx->stream>>>(sp.cell_count, sp.cell_tot, nc); ++ctx->launches;
  size_t bytes = ctx->cub_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(ctx->cub_temp, bytes, sp.cell_tot, sp.cell_off, (int)(nc + 1),
                                                ctx->stream);
  if (e != cudaSuccess) return fail(ctx, PIC_ECUDA, std::string("scan: ") + cudaGetErrorString(e));
  if (sp.n_raw > 0) {
    // the scan input is dead now: it becomes the arrivals' cursor
    PIC_CUDA(cudaMemsetAsync(sp.cell_tot, 0, sizeof(uint32_t) * (nc + 1), ctx->stream));
    perm_kernel<<<grid_for(sp.n_raw), 256, 0, ctx->stream>>>(sp.key_new, sp.rank, sp.cell_off, sp.cell_count,
                                                             sp.cell_tot, sp.d_nraw, sp.perm, nc, ctx->stats);
    ++ctx->launches;
  }
  PIC_CUDA(cudaGetLastError());
  sp.order_valid = true;
  sp.order_dirty = false;
  return PIC_OK;
}

pic_status ensure_order(Ctx *ctx, int s) {
  return ctx->sp[s].order_dirty ? build_order(ctx, s) : PIC_OK;
}

}  // namespace pic
