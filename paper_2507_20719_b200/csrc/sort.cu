// sort.cu — tile-major cell sort of the particle store (not
// a step of the paper, which sorts only for coalescence).
//
// key_new = tile-major cell key of the current position (pic_internal.cuh
// tile_key; written by the mover or recompute_keys).  CUB onesweep radix sort
// of (key_new, index) -> (key, idx) over the used key bits; each of the 8
// per-particle arrays is then gathered through the single scratch array (8 B
// per particle of extra memory instead of a second store); finally the tile
// segment starts tile_start[t] = lower_bound(key, t * TILE^3).
#include <cub/device/device_radix_sort.cuh>

#include "pic_internal.cuh"

namespace pic {

__global__ void iota_u32_kernel(uint32_t *a, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    a[p] = (uint32_t)p;
}

__global__ void gather_kernel(const double *__restrict__ src, const uint32_t *__restrict__ idx,
                              double *__restrict__ dst, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    dst[p] = src[__ldg(idx + p)];
}

__global__ void tile_start_kernel(const uint32_t *__restrict__ key, int64_t n, int64_t ntiles,
                                  uint32_t *__restrict__ start) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t target = (uint64_t)t * TILE3;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((uint64_t)key[mid] < target) lo = mid + 1; else hi = mid;
    }
    start[t] = (uint32_t)lo;
  }
}

size_t sort_temp_bytes(int64_t cap) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)cap, 0, 32);
  return bytes + 1024;
}

static unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

pic_status sort_species(Ctx *ctx, int s) {
  SpeciesStore &sp = ctx->sp[s];
  const int64_t n = sp.n;
  const int64_t ntiles = ctx->geom.ntiles;
  if (n >= 2) {
    int end_bit = 1;
    while (end_bit < 32 && (int64_t(1) << end_bit) < ntiles * TILE3) ++end_bit;
    // reserved tail keys (0xFFFFFFFD..F) only exist between the mover and the
    // exchange; the exchange recomputes the keys of every live particle.
    iota_u32_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.idx_alt, n); ++ctx->launches;
    size_t bytes = ctx->cub_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(ctx->cub_temp, bytes, sp.key_new, sp.key, sp.idx_alt,
                                                    sp.idx, (int)n, 0, end_bit, ctx->stream);
    if (e != cudaSuccess) return fail(ctx, PIC_ECUDA, std::string("radix sort: ") + cudaGetErrorString(e));
    for (int k = 0; k < 8; ++k) {
      double *src = (k < 7) ? sp.a[k] : (double *)sp.id;
      gather_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(src, sp.idx, ctx->scratch, n); ++ctx->launches;
      if (k < 7) sp.a[k] = ctx->scratch;
      else sp.id = (int64_t *)ctx->scratch;
      ctx->scratch = src;
    }
  } else if (n == 1) {
    PIC_CUDA(cudaMemcpyAsync(sp.key, sp.key_new, 4, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  tile_start_kernel<<<grid_for(ntiles + 1), 256, 0, ctx->stream>>>(sp.key, n, ntiles, sp.tile_start); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  sp.sorted = true;
  return PIC_OK;
}

}  // namespace pic
