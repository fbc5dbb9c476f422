// sort.cu — cell sort of the particle store (not a step of
// the paper, which sorts only for coalescence).
//
// key = local cell index of the current position (written by the mover or by
// recompute_keys); CUB onesweep radix sort of (key, index) over the used key
// bits; then each of the 8 per-particle arrays is gathered through the single
// scratch array (8 B/particle of extra memory instead of a second store).
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
    dst[p] = src[idx[p]];
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
  if (n < 2) { sp.sorted = true; return PIC_OK; }
  int end_bit = 1;
  const int64_t cells = ctx->geom.k_n[0] * ctx->geom.k_n[1] * ctx->geom.k_n[2];
  while (end_bit < 32 && (int64_t(1) << end_bit) < cells + 1) ++end_bit;
  // reserved tail keys (0xFFFFFFFx) need all 32 bits; they only occur between
  // the mover and the exchange, when the sort is not called.
  iota_u32_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(sp.idx_alt, n); ++ctx->launches;
  size_t bytes = ctx->cub_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(ctx->cub_temp, bytes, sp.key, sp.key_alt, sp.idx_alt,
                                                  sp.idx, (int)n, 0, end_bit, ctx->stream);
  if (e != cudaSuccess) return fail(ctx, PIC_ECUDA, std::string("radix sort: ") + cudaGetErrorString(e));
  std::swap(sp.key, sp.key_alt);
  for (int k = 0; k < 8; ++k) {
    double *src = (k < 7) ? sp.a[k] : (double *)sp.id;
    gather_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(src, sp.idx, ctx->scratch, n); ++ctx->launches;
    if (k < 7) sp.a[k] = ctx->scratch;
    else sp.id = (int64_t *)ctx->scratch;
    ctx->scratch = src;
  }
  PIC_CUDA(cudaGetLastError());
  sp.sorted = true;
  return PIC_OK;
}

}  // namespace pic
