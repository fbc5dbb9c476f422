// Shared-memory wavefronts per cp.async (LDGSTS) for the mover's source ring
// (ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ldgsts.sum... see the
// command in DESIGN.md §11).  Each warp copies 8-byte elements to 32
// consecutive doubles of shared memory from: PAT 0 32 consecutive aligned
// elements, 1 consecutive starting one element off a 128-B line, 2 with a gap
// every 8 elements, 3 a random permutation within 64 elements, 4 fully random;
// W = 16: 16-byte copies of consecutive aligned pairs (16 lanes).
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 256;

template <int PAT, int W>
__global__ void ldgsts_pattern(const double *__restrict__ src, double *out, uint32_t n) {
  __shared__ __align__(128) double ring[8][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t base = ((blockIdx.x * 8 + warp) * ITERS + it) * 64u % (n - 4096);
    uint32_t e;
    if (PAT == 0) e = base + lane;
    if (PAT == 1) e = base + 1 + lane;
    if (PAT == 2) e = base + lane + lane / 8;
    if (PAT == 3) e = base + ((lane * 37 + it) & 63);
    if (PAT == 4) e = (base * 2654435761u + lane * 40503u) % (n - 64);
    double *d = &ring[warp][it & 1][lane];
    if (W == 8) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
                   "l"(src + e) : "memory");
    } else if (lane < 16) {
      double *d2 = &ring[warp][it & 1][2 * lane];
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d2)),
                   "l"(src + (base & ~1u) + 2 * lane) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    acc += ring[warp][it & 1][lane];
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const uint32_t n = 1u << 26;
  double *src, *out;
  cudaMalloc(&src, sizeof(double) * n);
  cudaMemset(src, 0, sizeof(double) * n);
  cudaMalloc(&out, sizeof(double) * 148 * 256);
  ldgsts_pattern<0, 8><<<148, 256>>>(src, out, n);
  ldgsts_pattern<1, 8><<<148, 256>>>(src, out, n);
  ldgsts_pattern<2, 8><<<148, 256>>>(src, out, n);
  ldgsts_pattern<3, 8><<<148, 256>>>(src, out, n);
  ldgsts_pattern<4, 8><<<148, 256>>>(src, out, n);
  ldgsts_pattern<0, 16><<<148, 256>>>(src, out, n);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
