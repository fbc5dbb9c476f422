// Shared-memory wavefronts per LDS for the address patterns of the mover's
// gather (run under ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum
// / smsp__inst_executed_op_shared_ld.sum per kernel;
// profiles/r02_microbench_lds_wavefronts.json).  Measured on B200: a full-warp
// LDS.128 takes 2 wavefronts when every aligned group of 4 lanes reads
// addresses of the form [a a a a], [a b a b] or [a a b b] (one cell, cells in
// 4-lane blocks, alternating lanes), and 4 as soon as one group does not
// ([a b a a]: a single lane in another cell), +1 per bank conflict; with the active lanes in
// one half-warp 1 (in both halves 2); 32 distinct addresses 4.  An LDS.64 costs the same
// wavefronts as an LDS.128 (twice per byte).  DESIGN.md §11.
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 1024;

__device__ __forceinline__ int node_of(int pat, int lane) {
  switch (pat) {
    case 0: return 100;                                    // one cell
    case 1: return 100 + (lane >> 4);                      // two x-neighbour cells, 16 + 16 lanes
    case 2: return 100 + (lane >> 3);                      // four x-neighbour nodes, 8 lanes each
    case 3: return 100 + 7 * (lane >> 4);                  // y-neighbours
    case 4: return 100 + 49 * (lane >> 4);                 // z-neighbours
    case 5: return lane;                                   // 32 distinct nodes
    case 6: return 100 + (lane >= 28);
    case 7: return 100 + (lane == 5);                      // one lane in the x-neighbour cell
    case 8: return 100 + (lane == 5 || lane == 21);
    case 9: return 100 + 8 * (lane == 5);                  // xy-diagonal (same banks)
    case 10: return 100 + (lane & 1);                      // alternating lanes
    case 11: return 100 + (lane == 3) + 7 * (lane == 12) + 49 * (lane == 25);
    case 12: return 100 + 7 * (lane == 5);
    case 13: return 100 + (lane == 5) + (lane == 6);
    case 14: return 100 + (lane == 31);
    case 15: return 100 + (lane == 0);
    case 16: return 100 + (lane < 4);
    case 17: return 100 + (lane >= 24 && lane < 28);
    case 18: return 100 + (lane >= 8 && lane < 16);
    case 19: return 100 + (lane >= 4 && lane < 8);
    case 20: return 100 + (lane < 8);
    case 21: return 100 + (lane == 5) * 2;
    case 22: return 100 + ((lane & 3) == 1);
    case 23: return 100 + ((lane & 7) == 5);
    case 24: return 100 + (lane == 5 || lane == 7);        // a lane and its i ^ 2 partner
    case 25: return 100 + (lane & 2) / 2;                  // i and i ^ 2 always differ
  }
  return 100;
}

// PRED: which lanes issue the loads (0 all; 1 lane 5 only; 2 lanes 5, 21; 3 lanes 5, 7;
// 4 lanes 5, 12, 21, 30; 5 lanes 0..15)
__device__ __forceinline__ bool active(int pred, int lane) {
  switch (pred) {
    case 1: return lane == 5;
    case 2: return lane == 5 || lane == 21;
    case 3: return lane == 5 || lane == 7;
    case 4: return lane == 5 || lane == 12 || lane == 21 || lane == 30;
    case 5: return lane < 16;
  }
  return true;
}

template <int PAT, int PRED, int W>
__global__ void lds_pattern(double *out, int salt) {
  __shared__ __align__(128) double box[7 * 7 * 7 * 6];
  for (int i = threadIdx.x; i < 7 * 7 * 7 * 6; i += blockDim.x) box[i] = i * 0.5 + salt;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int node = node_of(PAT, lane) + (PRED ? 7 * (lane & 1) : 0);  // predicated lanes: distinct cells
  double acc = 0.0;
  if (active(PRED, lane)) {
    for (int it = 0; it < ITERS; ++it) {
      const double *p = box + 6 * ((node + it) % 200);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double *q = p + 6 * (c & 1) + 42 * ((c >> 1) & 1) + 2 * (c >> 2);
        if (W == 16) {
          const double2 v = *reinterpret_cast<const double2 *>(q);
          acc += v.x * v.y;
        } else {
          acc += q[0] * q[1];
        }
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

#define RUN(P, R, W) lds_pattern<P, R, W><<<148, 256>>>(out, 1)
int main() {
  double *out;
  cudaMalloc(&out, sizeof(double) * 148 * 256);
  RUN(0, 0, 16); RUN(1, 0, 16); RUN(2, 0, 16); RUN(3, 0, 16); RUN(4, 0, 16); RUN(5, 0, 16);
  RUN(6, 0, 16); RUN(7, 0, 16); RUN(8, 0, 16); RUN(9, 0, 16); RUN(10, 0, 16); RUN(11, 0, 16);
  RUN(12, 0, 16); RUN(13, 0, 16); RUN(14, 0, 16); RUN(15, 0, 16); RUN(16, 0, 16); RUN(17, 0, 16);
  RUN(18, 0, 16); RUN(19, 0, 16); RUN(20, 0, 16); RUN(21, 0, 16); RUN(22, 0, 16); RUN(23, 0, 16);
  RUN(24, 0, 16); RUN(25, 0, 16);
  RUN(0, 1, 16); RUN(0, 2, 16); RUN(0, 3, 16); RUN(0, 4, 16); RUN(0, 5, 16);
  RUN(0, 0, 8); RUN(7, 0, 8); RUN(10, 0, 8); RUN(5, 0, 8); RUN(0, 1, 8); RUN(0, 4, 8);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
