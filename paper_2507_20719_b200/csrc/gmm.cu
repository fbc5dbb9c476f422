// gmm.cu — NEXT-4: physics-aware compression of the velocity distribution
// (PAPER.md:366-379): 3-D velocity binning of a species on this rank, then a
// Gaussian-mixture fit of the histogram by EM (readings R32, R33).
//
// bin_kernel: grid-stride over the live particles; per-CTA histogram in
// shared memory (B <= 24, fp64 shared atomics), merged with global atomics.
// em_kernel: a cluster of EM_CLUSTER CTAs of 256 threads runs the whole fit.
// Every CTA computes the weighted moments and the heaviest-bin +
// farthest-point seeding (deterministic argmax, lowest index on ties) itself;
// in each of the n_em EM iterations the CTAs split the bins, reduce their
// per-thread partial sums in a fixed order (warp shuffles, then warp partials
// summed by one thread each), and every CTA adds the CTAs' partials in rank
// order through distributed shared memory, so all hold the same parameters.
#include <cooperative_groups.h>

#include "pic_internal.cuh"

namespace pic {
namespace cg = cooperative_groups;

constexpr int GMM_BMAX_SMEM = 24;   // shared-memory histogram up to 24^3 bins
constexpr int GMM_BMAX = 64;        // histogram buffer in the workspace: 64^3
constexpr int GMM_MMAX = 8;         // components (per-thread accumulators in registers)
constexpr int EM_THREADS = 256;
constexpr int EM_CLUSTER = 8;       // CTAs (SMs) per fit (portable cluster size)

struct BinArgs {
  const double *u, *v, *w, *q;
  const uint32_t *perm, *nlive;
  int B;
  double vmax;
  double *hist;                    // [B^3] global
  unsigned long long *clipped;
};

__device__ __forceinline__ int vbin(double vel, double vmax, int B, bool &clip) {
  double t = floor((vel + vmax) / (2.0 * vmax) * (double)B);
  if (t < 0.0) { t = 0.0; clip = true; }
  if (t > (double)(B - 1)) { t = (double)(B - 1); clip = true; }
  return (int)t;
}

__global__ void bin_kernel(const BinArgs A) {
  extern __shared__ double sh[];
  const int nb = A.B * A.B * A.B;
  const bool priv = A.B <= GMM_BMAX_SMEM;
  if (priv)
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0.0;
  __syncthreads();
  const int64_t n = *A.nlive;
  unsigned long long clips = 0;
  for (int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; qi < n; qi += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = A.perm[qi];
    bool clip = false;
    const int bx = vbin(A.u[p], A.vmax, A.B, clip), by = vbin(A.v[p], A.vmax, A.B, clip),
              bz = vbin(A.w[p], A.vmax, A.B, clip);
    clips += clip ? 1ull : 0ull;
    const int b = (bz * A.B + by) * A.B + bx;
    const double wgt = fabs(A.q[p]);
    if (priv) atomicAdd(sh + b, wgt);
    else atomicAdd(A.hist + b, wgt);
  }
  if (clips) atomicAdd(A.clipped, clips);
  __syncthreads();
  if (priv)
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (sh[i] != 0.0) atomicAdd(A.hist + i, sh[i]);
}

// ------------------------------------------------------------------ EM ----
struct EmArgs {
  const double *hist;
  int B, M, n_em;
  double vmax;
  double *alpha, *mu, *sigma;      // [M], [M][3], [M][6] (device)
  int *status;                     // 0 ok, -1 too few occupied bins
};

// Block sum of K values per thread (fixed order): shuffles within warps, then
// thread k sums the warps' partials for value k.  out[k] valid for all threads.
template <int K>
__device__ void block_sum(double (&v)[K], double *scratch /* [EM_THREADS / 32][K] */, double *out /* [K] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[warp * K + k] = v[k];
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < EM_THREADS / 32; ++w) s += scratch[w * K + k];
    out[k] = s;
  }
  __syncthreads();
}

// Block argmax of (value, index): largest value, lowest index on ties.
__device__ void block_argmax(double val, int64_t idx, double *sv, int64_t *si, double *bv, int64_t *bi) {
  sv[threadIdx.x] = val;
  si[threadIdx.x] = idx;
  __syncthreads();
  for (int s = EM_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double a = sv[threadIdx.x], b = sv[threadIdx.x + s];
      const int64_t ia = si[threadIdx.x], ib = si[threadIdx.x + s];
      if (b > a || (b == a && ib < ia)) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  *bv = sv[0];
  *bi = si[0];
  __syncthreads();
}

// MM: the number of components (a template parameter, so that the per-thread
// accumulators of the EM loop are exactly M x 10 registers)
template <int MM>
__global__ void __launch_bounds__(EM_THREADS) em_kernel(const EmArgs A) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  __shared__ double part[2][MM * 10];            // this CTA's partial sums, by iteration parity
  __shared__ double s_alpha[MM], s_mu[MM][3], s_sig[MM][6];
  __shared__ double scratch[(EM_THREADS / 32) * GMM_MMAX * 10];
  __shared__ double red[GMM_MMAX * 10];
  __shared__ double sv[EM_THREADS];
  __shared__ int64_t si[EM_THREADS];
  __shared__ double par_inv[GMM_MMAX][6], par_nrm[GMM_MMAX];
  __shared__ double smu[GMM_MMAX][3];
  const int B = A.B, M = MM;
  const int64_t nb = (int64_t)B * B * B;
  const double bw = 2.0 * A.vmax / (double)B, eps = 1e-6 * bw * bw;
  const double two_pi3 = pow(2.0 * 3.14159265358979323846, 1.5);
  auto centre = [&](int64_t b, int d) {
    const int64_t c = d == 0 ? b % B : (d == 1 ? (b / B) % B : b / ((int64_t)B * B));
    return -A.vmax + ((double)c + 0.5) * bw;
  };
  // weighted moments: W, first moments, occupied count
  {
    double v[5] = {0, 0, 0, 0, 0};
    for (int64_t b = threadIdx.x; b < nb; b += EM_THREADS) {
      const double h = A.hist[b];
      if (h > 0.0) {
        v[0] += h;
        for (int d = 0; d < 3; ++d) v[1 + d] += h * centre(b, d);
        v[4] += 1.0;
      }
    }
    block_sum<5>(v, scratch, red);
  }
  const double W = red[0];
  const double m1[3] = {red[1] / W, red[2] / W, red[3] / W};
  if (red[4] < (double)M) {
    if (threadIdx.x == 0) *A.status = -1;
    return;
  }
  __syncthreads();
  double cov[6];
  {
    const int ia[6] = {0, 0, 0, 1, 1, 2}, ib[6] = {0, 1, 2, 1, 2, 2};
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t b = threadIdx.x; b < nb; b += EM_THREADS) {
      const double h = A.hist[b];
      if (h > 0.0)
        for (int k = 0; k < 6; ++k) v[k] += h * (centre(b, ia[k]) - m1[ia[k]]) * (centre(b, ib[k]) - m1[ib[k]]);
    }
    block_sum<6>(v, scratch, red);
    for (int k = 0; k < 6; ++k) cov[k] = red[k] / W;
    cov[0] += eps; cov[3] += eps; cov[5] += eps;
  }
  // seeding: heaviest bin, then farthest points
  {
    double best = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t b = threadIdx.x; b < nb; b += EM_THREADS) {
      const double h = A.hist[b];
      if (h > 0.0 && (h > best || (h == best && b < bi))) { best = h; bi = b; }
    }
    double bv;
    int64_t idx;
    block_argmax(best, bi, sv, si, &bv, &idx);
    if (threadIdx.x == 0)
      for (int d = 0; d < 3; ++d) smu[0][d] = centre(idx, d);
    __syncthreads();
    for (int i = 1; i < M; ++i) {
      double far = -1.0;
      int64_t fi = INT64_MAX;
      for (int64_t b = threadIdx.x; b < nb; b += EM_THREADS) {
        if (!(A.hist[b] > 0.0)) continue;
        double dmin = INFINITY;
        for (int j = 0; j < i; ++j) {
          double dd = 0.0;
          for (int d = 0; d < 3; ++d) {
            const double t = centre(b, d) - smu[j][d];
            dd += t * t;
          }
          dmin = fmin(dmin, dd);
        }
        if (dmin > far || (dmin == far && b < fi)) { far = dmin; fi = b; }
      }
      block_argmax(far, fi, sv, si, &bv, &idx);
      if (threadIdx.x == 0)
        for (int d = 0; d < 3; ++d) smu[i][d] = centre(idx, d);
      __syncthreads();
    }
  }
  if (threadIdx.x < M) {
    s_alpha[threadIdx.x] = 1.0 / (double)M;
    for (int d = 0; d < 3; ++d) s_mu[threadIdx.x][d] = smu[threadIdx.x][d];
    for (int k = 0; k < 6; ++k) s_sig[threadIdx.x][k] = cov[k];
  }
  __syncthreads();
  const int ia[6] = {0, 0, 0, 1, 1, 2}, ib[6] = {0, 1, 2, 1, 2, 2};
  for (int it = 0; it < A.n_em; ++it) {
    if (threadIdx.x < M) {
      const double *S = s_sig[threadIdx.x];
      const double a = S[0], b = S[1], c = S[2], d = S[3], e = S[4], f = S[5];
      const double iA = d * f - e * e, iB = -(b * f - c * e), iC = b * e - c * d;
      const double iD = a * f - c * c, iE = -(a * e - b * c), iF = a * d - b * b;
      const double det = a * iA + b * iB + c * iC;
      double *o = par_inv[threadIdx.x];
      o[0] = iA / det; o[1] = iB / det; o[2] = iC / det; o[3] = iD / det; o[4] = iE / det; o[5] = iF / det;
      par_nrm[threadIdx.x] = s_alpha[threadIdx.x] / (two_pi3 * sqrt(det));
      for (int dd = 0; dd < 3; ++dd) smu[threadIdx.x][dd] = s_mu[threadIdx.x][dd];
    }
    __syncthreads();
    double acc[MM * 10];
#pragma unroll
    for (int k = 0; k < MM * 10; ++k) acc[k] = 0.0;
    // this thread's bins b = b0 + j S (S = all threads of the cluster), their
    // (ix, iy, iz) advanced incrementally (no 64-bit division per bin)
    constexpr int S = EM_THREADS * EM_CLUSTER;
    const int b0 = rank * EM_THREADS + (int)threadIdx.x;
    const int dX = S % B, dY = (S / B) % B, dZ = S / (B * B);
    int ix = b0 % B, iy = (b0 / B) % B, iz = b0 / (B * B);
    for (int64_t bb = b0; bb < nb; bb += S) {
      const double h = A.hist[bb];
      const double cx = -A.vmax + ((double)ix + 0.5) * bw, cy = -A.vmax + ((double)iy + 0.5) * bw,
                   cz = -A.vmax + ((double)iz + 0.5) * bw;
      ix += dX;
      if (ix >= B) { ix -= B; ++iy; }
      iy += dY;
      if (iy >= B) { iy -= B; ++iz; }
      iz += dZ;
      if (!(h > 0.0)) continue;
      double r[MM], tot = 0.0;
#pragma unroll
      for (int i = 0; i < MM; ++i) {
        const double x = cx - smu[i][0], y = cy - smu[i][1], z = cz - smu[i][2];
        const double *Q = par_inv[i];
        const double q2 = Q[0] * x * x + Q[3] * y * y + Q[5] * z * z + 2.0 * (Q[1] * x * y + Q[2] * x * z + Q[4] * y * z);
        r[i] = par_nrm[i] * exp(-0.5 * q2);
        tot += r[i];
      }
      if (!(tot > 0.0)) continue;
      const double cc[3] = {cx, cy, cz};
#pragma unroll
      for (int i = 0; i < MM; ++i) {
        const double wr = h * (r[i] / tot);
        double *a = acc + 10 * i;
        a[0] += wr;
#pragma unroll
        for (int d = 0; d < 3; ++d) a[1 + d] += wr * cc[d];
#pragma unroll
        for (int k = 0; k < 6; ++k) a[4 + k] += wr * cc[ia[k]] * cc[ib[k]];
      }
    }
    block_sum<MM * 10>(acc, scratch, red);
    // the cluster's sum of the CTAs' partials, in rank order, in every CTA
    double *mine = part[it & 1];
    if (threadIdx.x < MM * 10) mine[threadIdx.x] = red[threadIdx.x];
    cluster.sync();
    if (threadIdx.x < MM * 10) {
      double t = 0.0;
      for (int r = 0; r < EM_CLUSTER; ++r) t += cluster.map_shared_rank(mine, r)[threadIdx.x];
      red[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x < M) {
      const double *a = red + 10 * threadIdx.x;
      if (a[0] > 0.0) {
        const int i = threadIdx.x;
        s_alpha[i] = a[0] / W;
        for (int d = 0; d < 3; ++d) s_mu[i][d] = a[1 + d] / a[0];
        for (int k = 0; k < 6; ++k)
          s_sig[i][k] = a[4 + k] / a[0] - s_mu[i][ia[k]] * s_mu[i][ib[k]] + ((ia[k] == ib[k]) ? eps : 0.0);
      }
    }
    __syncthreads();
  }
  if (rank == 0 && threadIdx.x < M) {
    const int i = threadIdx.x;
    A.alpha[i] = s_alpha[i];
    for (int d = 0; d < 3; ++d) A.mu[3 * i + d] = s_mu[i][d];
    for (int k = 0; k < 6; ++k) A.sigma[6 * i + k] = s_sig[i][k];
  }
  if (rank == 0 && threadIdx.x == 0) *A.status = 0;
  cluster.sync();   // no CTA leaves while another may still read its partials
}

pic_status gmm_fit(Ctx *ctx, int s, int B, double vmax, int M, int n_em, double *alpha, double *mu, double *sigma,
                   double *hist_out, int64_t *clipped) {
  if (B < 1 || B > GMM_BMAX || !(vmax > 0.0) || M < 1 || M > GMM_MMAX || n_em < 0)
    return fail(ctx, PIC_EINVAL, "pic_gmm: 1 <= B <= 64, vmax > 0, 1 <= M <= 8, n_em >= 0");
  SpeciesStore &sp = ctx->sp[s];
  const int64_t nb = (int64_t)B * B * B;
  double *hist = ctx->gmm_buf;                       // [64^3] + params
  double *par = hist + (int64_t)GMM_BMAX * GMM_BMAX * GMM_BMAX;
  unsigned long long *clip = reinterpret_cast<unsigned long long *>(ctx->dev_counts + 61);
  int *status = reinterpret_cast<int *>(ctx->dev_counts + 62);
  PIC_CUDA(cudaMemsetAsync(hist, 0, sizeof(double) * nb, ctx->stream));
  PIC_CUDA(cudaMemsetAsync(clip, 0, sizeof(unsigned long long), ctx->stream));
  BinArgs Bn;
  Bn.u = sp.a[3]; Bn.v = sp.a[4]; Bn.w = sp.a[5]; Bn.q = sp.a[6];
  Bn.perm = sp.perm;
  Bn.nlive = sp.cell_off + ctx->geom.ncells;
  Bn.B = B;
  Bn.vmax = vmax;
  Bn.hist = hist;
  Bn.clipped = clip;
  const size_t smem = B <= GMM_BMAX_SMEM ? sizeof(double) * nb : 0;
  PIC_CUDA(cudaFuncSetAttribute(bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(double) * GMM_BMAX_SMEM * GMM_BMAX_SMEM * GMM_BMAX_SMEM)));
  bin_kernel<<<kSMs * 2, 256, smem, ctx->stream>>>(Bn); ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  EmArgs E;
  E.hist = hist;
  E.B = B;
  E.M = M;
  E.n_em = n_em;
  E.vmax = vmax;
  E.alpha = par;
  E.mu = par + GMM_MMAX;
  E.sigma = par + 4 * GMM_MMAX;
  E.status = status;
  {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(EM_CLUSTER);
    lc.blockDim = dim3(EM_THREADS);
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = EM_CLUSTER;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    switch (M) {
      case 1: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<1>, E)); break;
      case 2: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<2>, E)); break;
      case 3: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<3>, E)); break;
      case 4: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<4>, E)); break;
      case 5: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<5>, E)); break;
      case 6: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<6>, E)); break;
      case 7: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<7>, E)); break;
      default: PIC_CUDA(cudaLaunchKernelEx(&lc, em_kernel<8>, E)); break;
    }
  }
  ++ctx->launches;
  PIC_CUDA(cudaGetLastError());
  int st_h = 0;
  unsigned long long clip_h = 0;
  PIC_CUDA(cudaMemcpyAsync(&st_h, status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  PIC_CUDA(cudaMemcpyAsync(&clip_h, clip, sizeof(clip_h), cudaMemcpyDeviceToHost, ctx->stream));
  if (alpha) PIC_CUDA(cudaMemcpyAsync(alpha, E.alpha, sizeof(double) * M, cudaMemcpyDefault, ctx->stream));
  if (mu) PIC_CUDA(cudaMemcpyAsync(mu, E.mu, sizeof(double) * 3 * M, cudaMemcpyDefault, ctx->stream));
  if (sigma) PIC_CUDA(cudaMemcpyAsync(sigma, E.sigma, sizeof(double) * 6 * M, cudaMemcpyDefault, ctx->stream));
  if (hist_out) PIC_CUDA(cudaMemcpyAsync(hist_out, hist, sizeof(double) * nb, cudaMemcpyDefault, ctx->stream));
  PIC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (clipped) *clipped = (int64_t)clip_h;
  if (st_h != 0) return fail(ctx, PIC_EINVAL, "pic_gmm: fewer occupied bins than components");
  return PIC_OK;
}

}  // namespace pic
