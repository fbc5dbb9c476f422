// control.cu — NEXT-3 particle control (readings R29-R31,
// DESIGN.md §3): the per-domain monitor, splitting and pair-wise coalescence.
//
// Splitting: one thread per live particle (cell order); Philox draws keyed by
// the particle id decide and orient the split; the second child is appended
// and ranked as an arrival (the order is rebuilt afterwards).  Coalescence:
// one CTA per tile, one warp per cell at a time; the cell's particles are
// bitonic-sorted in shared memory by (velocity bins, id), the warp picks the
// pairs (the definition's sequential scan, 32 records at a time), the lanes merge them (the keeper is written in place, the partner's
// key becomes KEY_DEAD) and the order is recounted.
#include "pic_internal.cuh"

namespace pic {

__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
__device__ __forceinline__ double unif53(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ int64_t child_id(int64_t parent, int64_t cycle) {
  uint64_t z = (uint64_t)parent ^ ((uint64_t)cycle << 48) ^ 0x5BD1E995ull;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (int64_t)((z & ((1ull << 61) - 1)) | (1ull << 61));
}

struct SplitArgs {
  Geom g;
  double *a[7];
  int64_t *id;
  const uint32_t *perm, *nlive;
  uint32_t *key_new, *rank, *cell_count;
  int64_t *d_nraw;
  int64_t cap;
  unsigned long long *stats;
  double p_split, eps;
  uint32_t seed_lo, seed_hi, cycle, species;
};

__global__ void __launch_bounds__(256) split_kernel(const SplitArgs A) {
  const int64_t n = *A.nlive;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((int64_t)blockIdx.x * blockDim.x >= n) return;   // whole warps leave together
  int64_t slot = -1;
  uint32_t k = KEY_DEAD;
  if (q < n) {
    const uint32_t p = A.perm[q];
    const uint64_t uid = (uint64_t)A.id[p];
    double r[6];
#pragma unroll
    for (int call = 0; call < 3; ++call) {
      uint32_t c[4] = {(uint32_t)uid, (uint32_t)(uid >> 32), A.cycle, (A.species << 8) | (0x80u + call)};
      philox10(c, A.seed_lo, A.seed_hi);
      r[2 * call] = unif53(c[0], c[1]);
      r[2 * call + 1] = unif53(c[2], c[3]);
    }
    if (r[0] < A.p_split) {
      const double two_pi = 2.0 * 3.14159265358979323846;
      const double rad1 = sqrt(-2.0 * log(1.0 - r[1])), rad2 = sqrt(-2.0 * log(1.0 - r[3]));
      const double nv[3] = {rad1 * cos(two_pi * r[2]), rad1 * sin(two_pi * r[2]), rad2 * cos(two_pi * r[4])};
      const double nrm = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
      if (nrm > 0.0) {
        // positions are in cell units: the displacement eps Delta_d e_d is eps e_d
        double lo[3], hi[3];
        bool ok = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double x = A.a[d][p], dd = A.eps * (nv[d] / nrm);
          lo[d] = x - dd;
          hi[d] = x + dd;
          const double c0 = floor(x);
          ok &= floor(lo[d]) == c0 && floor(hi[d]) == c0;
        }
        if (ok) {
          slot = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(A.d_nraw), 1ull);
          if (slot >= A.cap) {
            atomicAdd(&A.stats[ST_OVERFLOW], 1ull);
            slot = -1;
          } else {
            const double qh = A.a[6][p] * 0.5;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              A.a[d][slot] = hi[d];
              A.a[3 + d][slot] = A.a[3 + d][p];
              A.a[d][p] = lo[d];
            }
            A.a[6][slot] = qh;
            A.a[6][p] = qh;
            A.id[slot] = child_id((int64_t)uid, A.cycle);
            k = A.key_new[p];   // the parent's cell (key of its store position)
            A.key_new[slot] = k;
          }
        }
      }
    }
  }
  const bool counted = slot >= 0;
  const uint32_t rk = count_rank(A.cell_count, A.g.ncells, k, counted, true);
  if (counted) A.rank[slot] = rk;
}

// ---------------------------------------------------------- coalescence ----
// Every cell with >= 2 particles is coalesced (R31: "in cells
// with an excessive number of particles, we perform pair-wise merging").  Two
// paths reach the same sorted order (velocity bins, then id) and the same pairs:
//  * coalesce_kernel: a warp per cell, for cells of 2..COAL_MAX particles whose
//    bins fit the packed 63-bit key (|bin| < 2^20): bitonic sort in shared memory;
//  * coalesce_big_kernel: every other cell (overfull, or a bin beyond the
//    packed range), listed by the first kernel: a CTA per cell sorts the
//    unpacked keys (bins as fp64, id) in global scratch (the free B buffers of
//    the store) with a bitonic network of ascending compare-exchanges, which
//    handles any cell size.
constexpr int COAL_MAX = 512;        // shared-memory path: particles per cell
constexpr int COAL_WARPS = 8;
constexpr int64_t COAL_BIN_LIM = 1 << 20;   // |velocity bin| bound of the packed key
// per warp: packed bin key, id, particle index in the cell, pair list
constexpr size_t COAL_WARP_BYTES = COAL_MAX * (8 + 8 + 4) + (COAL_MAX / 2) * 4;
constexpr size_t COAL_SMEM = COAL_WARP_BYTES * COAL_WARPS;

struct CoalArgs {
  Geom g;
  double *a[7];
  const int64_t *id;
  const uint32_t *perm, *cell_off;
  uint32_t *key_new;
  double dv, frac;
  unsigned long long *merges;
  // cells for coalesce_big_kernel: list[2 e] = cell, list[2 e + 1] = scratch offset
  unsigned long long *n_big, *big_used;
  int64_t *big_list;
  int64_t cap;
  unsigned long long *stats;
};

// Global scratch of coalesce_big_kernel, one record per particle of a listed
// cell at [offset, offset + n_c): the sort keys and the particle position.
struct CoalBig {
  double *bx, *by, *bz;
  int64_t *id;
  uint32_t *idx;
  int32_t *pairs;
};

// (bx, by, bz) packed into 63 bits, bx most significant (lexicographic order)
__device__ __forceinline__ uint64_t pack_bins(int64_t bx, int64_t by, int64_t bz) {
  return ((uint64_t)(bx + COAL_BIN_LIM) << 42) | ((uint64_t)(by + COAL_BIN_LIM) << 21) | (uint64_t)(bz + COAL_BIN_LIM);
}


// Bitonic sort of N <= 256 records (key, id, index) held in registers, element
// i = lane + 32 r in slot r: the stages with j >= 32 compare two slots of the
// same lane, the others exchange with lane ^ j by shuffles.  Same network and
// comparisons as the shared-memory sort, so the same order.
constexpr int COAL_RREG = 8;
__device__ __forceinline__ void cx_slots(uint64_t (&k)[COAL_RREG], int64_t (&d)[COAL_RREG], int (&x)[COAL_RREG],
                                         int a, int b, bool up) {
  const bool b_less = k[b] < k[a] || (k[b] == k[a] && d[b] < d[a]);
  if (b_less == up) {
    const uint64_t tk = k[a]; k[a] = k[b]; k[b] = tk;
    const int64_t td = d[a]; d[a] = d[b]; d[b] = td;
    const int tx = x[a]; x[a] = x[b]; x[b] = tx;
  }
}
__device__ __forceinline__ void warp_sort_regs(uint64_t *key, int64_t *ids, int32_t *ix, int N, int lane) {
  uint64_t k[COAL_RREG];
  int64_t d[COAL_RREG];
  int x[COAL_RREG];
#pragma unroll
  for (int r = 0; r < COAL_RREG; ++r) {
    const int i = lane + 32 * r;
    const bool in = i < N;
    k[r] = in ? key[i] : ~0ull;
    d[r] = in ? ids[i] : INT64_MAX;
    x[r] = in ? ix[i] : -1;
  }
  for (int kk = 2; kk <= N; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int js = j >> 5;   // slot distance 1, 2 or 4
#pragma unroll
        for (int r = 0; r < COAL_RREG; ++r) {
          const bool up = ((lane + 32 * r) & kk) == 0;
          if (js == 1 && !(r & 1)) cx_slots(k, d, x, r, r + 1 < COAL_RREG ? r + 1 : r, up);
          if (js == 2 && !(r & 2)) cx_slots(k, d, x, r, r + 2 < COAL_RREG ? r + 2 : r, up);
          if (js == 4 && !(r & 4)) cx_slots(k, d, x, r, r + 4 < COAL_RREG ? r + 4 : r, up);
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < COAL_RREG; ++r) {
          const bool up = ((lane + 32 * r) & kk) == 0;
          const uint64_t pk = __shfl_xor_sync(0xffffffffu, k[r], j);
          const int64_t pd = __shfl_xor_sync(0xffffffffu, d[r], j);
          const int px = __shfl_xor_sync(0xffffffffu, x[r], j);
          const bool p_less = pk < k[r] || (pk == k[r] && pd < d[r]);
          if (p_less == (lower == up)) {
            k[r] = pk;
            d[r] = pd;
            x[r] = px;
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < COAL_RREG; ++r) {
    const int i = lane + 32 * r;
    if (i < N) {
      key[i] = k[r];
      ix[i] = x[r];
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * COAL_WARPS) coalesce_kernel(const CoalArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *base = smem_raw + warp * COAL_WARP_BYTES;
  uint64_t *key = reinterpret_cast<uint64_t *>(base);
  int64_t *ids = reinterpret_cast<int64_t *>(base + COAL_MAX * 8);
  int32_t *ix = reinterpret_cast<int32_t *>(base + COAL_MAX * 16);
  int32_t *pairs = reinterpret_cast<int32_t *>(base + COAL_MAX * 20);
  const int64_t tile = blockIdx.x;
  for (int cl = warp; cl < TILE3; cl += COAL_WARPS) {
    const int64_t c = tile * TILE3 + cl;
    const uint32_t q0 = A.cell_off[c], q1 = A.cell_off[c + 1];
    const int64_t nc64 = (int64_t)q1 - (int64_t)q0;
    if (nc64 < 2) continue;
    auto list_big = [&]() {
      if (lane == 0) {
        const unsigned long long e = atomicAdd(A.n_big, 1ull);
        A.big_list[2 * e] = c;
        A.big_list[2 * e + 1] = (int64_t)atomicAdd(A.big_used, (unsigned long long)nc64);
      }
    };
    if (nc64 > COAL_MAX) {
      list_big();
      continue;
    }
    const int nc = (int)nc64;
    int N = 1;
    while (N < nc) N <<= 1;
    bool wide = false;
    for (int i = lane; i < N; i += 32) {
      if (i < nc) {
        const uint32_t p = A.perm[q0 + i];
        const int64_t bx = (int64_t)floor(A.a[3][p] / A.dv), by = (int64_t)floor(A.a[4][p] / A.dv),
                      bz = (int64_t)floor(A.a[5][p] / A.dv);
        wide |= bx <= -COAL_BIN_LIM || bx >= COAL_BIN_LIM || by <= -COAL_BIN_LIM || by >= COAL_BIN_LIM ||
                bz <= -COAL_BIN_LIM || bz >= COAL_BIN_LIM;
        key[i] = pack_bins(bx, by, bz);
        ids[i] = A.id[p];
        ix[i] = i;
      } else {
        key[i] = ~0ull;
        ids[i] = INT64_MAX;
        ix[i] = -1;
      }
    }
    if (__any_sync(0xffffffffu, wide)) {   // a bin beyond the packed key: the unpacked path
      list_big();
      __syncwarp();
      continue;
    }
    __syncwarp();
    // bitonic sort by (key, id): in registers up to 256 records; above, in
    // shared memory, each lane taking compare-exchange pairs (i, i + j)
    // directly (i = the pair index with a 0 bit inserted at j)
    if (N <= 32 * COAL_RREG) warp_sort_regs(key, ids, ix, N, lane);
    else for (int kk = 2; kk <= N; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int q = lane; q < (N >> 1); q += 32) {
          const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
          const int l = i | j;
          const bool up = (i & kk) == 0;
          const uint64_t ka = key[i], kb = key[l];
          const int64_t ia = ids[i], ib = ids[l];
          const bool b_less = kb < ka || (kb == ka && ib < ia);
          if (b_less == up) {
            key[i] = kb; key[l] = ka;
            ids[i] = ib; ids[l] = ia;
            const int32_t t = ix[i]; ix[i] = ix[l]; ix[l] = t;
          }
        }
        __syncwarp();
      }
    }
    // pairs in sorted order.  The definition's sequential scan (pair t with
    // t + 1 when their bins agree, then skip both) pairs, within each run of
    // equal bins, the records at even offsets from the run's start with their
    // successors, and stops after mc pairs; the warp finds those records 32
    // at a time: run starts by a max-scan, leaders by offset parity, their
    // order by a ballot prefix.
    const int mc = (int)floor(A.frac * (double)nc);
    int np = 0, run0 = 0;
    for (int c0 = 0; c0 < nc; c0 += 32) {
      const int t = c0 + lane;
      const bool valid = t < nc;
      const uint64_t k = valid ? key[t] : ~0ull;
      const bool start = valid && (t == 0 || key[t - 1] != k);
      int st = start ? t : -1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, st, o);
        if (lane >= o) st = max(st, v);
      }
      st = max(st, run0);
      const bool leader = valid && ((t - st) & 1) == 0 && t + 1 < nc && key[t + 1] == k;
      const unsigned bal = __ballot_sync(0xffffffffu, leader);
      const int idx = np + __popc(bal & ((1u << lane) - 1u));
      if (leader && idx < mc) pairs[idx] = t;
      np += __popc(bal);
      run0 = __shfl_sync(0xffffffffu, st, 31);
    }
    np = min(np, mc);
    __syncwarp();
    for (int m = lane; m < np; m += 32) {
      const int t = pairs[m];
      const uint32_t p1 = A.perm[q0 + ix[t]], p2 = A.perm[q0 + ix[t + 1]];   // p1 has the smaller id
      const double qa = A.a[6][p1], qb = A.a[6][p2], qs = qa + qb;
#pragma unroll
      for (int d = 0; d < 6; ++d) A.a[d][p1] = (qa * A.a[d][p1] + qb * A.a[d][p2]) / qs;
      A.a[6][p1] = qs;
      A.key_new[p2] = KEY_DEAD;
    }
    if (lane == 0 && np) atomicAdd(A.merges, (unsigned long long)np);
    __syncwarp();
  }
}

// (bins, id) of record a < that of record b (the oracle's order, R31)
__device__ __forceinline__ bool big_less(const CoalBig &B, int64_t a, int64_t b) {
  if (B.bx[a] != B.bx[b]) return B.bx[a] < B.bx[b];
  if (B.by[a] != B.by[b]) return B.by[a] < B.by[b];
  if (B.bz[a] != B.bz[b]) return B.bz[a] < B.bz[b];
  return B.id[a] < B.id[b];
}
__device__ __forceinline__ void big_swap(const CoalBig &B, int64_t a, int64_t b) {
  double t;
  t = B.bx[a]; B.bx[a] = B.bx[b]; B.bx[b] = t;
  t = B.by[a]; B.by[a] = B.by[b]; B.by[b] = t;
  t = B.bz[a]; B.bz[a] = B.bz[b]; B.bz[b] = t;
  const int64_t i = B.id[a]; B.id[a] = B.id[b]; B.id[b] = i;
  const uint32_t x = B.idx[a]; B.idx[a] = B.idx[b]; B.idx[b] = x;
}

// One CTA per listed cell (grid-stride over the list).  Records are sorted
// ascending by a bitonic network whose every compare-exchange puts the smaller
// record at the lower index (first step of each merge compares i with its
// mirror in the block), so the virtual +infinity records that pad n_c to a
// power of two never move and are simply skipped.
__global__ void __launch_bounds__(256) coalesce_big_kernel(const CoalArgs A, const CoalBig B) {
  const unsigned long long nbig = *A.n_big;
  __shared__ int s_np;
  for (unsigned long long e = blockIdx.x; e < nbig; e += gridDim.x) {
    const int64_t c = A.big_list[2 * e], off = A.big_list[2 * e + 1];
    const uint32_t q0 = A.cell_off[c];
    const int64_t nc = (int64_t)A.cell_off[c + 1] - (int64_t)q0;
    PIC_DCHECK(off >= 0 && off + nc <= A.cap && (off + nc) / 2 <= A.cap && 2 * (int64_t)e + 1 < A.cap, A.stats);
    for (int64_t i = threadIdx.x; i < nc; i += blockDim.x) {
      const uint32_t p = A.perm[q0 + i];
      // + 0.0 maps a -0 bin to +0 (equal bins compare equal, as in the oracle)
      B.bx[off + i] = floor(A.a[3][p] / A.dv) + 0.0;
      B.by[off + i] = floor(A.a[4][p] / A.dv) + 0.0;
      B.bz[off + i] = floor(A.a[5][p] / A.dv) + 0.0;
      B.id[off + i] = A.id[p];
      B.idx[off + i] = p;
    }
    __syncthreads();
    int64_t N = 1;
    while (N < nc) N <<= 1;
    for (int64_t k = 2; k <= N; k <<= 1) {
      for (int64_t j = k >> 1; j > 0; j >>= 1) {
        for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
          // first step of the merge: mirror partner; later steps: i ^ j
          const int64_t l = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);
          if (l > i && l < nc && big_less(B, off + l, off + i)) big_swap(B, off + i, off + l);
        }
        __syncthreads();
      }
    }
    // pairs in sorted order (one thread, sequential like the definition)
    if (threadIdx.x == 0) {
      const int64_t mc = (int64_t)floor(A.frac * (double)nc);
      int np = 0;
      for (int64_t t = 0; t + 1 < nc && np < mc;) {
        const int64_t a = off + t, b = a + 1;
        if (B.bx[a] == B.bx[b] && B.by[a] == B.by[b] && B.bz[a] == B.bz[b]) {
          B.pairs[off / 2 + np++] = (int32_t)t;
          t += 2;
        } else {
          t += 1;
        }
      }
      s_np = np;
      if (np) atomicAdd(A.merges, (unsigned long long)np);
    }
    __syncthreads();
    const int np = s_np;
    for (int m = threadIdx.x; m < np; m += blockDim.x) {
      const int64_t t = off + B.pairs[off / 2 + m];
      const uint32_t p1 = B.idx[t], p2 = B.idx[t + 1];   // p1 has the smaller id
      const double qa = A.a[6][p1], qb = A.a[6][p2], qs = qa + qb;
#pragma unroll
      for (int d = 0; d < 6; ++d) A.a[d][p1] = (qa * A.a[d][p1] + qb * A.a[d][p2]) / qs;
      A.a[6][p1] = qs;
      A.key_new[p2] = KEY_DEAD;
    }
    __syncthreads();
  }
}

// Rank every position [0, *d_nraw) anew (after coalescence killed some).
__global__ void recount_kernel(const uint32_t *__restrict__ key_new, uint32_t *__restrict__ rank,
                               uint32_t *__restrict__ cell_count, int64_t ncells, const int64_t *__restrict__ d_nraw) {
  const int64_t n = *d_nraw;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t p = base + threadIdx.x;
    const bool act = p < n;
    const uint32_t k = act ? key_new[p] : KEY_DEAD;
    const bool counted = act && k < KEY_FIRST_RESERVED;
    const uint32_t r = count_rank(cell_count, ncells, k, counted, true);
    if (counted) rank[p] = r;
  }
}

pic_status control(Ctx *ctx, int s, int64_t target, double theta, double eps, double dv, uint64_t seed,
                   int32_t *action) {
  SpeciesStore &sp = ctx->sp[s];
  int64_t n = 0;
  pic_status st = live_count(ctx, s, &n);
  if (st != PIC_OK) return st;
  *action = 0;
  if (n == 0 || target <= 0) return PIC_OK;
  const Geom &g = ctx->geom;
  const uint32_t *nlive = sp.cell_off + g.ncells;
  if ((double)n < (double)target * (1.0 - theta)) {
    // splitting (R30): every live particle splits with probability p
    SplitArgs A;
    A.g = g;
    for (int k = 0; k < 7; ++k) A.a[k] = sp.a[k];
    A.id = sp.id;
    A.perm = sp.perm;
    A.nlive = nlive;
    A.key_new = sp.key_new;
    A.rank = sp.rank;
    A.cell_count = sp.cell_count;
    A.d_nraw = sp.d_nraw;
    A.cap = sp.cap;
    A.stats = ctx->stats;
    A.p_split = std::min(1.0, (double)(target - n) / (double)n);
    A.eps = eps;
    A.seed_lo = (uint32_t)seed;
    A.seed_hi = (uint32_t)(seed >> 32);
    A.cycle = (uint32_t)ctx->cycle;
    A.species = (uint32_t)s;
    split_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(A); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
    st = clamp_nraw(ctx, s);
    if (st != PIC_OK) return st;
    sp.n_raw = std::min<int64_t>(sp.cap, sp.n_raw + n);
    *action = 1;
    return build_order(ctx, s);
  }
  if ((double)n > (double)target * (1.0 + theta)) {
    // coalescence (R31): pairs in each cell, then a full recount of the order
    CoalArgs A;
    A.g = g;
    for (int k = 0; k < 7; ++k) A.a[k] = sp.a[k];
    A.id = sp.id;
    A.perm = sp.perm;
    A.cell_off = sp.cell_off;
    A.key_new = sp.key_new;
    A.dv = dv;
    A.frac = (double)(n - target) / (double)n;
    A.cap = sp.cap;
    A.stats = ctx->stats;
    A.merges = reinterpret_cast<unsigned long long *>(ctx->dev_counts + 60);
    A.n_big = reinterpret_cast<unsigned long long *>(ctx->dev_counts + 61);
    A.big_used = reinterpret_cast<unsigned long long *>(ctx->dev_counts + 62);
    // scratch of the unpacked path: the B buffers of the store are free between
    // cycles (cap records each; the cell list needs <= cap / 2 entries of 2 words,
    // the pair list <= cap / 2 ints at offset / 2)
    A.big_list = reinterpret_cast<int64_t *>(sp.b[4]);
    CoalBig B;
    B.bx = sp.b[0];
    B.by = sp.b[1];
    B.bz = sp.b[2];
    B.id = sp.id_b;
    B.idx = reinterpret_cast<uint32_t *>(sp.b[3]);
    B.pairs = reinterpret_cast<int32_t *>(sp.b[5]);
    PIC_CUDA(cudaMemsetAsync(A.merges, 0, 3 * sizeof(unsigned long long), ctx->stream));
    PIC_CUDA(cudaFuncSetAttribute(coalesce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)COAL_SMEM));
    coalesce_kernel<<<(unsigned)g.ntiles, 32 * COAL_WARPS, COAL_SMEM, ctx->stream>>>(A); ++ctx->launches;
    coalesce_big_kernel<<<kSMs * 2, 256, 0, ctx->stream>>>(A, B); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
    *action = 2;
    st = zero_cell_counts(ctx, s);
    if (st != PIC_OK) return st;
    // key_new holds the cell of every position below d_nraw (mover outputs and
    // appends); the merged partners now carry KEY_DEAD
    int64_t blocks = (sp.n_raw + 255) / 256;
    if (blocks > kSMs * 16) blocks = kSMs * 16;
    recount_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, ctx->stream>>>(sp.key_new, sp.rank, sp.cell_count,
                                                                                  g.ncells, sp.d_nraw); ++ctx->launches;
    PIC_CUDA(cudaGetLastError());
    return build_order(ctx, s);
  }
  return PIC_OK;
}

}  // namespace pic
