// Graph construction on the device: the inputs of the BFS hot path.
//
//   rmat_edges_device     <- generate_rmat   reference graph.py:68-85 (bit-exact)
//   permute_edges_device  <- build-defined seeded permutation (gap G1)
//   lattice_edges_device  <- config 4 lattice (gap G3)
//   build_csr_device      <- build_csr       reference graph.py:139-160
//
// Construction is input preparation, not the timed path; the sort and
// select primitives come from CUB (header-only, CUDA toolkit).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "lbfs_internal.cuh"

namespace lbfs {

// ---------------------------------------------------------------- PCG64
// numpy's PCG64: 128-bit LCG state, multiplier below, XSL-RR output of the
// post-step state; Generator.random() = (next64 >> 11) * 2^-53.
static constexpr uint64_t kPcgMultHi = 0x2360ED051FC65DA4ULL;
static constexpr uint64_t kPcgMultLo = 0x4385DF649FCCF645ULL;

struct U128 {
  uint64_t lo, hi;
};

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
  r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
  return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo);
  return r;
}

__device__ __forceinline__ uint64_t xsl_rr(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned r = (unsigned)(s.hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// jump tables: entry k advances the state by 2^k steps
struct JumpTable {
  PcgJump j[64];
};

static void host_jump(U128 inc, uint64_t delta, U128* mult_out, U128* plus_out) {
  U128 acc_mult{1, 0}, acc_plus{0, 0}, cur_mult{kPcgMultLo, kPcgMultHi}, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{1, 0}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  *mult_out = acc_mult;
  *plus_out = acc_plus;
}

__device__ __forceinline__ U128 apply_jump(const PcgJump& j, U128 s) {
  return add128(mul128(U128{j.mult_lo, j.mult_hi}, s), U128{j.plus_lo, j.plus_hi});
}

constexpr int kRmatPerThread = 32;

// One thread owns kRmatPerThread consecutive pairs and walks the 2*scale draw
// arrays in stream order: array j element k is stream position j*m + k.
// d > t  <=>  (x >> 11) > floor(t * 2^53) for the exact doubles involved, so
// the comparisons are integer compares against precomputed thresholds.
__global__ void __launch_bounds__(128) k_rmat(int scale, int64_t m, uint64_t t_ab, uint64_t t_a,
                                              uint64_t t_c, U128 s0, U128 inc, PcgJump jm,
                                              const JumpTable* __restrict__ table,
                                              uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  const int64_t lo = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRmatPerThread;
  if (lo >= m) return;
  // state after `lo` steps
  U128 s = s0;
  uint64_t d = (uint64_t)lo;
  for (int k = 0; d; ++k, d >>= 1)
    if (d & 1) s = apply_jump(table->j[k], s);
  uint32_t a_src[kRmatPerThread], a_dst[kRmatPerThread];
#pragma unroll
  for (int e = 0; e < kRmatPerThread; ++e) a_src[e] = a_dst[e] = 0;
  const int cnt = (int)min((int64_t)kRmatPerThread, m - lo);
  for (int b = 0; b < scale; ++b) {
    // array 2b: source bit
    uint32_t ii = 0;
    U128 t = s;
#pragma unroll
    for (int e = 0; e < kRmatPerThread; ++e) {
      t = add128(mul128(t, U128{kPcgMultLo, kPcgMultHi}), inc);
      ii |= (uint32_t)((xsl_rr(t) >> 11) > t_ab) << e;
    }
    s = apply_jump(jm, s);
    // array 2b+1: destination bit, threshold depends on the source bit
    t = s;
#pragma unroll
    for (int e = 0; e < kRmatPerThread; ++e) {
      t = add128(mul128(t, U128{kPcgMultLo, kPcgMultHi}), inc);
      const uint32_t iib = (ii >> e) & 1u;
      const uint64_t thr = iib ? t_c : t_a;
      a_src[e] |= iib << b;
      a_dst[e] |= (uint32_t)((xsl_rr(t) >> 11) > thr) << b;
    }
    s = apply_jump(jm, s);
  }
#pragma unroll
  for (int e = 0; e < kRmatPerThread; ++e) {
    if (e < cnt) {
      src[lo + e] = a_src[e];
      dst[lo + e] = a_dst[e];
    }
  }
}

static uint64_t threshold53(double t) {
  // floor(t * 2^53) for t in [0, 1]; exact because the scaling is by 2^53.
  if (t <= 0.0) return 0;  // k > 0 ... (t == 0 -> any k > 0 passes, k = 0 fails: d > 0)
  const double s = t * 9007199254740992.0;
  return (uint64_t)s;  // truncation == floor for s >= 0
}

void rmat_edges_device(int scale, int64_t m, double ab, double a_norm, double c_norm,
                       const uint64_t pcg[4], uint32_t* d_src, uint32_t* d_dst, cudaStream_t st) {
  if (m <= 0) return;
  const U128 s0{pcg[1], pcg[0]}, inc{pcg[3], pcg[2]};
  JumpTable h;
  for (int k = 0; k < 64; ++k) {
    U128 mu, pl;
    host_jump(inc, k < 63 ? (1ULL << k) : (1ULL << 63), &mu, &pl);
    h.j[k] = PcgJump{mu.lo, mu.hi, pl.lo, pl.hi};
  }
  U128 mu, pl;
  host_jump(inc, (uint64_t)m, &mu, &pl);
  PcgJump jm{mu.lo, mu.hi, pl.lo, pl.hi};
  JumpTable* d_table = dev_alloc<JumpTable>(1);
  LBFS_CUDA(cudaMemcpyAsync(d_table, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  // a threshold t with d > t: for t == 0 every positive k passes; floor() handles it
  const uint64_t tab = threshold53(ab), ta = threshold53(a_norm), tc = threshold53(c_norm);
  const int64_t threads = (m + kRmatPerThread - 1) / kRmatPerThread;
  const int64_t blocks = (threads + 127) / 128;
  LBFS_LAUNCH(k_rmat, (unsigned)blocks, 128, 0, st, scale, m, tab, ta, tc, s0, inc, jm, d_table,
              d_src, d_dst);
  LBFS_CUDA(cudaStreamSynchronize(st));
  dev_free(d_table);
}

// ---------------------------------------------------------------- permutation
// 4-round balanced Feistel network over 2*half bits (keys from splitmix64 of
// the seed), cycle-walked into [0, n). oracle/oracle.c restates it.
struct Feistel {
  uint64_t key[4];
  uint64_t mask;
  uint64_t n;
  int half;
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static Feistel feistel_make(uint64_t n, uint64_t seed) {
  Feistel f;
  int bits = 0;
  while (bits < 62 && (1ULL << bits) < n) ++bits;
  if (bits < 2) bits = 2;
  if (bits & 1) ++bits;
  f.half = bits / 2;
  f.mask = (1ULL << f.half) - 1;
  f.n = n;
  uint64_t st = seed ^ 0x6C616E6562667331ULL;  // "lanebfs1"
  for (int r = 0; r < 4; ++r) {
    st += 0x9E3779B97F4A7C15ULL;
    f.key[r] = mix64(st);
  }
  return f;
}

__device__ __forceinline__ uint32_t feistel_apply(const Feistel& f, uint64_t x) {
  do {
    uint64_t L = x >> f.half, R = x & f.mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t t = L ^ (mix64(R ^ f.key[r]) & f.mask);
      L = R;
      R = t;
    }
    x = (L << f.half) | R;
  } while (x >= f.n);
  return (uint32_t)x;
}

__global__ void k_permute(Feistel f, uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    src[i] = feistel_apply(f, src[i]);
    dst[i] = feistel_apply(f, dst[i]);
  }
}

void permute_edges_device(int64_t n, uint64_t seed, uint32_t* d_src, uint32_t* d_dst, int64_t m,
                          cudaStream_t st) {
  if (m <= 0) return;
  const Feistel f = feistel_make((uint64_t)n, seed);
  const int64_t blocks = std::min<int64_t>((m + 255) / 256, (int64_t)current_sm_count() * 16);
  LBFS_LAUNCH(k_permute, (unsigned)blocks, 256, 0, st, f, d_src, d_dst, m);
}

// ---------------------------------------------------------------- lattice
// vertex (r, c) = r*cols + c emits (v, v+1) if c+1 < cols, then (v, v+cols)
// if r+1 < rows; pairs are laid out in vertex order.
__global__ void k_lattice(int64_t rows, int64_t cols, uint32_t* __restrict__ src,
                          uint32_t* __restrict__ dst) {
  const int64_t nv = rows * cols;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = v / cols, c = v - r * cols;
    const int64_t down = (r + 1 < rows) ? 1 : 0;
    int64_t k = r * (2 * cols - 1) + c * (1 + down);
    if (c + 1 < cols) {
      src[k] = (uint32_t)v;
      dst[k] = (uint32_t)(v + 1);
      ++k;
    }
    if (down) {
      src[k] = (uint32_t)v;
      dst[k] = (uint32_t)(v + cols);
    }
  }
}

void lattice_edges_device(int64_t rows, int64_t cols, uint32_t* d_src, uint32_t* d_dst,
                          cudaStream_t st) {
  const int64_t nv = rows * cols;
  if (nv <= 0) return;
  const int64_t blocks = std::min<int64_t>((nv + 255) / 256, (int64_t)current_sm_count() * 16);
  LBFS_LAUNCH(k_lattice, (unsigned)blocks, 256, 0, st, rows, cols, d_src, d_dst);
}

// ---------------------------------------------------------------- build_csr
// dedup: keys (u << B) | v for every non-self-loop pair (and its reverse when
// symmetrising); self-loops get u = n so they sort last. Radix sort, unique,
// then row_ptr from the boundaries of u and col_idx from the low bits —
// exactly np.unique(src*n + dst) of graph.py:150 in the same order.
// no dedup: stable radix sort of (u, v) pairs by u over the concatenated
// [forward, reverse] list — np.argsort(kind="stable") of graph.py:153.
__global__ void k_make_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                            int64_t m, int B, uint64_t n, bool symmetrize,
                            uint64_t* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = src[i], v = dst[i];
    const bool loop = (u == v);
    keys[i] = loop ? (n << B) : ((u << B) | v);
    if (symmetrize) keys[m + i] = loop ? (n << B) : ((v << B) | u);
  }
}

__global__ void k_make_pairs(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                             int64_t m, bool symmetrize, uint32_t* __restrict__ ku,
                             uint32_t* __restrict__ kv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    ku[i] = src[i];
    kv[i] = dst[i];
    if (symmetrize) {
      ku[m + i] = dst[i];
      kv[m + i] = src[i];
    }
  }
}

// row_ptr[w] = first index whose row is >= w; rows given by key >> B.
__global__ void k_row_bounds_keys(const uint64_t* __restrict__ keys, int64_t nnz, int B, int64_t n,
                                  int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx) {
  const uint64_t vmask = (B >= 64) ? ~0ULL : ((1ULL << B) - 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = (i < nnz) ? (int64_t)(keys[i] >> B) : n;
    const int64_t pu = (i > 0) ? (int64_t)(keys[i - 1] >> B) : -1;
    for (int64_t w = pu + 1; w <= u; ++w) row_ptr[w] = i;
    if (i < nnz) col_idx[i] = (int32_t)(keys[i] & vmask);
  }
}

__global__ void k_row_bounds_u32(const uint32_t* __restrict__ rows, int64_t nnz, int64_t n,
                                 int64_t* __restrict__ row_ptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = (i < nnz) ? (int64_t)rows[i] : n;
    const int64_t pu = (i > 0) ? (int64_t)rows[i - 1] : -1;
    for (int64_t w = pu + 1; w <= u; ++w) row_ptr[w] = i;
  }
}

static int bits_for(uint64_t x) {  // bits needed to hold values in [0, x]
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

static unsigned grid_for(int64_t work, int threads = 256) {
  const int64_t cap = (int64_t)current_sm_count() * 16;
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  return (unsigned)std::min(b, cap);
}

Csr build_csr_device(int64_t n, const uint32_t* d_src, const uint32_t* d_dst, int64_t m,
                     bool symmetrize, bool dedup, cudaStream_t st) {
  Csr out;
  LBFS_CUDA(cudaGetDevice(&out.device));
  out.n = n;
  out.row_ptr = dev_alloc<int64_t>((size_t)n + 1);
  const int64_t total = symmetrize ? 2 * m : m;
  if (total == 0) {
    LBFS_CUDA(cudaMemsetAsync(out.row_ptr, 0, sizeof(int64_t) * (size_t)(n + 1), st));
    out.col_idx = dev_alloc<int32_t>(1);
    out.nnz = 0;
    LBFS_CUDA(cudaStreamSynchronize(st));
    return out;
  }
  if (dedup) {
    const int B = std::max(1, bits_for((uint64_t)(n - 1 > 0 ? n - 1 : 0)));
    const int end_bit = B + bits_for((uint64_t)n);
    uint64_t* k0 = dev_alloc<uint64_t>((size_t)total);
    uint64_t* k1 = dev_alloc<uint64_t>((size_t)total);
    LBFS_LAUNCH(k_make_keys, grid_for(m), 256, 0, st, d_src, d_dst, m, B, (uint64_t)n, symmetrize, k0);
    cub::DoubleBuffer<uint64_t> db(k0, k1);
    size_t tmp_bytes = 0;
    LBFS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, total, 0, end_bit, st));
    void* tmp = dev_alloc<uint8_t>(tmp_bytes);
    LBFS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, total, 0, end_bit, st));
    g_launches.fetch_add(2 * ((end_bit + 7) / 8), std::memory_order_relaxed);
    dev_free(tmp);
    uint64_t* sorted = db.Current();
    uint64_t* uniq = db.Alternate();
    int64_t* d_nsel = dev_alloc<int64_t>(1);
    tmp_bytes = 0;
    LBFS_CUDA(cub::DeviceSelect::Unique(nullptr, tmp_bytes, sorted, uniq, d_nsel, total, st));
    tmp = dev_alloc<uint8_t>(tmp_bytes);
    LBFS_CUDA(cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, uniq, d_nsel, total, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    int64_t nsel = 0;
    LBFS_CUDA(cudaMemcpyAsync(&nsel, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    LBFS_CUDA(cudaStreamSynchronize(st));
    dev_free(tmp);
    dev_free(d_nsel);
    // drop the (single, last) self-loop key if present
    if (nsel > 0) {
      uint64_t last = 0;
      LBFS_CUDA(cudaMemcpy(&last, uniq + nsel - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
      if ((int64_t)(last >> B) == n) --nsel;
    }
    out.nnz = nsel;
    out.col_idx = dev_alloc<int32_t>((size_t)nsel);
    LBFS_LAUNCH(k_row_bounds_keys, grid_for(nsel + 1), 256, 0, st, uniq, nsel, B, n, out.row_ptr,
                out.col_idx);
    LBFS_CUDA(cudaStreamSynchronize(st));
    dev_free(k0);
    dev_free(k1);
  } else {
    uint32_t* u0 = dev_alloc<uint32_t>((size_t)total);
    uint32_t* u1 = dev_alloc<uint32_t>((size_t)total);
    uint32_t* v0 = dev_alloc<uint32_t>((size_t)total);
    uint32_t* v1 = dev_alloc<uint32_t>((size_t)total);
    LBFS_LAUNCH(k_make_pairs, grid_for(m), 256, 0, st, d_src, d_dst, m, symmetrize, u0, v0);
    cub::DoubleBuffer<uint32_t> dk(u0, u1), dv(v0, v1);
    const int end_bit = std::max(1, bits_for((uint64_t)n));
    size_t tmp_bytes = 0;
    LBFS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, total, 0, end_bit, st));
    void* tmp = dev_alloc<uint8_t>(tmp_bytes);
    LBFS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dk, dv, total, 0, end_bit, st));
    g_launches.fetch_add(2 * ((end_bit + 7) / 8), std::memory_order_relaxed);
    out.nnz = total;
    out.col_idx = dev_alloc<int32_t>((size_t)total);
    LBFS_CUDA(cudaMemcpyAsync(out.col_idx, dv.Current(), sizeof(int32_t) * (size_t)total,
                              cudaMemcpyDeviceToDevice, st));
    LBFS_LAUNCH(k_row_bounds_u32, grid_for(total + 1), 256, 0, st, dk.Current(), total, n,
                out.row_ptr);
    LBFS_CUDA(cudaStreamSynchronize(st));
    dev_free(tmp);
    dev_free(u0);
    dev_free(u1);
    dev_free(v0);
    dev_free(v1);
  }
  return out;
}

void free_csr(Csr& c) {
  dev_free(c.row_ptr);
  dev_free(c.col_idx);
  c.row_ptr = nullptr;
  c.col_idx = nullptr;
}

}  // namespace lbfs
