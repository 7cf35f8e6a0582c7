// Partitioned top-down BFS: one rank per GPU, 1D word-cyclic
// partition of the degree-ordered internal ids. Rank g owns the ids of
// bitmap words w with w % P == g (every rank gets a share of the hubs, whose
// ids form the bitmap prefix) and stores their rows (neighbours as global
// internal ids). The visited bitmap and the frontier bitmap are replicated.
//
// One level, all on the caller's stream (the collectives between the steps
// are issued by the caller, e.g. torch.distributed over NCCL):
//   expand   the owned frontier with the single-GPU kernels in bitmap mode
//            (K1/K2, bfs.cu); a clear neighbour owned elsewhere is only
//            marked in the local visited bitmap (no parent)
//   pack     the marks of each peer's words (visited & ~prev) into that
//            peer's contiguous send slice                   -> all_to_all
//   merge    OR of the received slices, minus what is already visited, is
//            this rank's remote discoveries: set visited, parent = the first
//            neighbour of v in the replicated frontier F_L (v's row is local
//            and the graph symmetric, so one exists and lies one level up),
//            then k_compact over the owned words -> next frontier bins, levels,
//            the owned words of F_{L+1}, followed by the local counts
//            (4 words)                                   -> all_gather
//   sync     F_{L+1} in global word order; visited |= F_{L+1}; prev = visited;
//            the gathered counts summed on the device
//   done     host reads the summed counts: the layer (input, edges,
//            discovered) and termination, identical on every rank
// Sparse levels: when the level's global frontier edges E_L are
// small against the dense slices (2 (E_L + 8) <= W words), both exchanges
// carry id lists instead of bitmaps — a rank marks at most E_L vertices and
// discovers at most E_L, so slices of E_L + 1 (+ 4) words cannot overflow and
// every rank sizes them alike from E_L:
//   pack     [count, ids...] per peer (S words each)     -> all_to_all
//   merge    test-and-set of the received ids + parents, compaction, then the
//            owned new ids as [4 count words, count, ids...] (G words)
//                                                        -> all_gather
//   sync     F_{L+1} rebuilt from the lists; the rank's own sent marks
//            enter prev (visited & ~prev stays this level's marks only)
// The level structure is the reference's level-synchronous loop
// (traversal.py:90, 152, 366); the exchange replaces nothing in the
// reference (it is single-node CPU) and follows SURVEY §8e.
#include <algorithm>

#include "bfs_engine.cuh"

namespace lbfs {

// send[h*nwl + j] = marks of peer h's owned word j (global word j*P + h)
__global__ void k_part_pack(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ prev,
                            uint32_t* __restrict__ send, int64_t nwl, int part_log, int rank) {
  const int64_t total = nwl << part_log;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = i / nwl, j = i - h * nwl;
    const int64_t gw = (j << part_log) | h;
    send[i] = (h == rank) ? 0u : (visited[gw] & ~prev[gw]);
  }
}

// ---- sparse levels: id lists instead of bitmaps ----------------------------
// send[h*S] = number of ids for peer h, send[h*S + 1 + i] = the ids (global
// internal); the counts are zeroed by the caller. err counts overflows (none
// by construction: a rank marks at most E_L vertices).
__global__ void k_part_pack_sparse(const uint32_t* __restrict__ visited, const uint32_t* __restrict__ prev,
                                   int64_t nwords, int part_log, int rank, uint32_t* __restrict__ send, int64_t S,
                                   unsigned long long* err) {
  const int64_t mask = (1 << part_log) - 1;
  for (int64_t gw = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gw < nwords; gw += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = gw & mask;
    if (h == rank) continue;
    uint32_t m = visited[gw] & ~prev[gw];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t pos = atomicAdd(send + h * S, 1u);
      if (pos + 1 < (uint64_t)S) send[h * S + 1 + pos] = (uint32_t)(gw * 32 + b);
      else atomicAdd(err, 1ull);
    }
  }
}

// Received ids (owned by this rank): test-and-set; a new one gets its parent
// (first neighbour in F_L = fglob). Thread per list slot.
__global__ void k_part_merge_sparse(const uint32_t* __restrict__ recv, int64_t S, int nparts, int part_log, int rank,
                                    uint32_t* __restrict__ visited, const uint32_t* __restrict__ fglob,
                                    const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                    const int32_t* __restrict__ new2old, int32_t* __restrict__ pred_int,
                                    unsigned long long* __restrict__ scanned) {
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nparts * S; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / S, k = i - p * S;
    if (p == rank || k == 0 || k > (int64_t)recv[p * S]) continue;
    const int32_t v = (int32_t)recv[i];
    const uint32_t bit = 1u << (v & 31);
    if (atomicOr(visited + (v >> 5), bit) & bit) continue;
    const int64_t l = part_local(v, part_log);
    const int64_t e0 = row_ptr[l], e1 = row_ptr[l + 1];
    int32_t par = kSentinel;
    for (int64_t e = e0; e < e1; ++e) {
      const int32_t u = __ldg(col_idx + e);
      ++cnt;
      if ((__ldg(fglob + (u >> 5)) >> (u & 31)) & 1u) {
        par = __ldg(new2old + u);
        break;
      }
    }
    pred_int[l] = par;
  }
  if (cnt && scanned) atomicAdd(scanned, cnt);
}

// The owned new vertices (front: owned words of F_{L+1}, local numbering) as
// the list out[5 ...], out[4] = count (zeroed by the caller).
__global__ void k_part_listify(const uint32_t* __restrict__ front, int64_t nwl, int part_log, int rank,
                               uint32_t* __restrict__ out, int64_t cap, unsigned long long* err) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nwl; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = front[j];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t pos = atomicAdd(out + 4, 1u);
      if (pos < (uint64_t)cap) out[5 + pos] = (uint32_t)part_global(j * 32 + b, part_log, rank);
      else atomicAdd(err, 1ull);
    }
  }
}

// F_{L+1} from the gathered lists (fglob cleared by the caller): fglob,
// visited and prev get every listed id; then (second kernel) this rank's own
// sent marks enter prev.
__global__ void k_part_sync_sparse(const uint32_t* __restrict__ fgath, int64_t G, int nparts,
                                   uint32_t* __restrict__ fglob, uint32_t* __restrict__ visited,
                                   uint32_t* __restrict__ prev) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nparts * G; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / G, k = i - p * G;
    if (k < 5 || k - 5 >= (int64_t)fgath[p * G + 4]) continue;
    const uint32_t v = fgath[i];
    const uint32_t bit = 1u << (v & 31);
    atomicOr(fglob + (v >> 5), bit);
    atomicOr(visited + (v >> 5), bit);
    atomicOr(prev + (v >> 5), bit);
  }
}
__global__ void k_part_marks_to_prev(const uint32_t* __restrict__ send, int64_t S, int nparts, int rank,
                                     uint32_t* __restrict__ prev) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nparts * S; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / S, k = i - p * S;
    if (p == rank || k == 0 || k > (int64_t)send[p * S]) continue;
    const uint32_t v = send[i];
    atomicOr(prev + (v >> 5), 1u << (v & 31));
  }
}

// Warp per owned word (lane = bit): remote discoveries of this level and
// their parents. recv[p*nwl + j] is peer p's marks for owned word j.
// Without fglob (a heavy level: blind ORs wrote no parent) only visited is
// completed here; every new owned vertex, local or remote discovery, gets its
// parent from k_part_resolve on the side stream.
__global__ void k_part_merge(const uint32_t* __restrict__ recv, int64_t nwl, int part_log, int rank,
                             uint32_t* __restrict__ visited, const uint32_t* __restrict__ fglob,
                             const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                             const int32_t* __restrict__ new2old, int32_t* __restrict__ pred_int,
                             unsigned long long* __restrict__ scanned) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < nwl; j += nw) {
    uint32_t inc = 0;
    for (int p = 0; p < (1 << part_log); ++p)
      if (p != rank) inc |= __ldg(recv + (int64_t)p * nwl + j);
    const int64_t gw = (j << part_log) | rank;
    if (!inc) continue;  // warp-uniform
    const uint32_t vis = visited[gw];
    const uint32_t nb = fglob ? inc & ~vis : 0u;
    __syncwarp();
    if (lane == 0 && (inc & ~vis)) visited[gw] = vis | inc;
    if ((nb >> lane) & 1u) {
      const int64_t l = j * 32 + lane;
      const int64_t e0 = row_ptr[l], e1 = row_ptr[l + 1];
      int32_t par = kSentinel;
      for (int64_t e = e0; e < e1; ++e) {
        const int32_t u = __ldg(col_idx + e);
        ++cnt;
        if ((__ldg(fglob + (u >> 5)) >> (u & 31)) & 1u) {
          par = __ldg(new2old + u);
          break;
        }
      }
      pred_int[l] = par;  // always found: a marking peer expanded a neighbour in F_L
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if (lane == 0 && cnt && scanned) atomicAdd(scanned, cnt);
}

// Parents of the owned vertices at level lvl after a heavy level (side
// stream, off the critical path): the first neighbour in F_{lvl-1} (a
// snapshot of the replicated frontier bitmap taken before the next level
// overwrote it). Thread per owned vertex; vertices of later levels are only
// ever written from -1 to a level > lvl, so the concurrent compactions of the
// next levels never make a vertex look like one of this level.
__global__ void k_part_resolve(const int32_t* level_int, int64_t n_loc, int32_t lvl,
                               const uint32_t* __restrict__ fprev, const int64_t* __restrict__ row_ptr,
                               const int32_t* __restrict__ col_idx, const int32_t* __restrict__ new2old,
                               int32_t* __restrict__ pred_int, unsigned long long* __restrict__ scanned) {
  unsigned long long cnt = 0;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_loc; l += (int64_t)gridDim.x * blockDim.x) {
    if (level_int[l] != lvl) continue;
    const int64_t e0 = row_ptr[l], e1 = row_ptr[l + 1];
    int32_t par = kSentinel;
    for (int64_t e = e0; e < e1; ++e) {
      const int32_t u = __ldg(col_idx + e);
      ++cnt;
      if ((__ldg(fprev + (u >> 5)) >> (u & 31)) & 1u) {
        par = __ldg(new2old + u);
        break;
      }
    }
    pred_int[l] = par;
  }
  if (cnt && scanned) atomicAdd(scanned, cnt);
}

// local counts of the next frontier -> the 4 words after the frontier words
// of the all-gather slice (two little-endian 64-bit values)
__global__ void k_part_counts(const Counters* __restrict__ c, uint32_t* __restrict__ tail) {
  tail[0] = (uint32_t)c->discovered;
  tail[1] = (uint32_t)(c->discovered >> 32);
  tail[2] = (uint32_t)c->edges;
  tail[3] = (uint32_t)(c->edges >> 32);
}
// the level's local counters and the global counts -> mapped host memory,
// then the sequence word (the host spins on it: a blocking stream sync costs
// tens of microseconds of wake-up per level). The global counts are red
// (the start's all-reduced root counts) or, after a level, the sum of the P
// count tails of the gathered slices fgath.
__global__ void k_part_publish(const Counters* __restrict__ cnt, const unsigned long long* __restrict__ red,
                               const uint32_t* __restrict__ fgath, int nparts, int64_t stride, int64_t tail_off,
                               const unsigned long long* __restrict__ err, Counters* mail,
                               unsigned long long* red_mail, unsigned long long* seq, unsigned long long value) {
  const int t = threadIdx.x;
  constexpr int kWords = (int)(sizeof(Counters) / 8);
  if (cnt && t < kWords)
    reinterpret_cast<volatile unsigned long long*>(mail)[t] = reinterpret_cast<const unsigned long long*>(cnt)[t];
  if (t < 2) {
    unsigned long long s = 0;
    if (red) {
      s = red[t];
    } else {
      for (int p = 0; p < nparts; ++p) {
        const uint32_t* tail = fgath + p * stride + tail_off + 2 * t;
        s += (unsigned long long)tail[0] | ((unsigned long long)tail[1] << 32);
      }
    }
    reinterpret_cast<volatile unsigned long long*>(red_mail)[t] = s;
  }
  if (t == 2) reinterpret_cast<volatile unsigned long long*>(red_mail)[2] = err ? *err : 0ull;
  __syncwarp();
  if (t == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(seq) = value;
  }
}

// fgath[h*stride + j] = rank h's owned word j of F_{L+1} (stride = nwl + 4)
__global__ void k_part_sync(const uint32_t* __restrict__ fgath, uint32_t* __restrict__ fglob,
                            uint32_t* __restrict__ visited, uint32_t* __restrict__ prev, int64_t nwords, int64_t stride,
                            int part_log) {
  const int64_t mask = (1 << part_log) - 1;
  for (int64_t gw = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gw < nwords;
       gw += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t f = fgath[(gw & mask) * stride + (gw >> part_log)];
    fglob[gw] = f;
    const uint32_t v = visited[gw] | f;
    visited[gw] = v;
    prev[gw] = v;
  }
}

// Outputs in original ids, one sequential pass over them (4 per thread,
// gathered through old2new): owned reached vertices (their bit in the
// replicated visited bitmap) get their record, every other entry the fill
// (SENTINEL / -1), so the ranks' outputs combine by min / max. kVec: 16-byte
// aligned outputs.
template <bool kVec>
__global__ void __launch_bounds__(256) k_part_finalize(const int32_t* __restrict__ old2new,
                                                       const uint32_t* __restrict__ visited,
                                                       const int32_t* __restrict__ level_int,
                                                       const int32_t* __restrict__ pred_int, int64_t n, int64_t npad,
                                                       int part_log, int rank, int32_t* __restrict__ level_out,
                                                       int32_t* __restrict__ pred_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i * 4 < npad; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v4 = __ldg(reinterpret_cast<const int4*>(old2new) + i);  // (old2new is padded)
    const int32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
    int32_t p[4], lv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool ok = i * 4 + q < n && part_owned(v[q], part_log, rank) &&
                      ((__ldg(visited + (v[q] >> 5)) >> (v[q] & 31)) & 1u);
      const int32_t l = part_local(v[q], part_log);
      p[q] = ok && pred_out ? pred_int[l] : kSentinel;
      lv[q] = ok && level_out ? level_int[l] : -1;
    }
    if (pred_out) {  // npad is a multiple of 32
      if (kVec) reinterpret_cast<int4*>(pred_out)[i] = make_int4(p[0], p[1], p[2], p[3]);
      else
#pragma unroll
        for (int q = 0; q < 4; ++q) pred_out[i * 4 + q] = p[q];
    }
    if (level_out) {
      if (kVec && i * 4 + 3 < n) {
        reinterpret_cast<int4*>(level_out)[i] = make_int4(lv[0], lv[1], lv[2], lv[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i * 4 + q < n) level_out[i * 4 + q] = lv[q];
      }
    }
  }
}

static unsigned grid_for(int64_t work, int sm_count) { return clamp_grid((work + 255) / 256, (int64_t)sm_count * 8); }

void BfsEngine::part_start(int64_t root, cudaStream_t st, unsigned long long* red) {
  if (root < 0 || root >= n_) throw_inval("root out of range");
  part_st_ = st;
  if (side_pending_) {  // an abandoned BFS left side work: it reads level_int, which k_init resets
    LBFS_CUDA(cudaStreamSynchronize(res_st_));
    side_pending_ = false;
  }
  if (!h_red_) {
    void* m = nullptr;
    LBFS_CUDA(cudaHostAlloc(&m, 4 * sizeof(unsigned long long), cudaHostAllocMapped));
    h_red_ = reinterpret_cast<unsigned long long*>(m);
  }
  if (!part_err_) part_err_ = dev_alloc<unsigned long long>(1);
  LBFS_CUDA(cudaMemsetAsync(part_err_, 0, sizeof(unsigned long long), st));
  part_sparse_ = false;
  LBFS_LAUNCH(k_init, grid_for(std::max(nwords_, n_loc_) / 4, sm_count_), 256, 0, st, (uint4*)visited_,
              (uint4*)prev_, (nwords_ + 3) / 4, (int4*)level_int_, (n_loc_ + 3) / 4);
  if (fglob_) LBFS_CUDA(cudaMemsetAsync(fglob_, 0, sizeof(uint32_t) * (size_t)nwords_, st));
  if (resolve_cnt_) LBFS_CUDA(cudaMemsetAsync(resolve_cnt_, 0, sizeof(unsigned long long), st));
  LBFS_CUDA(cudaMemsetAsync(cnt_, 0, sizeof(Counters) * kCounterRing, st));
  LevelArgs a = level_args();
  a.next_small = q_small_[0];
  a.next_warp = q_warp_[0];
  a.next_cta = q_cta_[0];
  LBFS_LAUNCH(k_seed, 1, 1, 0, st, a, prev_, old2new_, (int32_t)root, &cnt_[0], fglob_, red);
  LBFS_CUDA(cudaMemcpyAsync(&h_cnt_[0], &cnt_[0], sizeof(Counters), cudaMemcpyDeviceToHost, st));
  layers_.clear();
  part_L_ = -1;  // until part_level_done has the summed root counts
  part_cur_ = 0;
  part_prev_bitmap_ = false;
}

void BfsEngine::part_expand(cudaStream_t st) {
  if (part_L_ < 0) throw_inval("part_expand before the start counts were summed");
  part_st_ = st;
  const int64_t L = part_L_;
  const Counters c = h_cnt_[L % kCounterRing];
  LBFS_CUDA(cudaMemsetAsync(&cnt_[(L + 1) % kCounterRing], 0, sizeof(Counters), st));
  LevelArgs a = level_args();
  // bitmap mode (the exchange works on bitmaps, and queue-mode settling
  // would elect winners for vertices this rank does not own); heavy levels
  // (the level's global frontier edges >= nnz / heavy_div) use the blind-OR
  // semantics: no parent is written during the expansion, part_merge resolves
  // the parents of every new owned vertex
  part_heavy_ = stage_ && heavy_div_ > 0 && part_edges_ * (unsigned long long)heavy_div_ >= (unsigned long long)nnz_ &&
                !part_heavy_off_;
  expand_level(a, c, part_heavy_ ? kHeavy : kBitmapOut, part_prev_bitmap_, part_cur_, L, st);
  if (part_heavy_) merge_hot(st);
}

void BfsEngine::part_pack(uint32_t* send, cudaStream_t st) {
  part_st_ = st;
  part_send_ = send;
  if (part_sparse_) {
    LBFS_CUDA(cudaMemsetAsync(send, 0, sizeof(uint32_t) * (size_t)(nparts_ * part_S_), st));
    LBFS_LAUNCH(k_part_pack_sparse, grid_for(nwords_, sm_count_), 256, 0, st, visited_, prev_, nwords_, part_log_,
                part_rank_, send, part_S_, part_err_);
    return;
  }
  LBFS_LAUNCH(k_part_pack, grid_for(nwords_, sm_count_), 256, 0, st, visited_, prev_, send, nwl_, part_log_,
              part_rank_);
}

void BfsEngine::part_plan(int64_t* a2a_words, int64_t* gather_words) const {
  if (a2a_words) *a2a_words = part_sparse_ ? part_S_ : nwl_;
  if (gather_words) *gather_words = part_sparse_ ? part_G_ : nwl_ + 4;
}

// the next level's exchange format, from its global frontier edges (the same
// on every rank)
void BfsEngine::part_choose_format() {
  const int64_t E = (int64_t)part_edges_;
  part_sparse_ = nparts_ > 1 && part_sparse_mode_ != 0 &&
                 (part_sparse_mode_ == 2 ? E + 8 <= nwl_ : 2 * (E + 8) <= nwl_);
  part_S_ = (E + 1 + 3) & ~int64_t(3);
  part_G_ = (E + 5 + 3) & ~int64_t(3);
}

void BfsEngine::part_merge(const uint32_t* recv, uint32_t* fsend, cudaStream_t st) {
  part_st_ = st;
  const int64_t L = part_L_;
  if (part_sparse_) {  // (never heavy: a sparse level is small)
    LBFS_LAUNCH(k_part_merge_sparse, grid_for(nparts_ * part_S_, sm_count_), 256, 0, st, recv, part_S_, nparts_,
                part_log_, part_rank_, visited_, fglob_, row_ptr_, col_idx_, new2old_, pred_int_, resolve_cnt_);
    compact_level(part_cur_, L, nullptr, st);
    LBFS_CUDA(cudaMemsetAsync(fsend + 4, 0, sizeof(uint32_t), st));
    LBFS_LAUNCH(k_part_listify, grid_for(nwl_, sm_count_), 256, 0, st, front_, nwl_, part_log_, part_rank_, fsend,
                part_G_ - 5, part_err_);
    LBFS_LAUNCH(k_part_counts, 1, 1, 0, st, &cnt_[(L + 1) % kCounterRing], fsend);
    return;
  }
  if (nparts_ > 1)
    LBFS_LAUNCH(k_part_merge, grid_for(nwl_ * 32, sm_count_), 256, 0, st, recv, nwl_, part_log_, part_rank_,
                visited_, part_heavy_ ? nullptr : fglob_ /* F_L */, row_ptr_, col_idx_, new2old_, pred_int_,
                resolve_cnt_);
  uint32_t* snap = nullptr;
  if (part_heavy_) {  // F_L, for the parents of this level's vertices (resolved after the compaction)
    const int k = snap_next_;
    snap_next_ ^= 1;
    if (!snap_[k]) snap_[k] = dev_alloc<uint32_t>((size_t)nwords_ + 4);
    if (snap_used_[k]) LBFS_CUDA(cudaStreamWaitEvent(st, ev_snap_[k], 0));  // its last reader is done
    snap = snap_[k];
    LBFS_CUDA(cudaMemcpyAsync(snap, nparts_ > 1 ? fglob_ : front_, sizeof(uint32_t) * (size_t)nwords_,
                              cudaMemcpyDeviceToDevice, st));
    compact_level(part_cur_, L, fsend, st);
    LBFS_CUDA(cudaEventRecord(ev_resolve_, st));
    LBFS_CUDA(cudaStreamWaitEvent(res_st_, ev_resolve_, 0));
    LBFS_LAUNCH(k_part_resolve, grid_for(n_loc_, sm_count_), 256, 0, res_st_, level_int_, n_loc_, (int32_t)(L + 1),
                snap, row_ptr_, col_idx_, new2old_, pred_int_, resolve_cnt_);
    LBFS_CUDA(cudaEventRecord(ev_snap_[k], res_st_));
    snap_used_[k] = true;
    side_pending_ = true;
  } else {
    compact_level(part_cur_, L, fsend, st);
  }
  LBFS_LAUNCH(k_part_counts, 1, 1, 0, st, &cnt_[(L + 1) % kCounterRing], fsend + nwl_);
}

void BfsEngine::part_sync(const uint32_t* fgath, cudaStream_t st) {
  part_st_ = st;
  // (one partition: visited and prev are already complete after k_compact)
  if (part_sparse_) {
    LBFS_CUDA(cudaMemsetAsync(fglob_, 0, sizeof(uint32_t) * (size_t)nwords_, st));
    LBFS_LAUNCH(k_part_sync_sparse, grid_for(nparts_ * part_G_, sm_count_), 256, 0, st, fgath, part_G_, nparts_,
                fglob_, visited_, prev_);
    LBFS_LAUNCH(k_part_marks_to_prev, grid_for(nparts_ * part_S_, sm_count_), 256, 0, st, part_send_, part_S_,
                nparts_, part_rank_, prev_);
  } else if (nparts_ > 1) {
    LBFS_LAUNCH(k_part_sync, grid_for(nwords_, sm_count_), 256, 0, st, fgath, fglob_, visited_, prev_, nwords_,
                nwl_ + 4, part_log_);
  }
  part_fgath_ = fgath;  // (part_level_done sums its count tails)
}

void BfsEngine::part_level_done(const unsigned long long* red_global, lbfs_layer* layer, int* done) {
  cudaStream_t st = part_st_;
  const int64_t L = part_L_;
  const int slot = (int)((L + 1) % kCounterRing);
  if (!red_global && (L < 0 || !part_fgath_)) throw_inval("part_level_done: the start needs the summed root counts");
  const unsigned long long want = ++seq_;
  // (a level: the global counts are the sum of the gathered slices' tails)
  LBFS_LAUNCH(k_part_publish, 1, 32, 0, st, L >= 0 ? &cnt_[slot] : nullptr, red_global, part_fgath_, nparts_,
              part_sparse_ ? part_G_ : nwl_ + 4, part_sparse_ ? int64_t(0) : nwl_, part_err_, h_mail_, h_red_, h_seq_,
              want);
  part_fgath_ = nullptr;
  wait_mail(want, st);
  std::atomic_thread_fence(std::memory_order_acquire);  // (the mailbox is read after the sequence word)
  if (L >= 0) h_cnt_[slot] = *const_cast<const Counters*>(h_mail_);
  if (reinterpret_cast<volatile unsigned long long*>(h_red_)[2])
    throw Failure(LBFS_ECUDA, "internal: sparse exchange slice overflow");
  const unsigned long long disc = reinterpret_cast<volatile unsigned long long*>(h_red_)[0],
                           edges = reinterpret_cast<volatile unsigned long long*>(h_red_)[1];
  if (L < 0) {  // start: the summed root counts (1, deg(root)) become frontier 0
    part_in_ = disc;
    part_edges_ = edges;
    part_L_ = 0;
    part_choose_format();
    if (layer) *layer = lbfs_layer{0, 0, 0};
    if (done) *done = disc == 0;
    return;
  }
  const lbfs_layer ly{(int64_t)part_in_, (int64_t)part_edges_, (int64_t)disc};
  layers_.push_back(ly);
  if (trace_)
    fprintf(stderr, "[lbfs] rank %d L%-3lld in=%-9llu edges=%-10llu local bins %llu/%llu/%llu/%llu disc=%llu\n",
            part_rank_, (long long)L, part_in_, part_edges_, h_cnt_[slot].bin[0], h_cnt_[slot].bin[1],
            h_cnt_[slot].bin[2], h_cnt_[slot].bin[3], disc);
  if (layer) *layer = ly;
  if (done) *done = disc == 0;
  part_in_ = disc;
  part_edges_ = edges;
  part_L_ = L + 1;
  part_choose_format();
  part_cur_ ^= 1;
  part_prev_bitmap_ = true;
}

void BfsEngine::part_finish(int32_t* d_pred, int32_t* d_level, cudaStream_t st) {
  part_st_ = st;
  if (side_pending_) {  // heavy-level parents resolved on the side stream
    LBFS_CUDA(cudaEventRecord(ev_side_done_, res_st_));
    LBFS_CUDA(cudaStreamWaitEvent(st, ev_side_done_, 0));
    side_pending_ = false;
  }
  if (!d_pred && !d_level) return;
  const bool vec = ((uintptr_t)d_pred % 16) == 0 && ((uintptr_t)d_level % 16) == 0;
  if (vec)
    LBFS_LAUNCH(k_part_finalize<true>, grid_for(npad_ / 4, sm_count_), 256, 0, st, old2new_, visited_, level_int_,
                pred_int_, n_, npad_, part_log_, part_rank_, d_level, d_pred);
  else
    LBFS_LAUNCH(k_part_finalize<false>, grid_for(npad_ / 4, sm_count_), 256, 0, st, old2new_, visited_, level_int_,
                pred_int_, n_, npad_, part_log_, part_rank_, d_level, d_pred);
}

unsigned long long BfsEngine::resolve_scanned() const {
  if (!resolve_cnt_) return 0;
  unsigned long long v = 0;
  LBFS_CUDA(cudaMemcpy(&v, resolve_cnt_, sizeof(v), cudaMemcpyDeviceToHost));
  return v;
}

}  // namespace lbfs
