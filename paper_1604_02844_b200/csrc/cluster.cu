// Small-frontier levels on one thread-block cluster (K5 on the device for
// the latency-bound part of the level loop, traversal.py:90/152/366).
//
// A level whose frontier has few edges (the 4096^2 lattice: every one of its
// ~5-8 K levels; R-MAT: the first and the last levels) is bounded by latency,
// not bandwidth: load a row, claim its neighbours, append the winners,
// synchronise. This kernel runs consecutive such levels inside ONE cluster of
// C CTAs (C = 16 with non-portable cluster sizes, else 8), 512 threads each:
//
//   * visited bitmap in distributed shared memory (when it fits: n <= ~64 M
//     vertices at C = 16): 32-byte sectors of the global bitmap are dealt to
//     the C CTAs round robin. A neighbour is not claimed remotely (remote
//     atomics are rate-bound: ~17 K claims per lattice level on 16 SMs): the
//     candidate (neighbour, parent) is stored into the mailbox of the CTA
//     owning its sector — a private region per sender there, slot from a
//     local counter — and after a cluster barrier the owner claims its
//     candidates with local shared-memory atomics (the winner is the one
//     whose old word lacked the bit: the atomicOr election of
//     traversal.py:143-148) and appends the winners to its own queue. A full
//     region falls back to `atom.shared::cluster.or` claims and remote
//     pushes. Larger graphs, and late segments of shallow traversals, claim
//     on the global bitmap in L2;
//   * per-CTA frontier queues in shared memory (small-degree vertices live
//     on the CTA that owns their bitmap sector), vertices of degree >= 32 in
//     a cluster-wide list in global memory whose rows every warp of the
//     cluster shares in 512-element chunks;
//   * two hardware cluster barriers per level (candidates delivered; winners
//     counted): the level's counts are added into every CTA's totals through
//     DSMEM, so all CTAs take the same continue / exit decision.
//
// The loop leaves when the frontier is empty (BFS done) or its edge count
// exceeds exit_edges (the full-GPU kernels take over): the frontier is then
// written in the host loop's queue format, the bitmap slices back to
// visited/prev, and the level counters to the mapped mailbox.
#include "bfs_engine.cuh"

namespace lbfs {

namespace {

constexpr unsigned kF = 0xFFFFFFFFu;
constexpr int kCT = kClusterThreads;
constexpr int kCW = kCT / 32;
#ifndef LBFS_BIG_CHUNK
#define LBFS_BIG_CHUNK 512
#endif
constexpr int kBigChunk = LBFS_BIG_CHUNK;  // elements per warp task of a degree >= 32 row

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Level barrier without release semantics: it does not wait for the level's
// fire-and-forget global stores (levels, parents, visited/prev copies),
// which nothing reads before the kernel ends. What the next level does read
// is complete before a thread arrives: bitmap claims and the counts are
// atomics whose returned values were consumed, the frontier queues are
// CTA-local (ordered by __syncthreads), and the few global list appends are
// fenced by their writers.
__device__ __forceinline__ void cl_level_sync() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long atom_add_dsm64(uint32_t a, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.relaxed.cluster.shared::cluster.add.u64 %0, [%1], %2;" : "=l"(old) : "r"(a), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_dsm32(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.cluster.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_exch_dsm32(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cluster.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long atom_exch_dsm64(uint32_t a, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.relaxed.cluster.shared::cluster.exch.b64 %0, [%1], %2;" : "=l"(old) : "r"(a), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_dsm64(uint32_t a, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void st_dsm32(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_dsm32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ unsigned long long ld_dsm64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_or_dsm(uint32_t a, uint32_t bit) {
  uint32_t old;
  asm volatile("atom.relaxed.cluster.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(bit) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void red_or_g(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ int4 ld_nc4(const int32_t* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// degree class of a small-region id: the d in [1, 31] with T[d+1] <= v < T[d]
__device__ __forceinline__ int small_degree(const int32_t* T, int32_t v) {
  int d = 1;
#pragma unroll
  for (int step = 16; step; step >>= 1)
    if (d + step <= kSmallMax - 1 && T[d + step] > v) d += step;
  return d;
}

struct ClusterSmem {
  int32_t T[kSmallMax + 2];
  int64_t B[kSmallMax + 1];
  uint32_t rbase[kMaxCluster];    // shared::cluster address of each CTA's bitmap slice
  uint32_t rq[2][kMaxCluster];    // ... of each CTA's small queues (parity 0 / 1)
  uint32_t rqcnt[kMaxCluster];    // ... of each CTA's qcnt[0]
  unsigned long long tot[3][2];   // cluster totals (discovered, edges) of level L in slot L % 3,
                                  // added into every CTA's copy by every CTA
  unsigned long long red[2][kCW];
  int32_t qcnt[2];                // entries appended to this CTA's small queue (parity)
  int32_t scnt[kMaxCluster];      // entries staged for each CTA's next queue
  // candidate mailboxes (DSMEM mode): a neighbour is not claimed remotely but
  // sent to the CTA owning its bitmap sector, which claims it in its own
  // shared memory and appends the winners to its own queue
  uint32_t rmail[kMaxCluster];    // shared::cluster address of each CTA's mailbox area
  uint32_t rincnt[kMaxCluster];   // ... of each CTA's in_cnt[0]
  int32_t out_cnt[kMaxCluster];   // candidates sent to each CTA this level (may exceed the cap: the rest went the remote way)
  int32_t in_cnt[kMaxCluster];    // candidates received from each CTA this level (written by the senders)
  int32_t off[kCW][33];           // per-warp group offsets (window path)
  int64_t start[kCW][32];
  int32_t par[kCW][32];
  unsigned long long tm[4];       // LBFS_CLUSTER_PROF: latest stage times of the level in this CTA
};

struct Ctx {
  const ClusterArgs* p;
  ClusterSmem* s;
  QEntry* q0;        // this CTA's small queues in shared memory (parity 0 / 1)
  QEntry* q1;
  QEntry* stage;     // [kMaxCluster][kClusterStage] winners staged per target CTA
  unsigned long long* mail;  // [kMaxCluster][mail_cap] candidates received, by sender
  int32_t mail_cap;          // 0: claim remotely (no mailboxes)
  uint32_t vis_base; // shared address of this CTA's slice
  uint32_t rank, csize, clog;
  int32_t next_level;
  int nx;            // parity of the queue being appended
  int64_t big_slot;  // ring slot (level % 3) of the big list being appended
  unsigned long long disc, edges;
  unsigned long long* wt;  // LBFS_CLUSTER_PROF_LEVEL: this warp's timeline of the captured level (lane 0)
  uint32_t wdone;          // stamps already taken
};
__device__ __forceinline__ void wstamp(Ctx& x, int k, int lane) {
  if (x.wt && !((x.wdone >> k) & 1u)) {
    x.wdone |= 1u << k;
    if (lane == 0) x.wt[k] = gtimer();
  }
}

__device__ __forceinline__ QEntry* spill_of(const Ctx& x, uint32_t rank, int buf) {
  return x.p->spill_small + ((int64_t)rank * 2 + buf) * x.p->cap;
}
// entry i of CTA t's next queue: its shared memory, or its spill area
__device__ __forceinline__ unsigned long long push_entry(const Ctx& x, uint32_t t, int32_t i, QEntry e) {
  const unsigned long long v = ((unsigned long long)(uint32_t)e.par << 32) | (uint32_t)e.v;
  if (i < x.p->qs) return atom_exch_dsm64(x.s->rq[x.nx][t] + 8u * (uint32_t)i, v);
  return atomicExch(reinterpret_cast<unsigned long long*>(spill_of(x, t, x.nx) + (i - x.p->qs)), v);
}
__device__ __forceinline__ QEntry qget(const Ctx& x, int cur, int32_t i) {
  if (i < x.p->qs) return (cur ? x.q1 : x.q0)[i];
  const uint2 e = __ldcg(reinterpret_cast<const uint2*>(spill_of(x, x.rank, cur) + (i - x.p->qs)));
  return QEntry{(int32_t)e.x, (int32_t)e.y};
}

// Claim vertex v's bit: its word in the owner CTA's slice (DSMEM) or in the
// global bitmap (L2); returns the old word.
template <bool DSM>
__device__ __forceinline__ uint32_t claim(const Ctx& x, int32_t v) {
  const uint32_t bit = 1u << (v & 31);
  const uint32_t gw = (uint32_t)v >> 5;
  if constexpr (DSM) {
    const uint32_t sec = gw >> 3;
    const uint32_t owner = sec & (x.csize - 1);
    const uint32_t lw = ((sec >> x.clog) << 3) | (gw & 7u);
    return atom_or_dsm(x.s->rbase[owner] + 4u * lw, bit);
  } else {
    return atomicOr(x.p->visited + gw, bit);
  }
}

template <bool DSM>
__device__ __forceinline__ uint32_t peek(const Ctx& x, int32_t v) {
  const uint32_t gw = (uint32_t)v >> 5;
  if constexpr (DSM) {
    const uint32_t sec = gw >> 3;
    const uint32_t owner = sec & (x.csize - 1);
    const uint32_t lw = ((sec >> x.clog) << 3) | (gw & 7u);
    return ld_dsm32(x.s->rbase[owner] + 4u * lw);
  } else {
    return __ldcg(x.p->visited + gw);
  }
}

// The records of a vertex taken off a small queue (written when it is
// expanded): level, parent, and its bit in the global bitmaps (DSMEM mode
// claims in shared memory; the host levels need visited/prev).
template <bool DSM>
__device__ __forceinline__ void write_record(const ClusterArgs& p, QEntry e, int32_t level) {
  p.level_int[e.v] = level;
  p.pred_int[e.v] = e.par;
  const uint32_t bit = 1u << (e.v & 31);
  if constexpr (DSM) red_or_g(p.visited + (e.v >> 5), bit);
  red_or_g(p.prev + (e.v >> 5), bit);
}

// Claim a batch of 4 neighbours per lane (elements outside okm hold junk);
// winners join the next frontier (warp-collective).
template <bool DSM>
__device__ __forceinline__ void settle4_remote(Ctx& x, const int32_t (&nb)[4], uint32_t okm, const int32_t (&par)[4],
                                               int lane) {
  const ClusterArgs& p = *x.p;
  if (p.prof && lane == 0) atomicMax(&x.s->tm[0], gtimer());  // (the loads of nb have returned)
  if (x.wt) {
    const uint32_t w = __reduce_or_sync(kF, (uint32_t)(nb[0] | nb[1] | nb[2] | nb[3]));
    if (w != 0x7fffffffu) wstamp(x, 2, lane);
  }
  uint32_t old[4];
  if (p.dbg & 16) {  // (experiment) read the word first, claim only a clear bit
    uint32_t cur[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cur[k] = ((okm >> k) & 1u) ? peek<DSM>(x, nb[k]) : kF;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((cur[k] >> (nb[k] & 31)) & 1u)) okm &= ~(1u << k);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) old[k] = ((okm >> k) & 1u) ? claim<DSM>(x, nb[k]) : kF;
  uint32_t win = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) win |= (((old[k] >> (nb[k] & 31)) & 1u) ^ 1u) << k;
  if (p.prof) {
    const uint32_t w = __reduce_or_sync(kF, win);  // the atomics have returned
    if (lane == 0) atomicMax(&x.s->tm[1], gtimer() + (w & 0));
    wstamp(x, 3, lane);
  }
  if (!__any_sync(kF, win != 0)) return;
  uint32_t small = 0, big = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!((win >> k) & 1u)) continue;
    const int32_t w = nb[k];
    x.disc += 1;
    if (w >= p.t_warp && w < p.t_nz) {  // small row: degree class in closed form, row prefetched into L2
      const int d = small_degree(x.s->T, w);
      x.edges += (unsigned long long)d;
      small |= 1u << k;
      if (!(p.dbg & 1)) {
        prefetch_l2(p.col_idx + x.s->B[d] + (int64_t)(w - x.s->T[d + 1]) * d);
        prefetch_l2(p.new2old + w);
      }
    } else {  // degree >= 32 (the cluster-wide list) or 0: records now
      write_record<DSM>(p, QEntry{w, par[k]}, x.next_level);
      big |= (uint32_t)(w < p.t_warp) << k;
    }
  }
  if (__any_sync(kF, big != 0)) {
    // rows of degree >= 32: the cluster-wide list, one reservation per warp;
    // the entries are written with atomic exchanges (consumed, so performed
    // before the relaxed level barrier; other CTAs read them next level)
    int64_t st[4];
    int32_t dg[4], uo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool b = (big >> k) & 1u;
      st[k] = b ? __ldg(p.row_ptr + nb[k]) : 0;
      dg[k] = b ? (int32_t)(__ldg(p.row_ptr + nb[k] + 1) - st[k]) : 0;
      uo[k] = b ? __ldg(p.new2old + nb[k]) : 0;
    }
    const uint32_t nbig = (uint32_t)__popc(big);
    uint32_t incl = nbig;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kF, incl, o);
      if (lane >= o) incl += t;
    }
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(p.big_cnt + x.big_slot, (unsigned long long)incl);
    base = __shfl_sync(kF, base, 31) + (incl - nbig);
    unsigned long long sink = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!((big >> k) & 1u)) continue;
      x.edges += (unsigned long long)dg[k];
      unsigned long long* e = reinterpret_cast<unsigned long long*>(p.big + x.big_slot * p.cap + (int64_t)base++);
      sink |= atomicExch(e, (unsigned long long)st[k]);
      sink |= atomicExch(e + 1, ((unsigned long long)(uint32_t)uo[k] << 32) | (uint32_t)dg[k]);
    }
    asm volatile("mov.b64 %0, %0;" : "+l"(sink));
  }
  // small winners join the next-level queue of the CTA owning their bitmap
  // sector (uniform over the cluster, so the frontier spreads over every CTA
  // whoever found it). They are staged per target in this CTA's shared memory
  // (one local atomic per target per warp) and pushed after the expansion,
  // one remote reservation per target (push_staged); a full stage sends the
  // entry at once.
  if (!__any_sync(kF, small != 0)) {
    wstamp(x, 4, lane);
    return;
  }
  unsigned long long sink = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool has = (small >> k) & 1u;
    const uint32_t tgt = has ? ((uint32_t)nb[k] >> 8) & (x.csize - 1) : 0xFFFFu;
    const uint32_t peers = __match_any_sync(kF, tgt);
    if (has) {
      const int leader = __ffs(peers) - 1;
      int32_t base = 0;
      if (lane == leader) base = atomicAdd(&x.s->scnt[tgt], __popc(peers));
      base = __shfl_sync(peers, base, leader);
      const int32_t i = base + __popc(peers & ((1u << lane) - 1u));
      const QEntry ent{nb[k], par[k]};
      if (i < kClusterStage) {
        x.stage[tgt * kClusterStage + i] = ent;
      } else {  // stage full: reserve a slot in the target's queue now
        const int32_t j = (int32_t)atom_add_dsm32(x.s->rqcnt[tgt] + 4u * (uint32_t)x.nx, 1u);
        sink |= push_entry(x, tgt, j, ent);
      }
    }
  }
  asm volatile("mov.b64 %0, %0;" : "+l"(sink));  // (performed before the level barrier)
  wstamp(x, 4, lane);
}

// Claim a batch of 4 neighbours per lane (warp-collective). DSMEM mode with
// mailboxes: a remote claim is an atomic round trip through the SM-to-SM
// network, and their rate (not their latency) bounds a level — ~17 K claims
// per lattice level on 16 SMs. So a candidate (neighbour, parent) is written
// into the mailbox of the CTA owning the neighbour's bitmap sector instead (a
// plain remote store into this sender's private region there: one local
// shared-memory atomic for the slot, no remote atomic); after the cluster
// barrier the owner claims its candidates locally (accept_mail). A full
// region sends the rest the remote-claim way.
template <bool DSM>
__device__ __forceinline__ void settle4(Ctx& x, const int32_t (&nb)[4], uint32_t okm, const int32_t (&par)[4], int lane) {
  if constexpr (DSM) {
    if (x.mail_cap > 0) {
      ClusterSmem& s = *x.s;
      if (x.wt) {  // (LBFS_CLUSTER_PROF_LEVEL) the loads of nb have returned
        const uint32_t w = __reduce_or_sync(kF, (uint32_t)(nb[0] | nb[1] | nb[2] | nb[3]));
        if (w != 0x7fffffffu) wstamp(x, 2, lane);
      }
      int32_t slot[4];
      uint32_t tgt[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tgt[k] = (((uint32_t)nb[k] >> 8) & (x.csize - 1));  // owner of the 32-byte bitmap sector (256 ids)
        slot[k] = ((okm >> k) & 1u) ? atomicAdd(&s.out_cnt[tgt[k]], 1) : 0;
      }
      uint32_t ovf = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!((okm >> k) & 1u)) continue;
        if (slot[k] < x.mail_cap)
          st_dsm64(s.rmail[tgt[k]] + 8u * (uint32_t)((int32_t)x.rank * x.mail_cap + slot[k]),
                   ((unsigned long long)(uint32_t)par[k] << 32) | (uint32_t)nb[k]);
        else
          ovf |= 1u << k;
      }
      if (__any_sync(kF, ovf != 0)) settle4_remote<DSM>(x, nb, ovf, par, lane);
      return;
    }
  }
  settle4_remote<DSM>(x, nb, okm, par, lane);
}

// (after the barrier that follows the expansion) warp w claims the candidates
// CTA w sent to this CTA, in this CTA's own slice of the bitmap; the winners
// join this CTA's next queue (rows of degree >= 32: the cluster-wide list).
__device__ __forceinline__ void accept_mail(Ctx& x, uint32_t* slice, int lane, int wib) {
  const ClusterArgs& p = *x.p;
  ClusterSmem& s = *x.s;
  if (wib >= (int)x.csize) return;
  const int32_t cnt = min(s.in_cnt[wib], x.mail_cap);
  const unsigned long long* mb = x.mail + (size_t)wib * x.mail_cap;
  QEntry* qn = x.nx ? x.q1 : x.q0;
  // 4 candidates per lane per step: their claims, degree look-ups and row
  // prefetches overlap (a step is a chain of shared-memory round trips)
  for (int32_t i0 = 0; i0 < cnt; i0 += 128) {
    int32_t w[4], par[4];
    uint32_t win = 0, small = 0, big = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t i = i0 + k * 32 + lane;
      const unsigned long long e = i < cnt ? mb[i] : 0ull;
      w[k] = (int32_t)(uint32_t)e;
      par[k] = (int32_t)(uint32_t)(e >> 32);
      if (i < cnt) {
        const uint32_t gw = (uint32_t)w[k] >> 5, bit = 1u << (w[k] & 31);
        const uint32_t lw = (((gw >> 3) >> x.clog) << 3) | (gw & 7u);
        win |= (uint32_t)!(atomicOr(slice + lw, bit) & bit) << k;
      }
    }
    wstamp(x, 8, lane);   // (claims returned)
    if (!__any_sync(kF, win != 0)) continue;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!((win >> k) & 1u)) continue;
      x.disc += 1;
      if (w[k] >= p.t_warp && w[k] < p.t_nz) {
        const int d = small_degree(s.T, w[k]);
        x.edges += (unsigned long long)d;
        small |= 1u << k;
        if (!(p.dbg & 1)) {
          prefetch_l2(p.col_idx + s.B[d] + (int64_t)(w[k] - s.T[d + 1]) * d);
          prefetch_l2(p.new2old + w[k]);
        }
      } else {  // degree >= 32 (the cluster-wide list) or 0: records now
        write_record<true>(p, QEntry{w[k], par[k]}, x.next_level);
        big |= (uint32_t)(w[k] < p.t_warp) << k;
      }
    }
    wstamp(x, 9, lane);   // (degrees, prefetches issued)
    // small winners: one reservation in this CTA's next queue per warp step
    {
      const uint32_t mine = (uint32_t)__popc(small);
      uint32_t incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kF, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t tot = __shfl_sync(kF, incl, 31);
      if (tot) {
        int32_t base = 0;
        if (lane == 31) base = atomicAdd(&s.qcnt[x.nx], (int32_t)tot);
        int32_t j = __shfl_sync(kF, base, 31) + (int32_t)(incl - mine);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!((small >> k) & 1u)) continue;
          if (j < p.qs) qn[j] = QEntry{w[k], par[k]};
          else spill_of(x, x.rank, x.nx)[j - p.qs] = QEntry{w[k], par[k]};
          ++j;
        }
      }
    }
    wstamp(x, 10, lane);  // (queue appended)
    if (__any_sync(kF, big != 0)) {  // rows of degree >= 32: the cluster-wide list
      int64_t st[4];
      int32_t dg[4], uo[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool b = (big >> k) & 1u;
        st[k] = b ? __ldg(p.row_ptr + w[k]) : 0;
        dg[k] = b ? (int32_t)(__ldg(p.row_ptr + w[k] + 1) - st[k]) : 0;
        uo[k] = b ? __ldg(p.new2old + w[k]) : 0;
      }
      const uint32_t nbig = (uint32_t)__popc(big);
      uint32_t incl = nbig;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kF, incl, o);
        if (lane >= o) incl += t;
      }
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(p.big_cnt + x.big_slot, (unsigned long long)incl);
      base = __shfl_sync(kF, base, 31) + (incl - nbig);
      unsigned long long sink = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!((big >> k) & 1u)) continue;
        x.edges += (unsigned long long)dg[k];
        unsigned long long* e2 = reinterpret_cast<unsigned long long*>(p.big + x.big_slot * p.cap + (int64_t)base++);
        sink |= atomicExch(e2, (unsigned long long)st[k]);
        sink |= atomicExch(e2 + 1, ((unsigned long long)(uint32_t)uo[k] << 32) | (uint32_t)dg[k]);
      }
      asm volatile("mov.b64 %0, %0;" : "+l"(sink));
    }
  }
}

// After the expansion (CTA-synchronised): warp t pushes the entries staged
// for CTA t — one remote reservation, then one atomic exchange per entry,
// so everything is performed before the thread arrives at the relaxed level
// barrier (the returned values are consumed).
__device__ __forceinline__ void push_staged(Ctx& x, int lane, int wib) {
  for (uint32_t t = (uint32_t)wib; t < x.csize; t += kCW) {
    const int32_t cnt = min(x.s->scnt[t], kClusterStage);
    if (cnt == 0) continue;
    int32_t base = 0;
    if (lane == 0) base = (int32_t)atom_add_dsm32(x.s->rqcnt[t] + 4u * (uint32_t)x.nx, (uint32_t)cnt);
    base = __shfl_sync(kF, base, 0);
    unsigned long long sink = 0;
    for (int32_t i = lane; i < cnt; i += 32) sink |= push_entry(x, t, base + i, x.stage[t * kClusterStage + i]);
    asm volatile("mov.b64 %0, %0;" : "+l"(sink));
    __syncwarp();
    if (lane == 0) x.s->scnt[t] = 0;
  }
}

// A warp expands up to 32 frontier vertices (lane i < n owns v, parent
// uo = its original id). Degrees <= 8 (the lattice, most small levels): a
// lane walks its own row, all its loads in flight at once. Larger: the
// concatenated rows in 128-element windows, the owner of element e found by
// binary search over the offsets.
template <bool DSM>
__device__ __forceinline__ void expand_small_group(Ctx& x, int n, int32_t v, int lane, int wib) {
  const ClusterArgs& p = *x.p;
  ClusterSmem& s = *x.s;
  wstamp(x, 1, lane);
  int32_t d = 0;
  int64_t st = 0;
  if (lane < n) {
    if (v >= p.t_warp && v < p.t_nz) {
      d = small_degree(s.T, v);
      st = s.B[d] + (int64_t)(v - s.T[d + 1]) * d;
    } else if (v < p.t_warp) {  // (external entries may name a bigger row: read it)
      st = p.row_ptr[v];
      d = (int32_t)(p.row_ptr[v + 1] - st);
    }
  }
  const int32_t uo = lane < n ? __ldg(p.new2old + v) : 0;
  const int dmax = __reduce_max_sync(kF, (unsigned)d);
  wstamp(x, 11, lane);  // (degrees known, loads about to issue)
  if (dmax <= 8) {
    int32_t nb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) nb[k] = k < d ? __ldg(p.col_idx + st + k) : 0;
    const uint32_t okm = (1u << d) - 1u;
    const int32_t pr[4] = {uo, uo, uo, uo};
    settle4<DSM>(x, *reinterpret_cast<const int32_t(*)[4]>(nb), okm & 0xFu, pr, lane);
    if (dmax > 4) settle4<DSM>(x, *reinterpret_cast<const int32_t(*)[4]>(nb + 4), okm >> 4, pr, lane);
    return;
  }
  int incl = d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(kF, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(kF, incl, 31);
  __syncwarp();
  s.off[wib][lane] = incl - d;
  s.start[wib][lane] = st - (incl - d);
  s.par[wib][lane] = uo;
  if (lane == 0) s.off[wib][32] = total;
  __syncwarp();
  const int top = n > 1 ? 1 << (31 - __clz(n - 1)) : 0;
  for (int e0 = 0; e0 < total; e0 += 128) {
    int32_t nb[4], pr[4];
    uint32_t okm = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + k * 32 + lane;
      const bool ok = e < total;
      int lo = 0;
      for (int step = top; step; step >>= 1)
        if (s.off[wib][lo + step] <= e) lo += step;
      okm |= (uint32_t)ok << k;
      nb[k] = ok ? __ldg(p.col_idx + s.start[wib][lo] + e) : 0;
      pr[k] = s.par[wib][lo];
    }
    settle4<DSM>(x, nb, okm, pr, lane);
  }
  __syncwarp();
}

// A warp streams the slice [st, st+len) of one row (parent par, original id)
// with 128-bit loads, one window ahead.
template <bool DSM>
__device__ __forceinline__ void stream_slice(Ctx& x, int64_t st, int32_t len, int32_t par, int lane) {
  const ClusterArgs& p = *x.p;
  const int64_t end = st + len;
  int64_t pos = st & ~int64_t(3);
  auto load = [&](int64_t p0) {
    const int64_t i = p0 + lane * 4;
    return i < end ? ld_nc4(p.col_idx + i) : make_int4(0, 0, 0, 0);
  };
  int4 cur = load(pos);
  for (; pos < end; pos += 128) {
    const int4 nxt = pos + 128 < end ? load(pos + 128) : make_int4(0, 0, 0, 0);
    int32_t nb[4] = {cur.x, cur.y, cur.z, cur.w};
    uint32_t okm = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = pos + lane * 4 + q;
      okm |= (uint32_t)(i >= st && i < end) << q;
    }
    const int32_t pr[4] = {par, par, par, par};
    settle4<DSM>(x, nb, okm, pr, lane);
    cur = nxt;
  }
}

// Rows of a slice list shared by the whole cluster: entry j covers
// ceil(len_j / kBigChunk) chunk tasks; task t goes to cluster warp t % nw.
template <bool DSM>
__device__ __forceinline__ void expand_slices(Ctx& x, const CtaItem* items, int64_t n, int64_t gwarp, int64_t nw,
                                              int lane) {
  int64_t base = 0;
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    CtaItem it{0, 0, 0};
    if (j0 + lane < n) {
      const int4 r = __ldcg(reinterpret_cast<const int4*>(items + j0 + lane));
      it.start = (int64_t)(((uint64_t)(uint32_t)r.y << 32) | (uint32_t)r.x);
      it.len = r.z;
      it.u = r.w;
    }
    const int nch = (it.len + kBigChunk - 1) / kBigChunk;
    int incl = nch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kF, incl, o);
      if (lane >= o) incl += t;
    }
    const int tot = __shfl_sync(kF, incl, 31);
    // first task id >= base owned by this warp
    int64_t t = base + ((gwarp - base % nw) % nw + nw) % nw;
    for (; t < base + tot; t += nw) {
      const int r = (int)(t - base);
      const int q = __ffs(__ballot_sync(kF, incl > r)) - 1;  // entry of task r
      const int c = r - (__shfl_sync(kF, incl, q) - __shfl_sync(kF, nch, q));
      const int64_t st = __shfl_sync(kF, it.start, q) + (int64_t)c * kBigChunk;
      const int32_t len = min(kBigChunk, __shfl_sync(kF, it.len, q) - c * kBigChunk);
      stream_slice<DSM>(x, st, len, __shfl_sync(kF, it.u, q), lane);
    }
    base += tot;
  }
}

// Rows of a list of degree >= 32 vertex ids (the queue format's warp bin).
template <bool DSM>
__device__ __forceinline__ void expand_warp_ids(Ctx& x, const int32_t* ids, int64_t n, int64_t gwarp, int64_t nw,
                                                int lane) {
  const ClusterArgs& p = *x.p;
  for (int64_t i = gwarp; i < n; i += nw) {
    const int32_t v = __ldcg(ids + i);
    const int64_t st = p.row_ptr[v];
    stream_slice<DSM>(x, st, (int32_t)(p.row_ptr[v + 1] - st), __ldg(p.new2old + v), lane);
  }
}

__device__ __forceinline__ Counters ld_counters_cg(const Counters* c) {
  Counters r;
  const ulonglong2* s = reinterpret_cast<const ulonglong2*>(c);
  ulonglong2* d = reinterpret_cast<ulonglong2*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Counters) / 16); ++i) d[i] = __ldcg(s + i);
  return r;
}

}  // namespace

template <bool DSM>
__global__ void __launch_bounds__(kClusterThreads, 1) k_cluster_levels(const __grid_constant__ ClusterArgs p) {
  extern __shared__ __align__(16) uint8_t s_dyn[];
  __shared__ ClusterSmem s;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  griddep_wait();  // (a programmatic dependent launch behind k_init_seed / k_compact)
  const unsigned long long t_start = gtimer();  // (the segment's device time goes to the mailbox: no events around it)
  Ctx x;
  x.wt = nullptr;
  x.wdone = 0;
  x.p = &p;
  x.s = &s;
  x.rank = cl_rank();
  x.csize = cl_size();
  x.clog = 31 - __clz(x.csize);
  uint32_t* slice = reinterpret_cast<uint32_t*>(s_dyn);
  const int64_t slice_words = DSM ? p.slice_words : 0;
  x.q0 = reinterpret_cast<QEntry*>(s_dyn + slice_words * 4);
  x.q1 = x.q0 + p.qs;
  x.stage = x.q1 + p.qs;
  x.mail = reinterpret_cast<unsigned long long*>(x.stage + kMaxCluster * kClusterStage);
  x.mail_cap = DSM ? p.mail_cap : 0;
  x.vis_base = (uint32_t)__cvta_generic_to_shared(slice);
  if (tid < kSmallMax + 2) s.T[tid] = p.classes->T[tid];
  if (tid < kSmallMax + 1) s.B[tid] = p.classes->base[tid];
  if (tid < (int)x.csize) {
    s.rbase[tid] = mapa(x.vis_base, (uint32_t)tid);
    s.rq[0][tid] = mapa((uint32_t)__cvta_generic_to_shared(x.q0), (uint32_t)tid);
    s.rq[1][tid] = mapa((uint32_t)__cvta_generic_to_shared(x.q1), (uint32_t)tid);
    s.rqcnt[tid] = mapa((uint32_t)__cvta_generic_to_shared(&s.qcnt[0]), (uint32_t)tid);
    s.rmail[tid] = mapa((uint32_t)__cvta_generic_to_shared(x.mail), (uint32_t)tid);
    s.rincnt[tid] = mapa((uint32_t)__cvta_generic_to_shared(&s.in_cnt[0]), (uint32_t)tid);
  }
  if (tid < kMaxCluster) s.out_cnt[tid] = s.in_cnt[tid] = 0;
  if (tid < 2) s.qcnt[tid] = 0;
  if (tid < kMaxCluster) s.scnt[tid] = 0;
  if (tid < 4) s.tm[tid] = 0;
  if (tid < 6) (&s.tot[0][0])[tid] = 0ull;
  // the frontier of level L0 (the host may not know it: read its counters here)
  const Counters c0 = ld_counters_cg(p.ring + p.L0 % kCounterRing);
  const int64_t n_in_small = (int64_t)c0.bin[kBinSmall], n_in_items = (int64_t)c0.bin[kBinCta];
  const int64_t n_in_warp = p.in_bitmap ? 0 : (int64_t)c0.bin[kBinWarp];
  const int64_t n_in_items2 = p.in_bitmap ? (int64_t)c0.bin[kBinWSlice] : 0;
  if (x.rank == 0 && tid == 0) {
    p.big_cnt[(p.L0 + 1) % kCounterRing] = 0ull;  // appended during level L0
    p.big_cnt[(p.L0 + 2) % kCounterRing] = 0ull;
  }
  const bool run = c0.discovered > 0 && cluster_takes(c0.discovered, c0.edges, p.exit_edges, p.exit_hub_edges) &&
                   p.max_levels > 0;
  if (DSM && run) {  // this CTA's sectors of the visited bitmap
    const int64_t nsec = (p.nwords + 7) / 8, my = slice_words / 8;
    if (p.root_orig >= 0) {  // first level of a BFS: visited = {root}
      for (int64_t i = tid; i < my * 2; i += kCT) reinterpret_cast<uint4*>(slice)[i] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      if (tid == 0) {
        const uint32_t r = (uint32_t)__ldg(p.old2new + p.root_orig), gw = r >> 5, sec = gw >> 3;
        if ((sec & (x.csize - 1)) == x.rank) slice[((sec >> x.clog) << 3) | (gw & 7u)] = 1u << (r & 31);
      }
    } else {
      for (int64_t i = tid; i < my * 2; i += kCT) {
        const int64_t sec = (i >> 1) * x.csize + x.rank;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (sec < nsec) v = __ldcg(reinterpret_cast<const uint4*>(p.visited) + sec * 2 + (i & 1));
        reinterpret_cast<uint4*>(slice)[i] = v;
      }
    }
  }
  unsigned long long* prof = (p.prof && x.rank == 0 && tid == 0) ? p.prof : nullptr;  // LBFS_CLUSTER_PROF
  if (prof) prof[0] = gtimer();
  const int64_t gwarp = (int64_t)wib * x.csize + x.rank;  // cluster-wide warp id (CTAs interleaved)
  const int64_t nw = (int64_t)kCW * x.csize;
  const uint32_t tot_base = (uint32_t)__cvta_generic_to_shared(&s.tot[0][0]);
  cl_sync();  // slices loaded, rbase / counters / big_cnt visible cluster-wide
  if (prof) prof[1] = gtimer();
  int64_t L = p.L0;
  unsigned long long in_disc = c0.discovered, in_edges = c0.edges;
  bool done = false;
  if (run) {
    for (;;) {
      const int cur = (int)(L & 1);
      const int ts = (int)(L % 3);
      x.nx = cur ^ 1;
      x.next_level = (int32_t)(L + 1);
      x.big_slot = (L + 1) % kCounterRing;
      x.disc = 0;
      x.edges = 0;
      x.wt = (p.prof && x.rank == 0 && L == p.prof_level) ? p.prof + 512 + 16 * wib : nullptr;
      x.wdone = 0;
      wstamp(x, 0, lane);
      if (x.rank == 0 && tid == 0 && L > p.L0)  // read during level L-1, appended from level L+1
        s.tm[3] = atomicExch(p.big_cnt + (L + 2) % kCounterRing, 0ull);  // (performed before the barrier)
      if (L == p.L0) {
        // external frontier (host queue format, or a bitmap level's list + slices);
        // its records were written by the level that found it
        const int64_t ng = (n_in_small + 31) / 32;
        for (int64_t g = gwarp; g < ng; g += nw) {
          const int n = (int)min((int64_t)32, n_in_small - g * 32);
          const int32_t v = lane < n ? __ldcg(p.in_small + g * 32 + lane) : 0;
          expand_small_group<DSM>(x, n, v, lane, wib);
        }
        expand_warp_ids<DSM>(x, p.in_warp, n_in_warp, gwarp, nw, lane);
        expand_slices<DSM>(x, p.in_items, n_in_items, gwarp, nw, lane);
        expand_slices<DSM>(x, p.in_items2, n_in_items2, gwarp, nw, lane);
      } else {
        const int32_t ns = s.qcnt[cur];
        const int64_t nb = (int64_t)__ldcg(p.big_cnt + L % kCounterRing);
        for (int32_t g = wib; g * 32 < ns; g += kCW) {
          const int n = min(32, ns - g * 32);
          const QEntry e = lane < n ? qget(x, cur, g * 32 + lane) : QEntry{0, 0};
          if (lane < n) write_record<DSM>(p, e, (int32_t)L);  // (fire and forget, early in the level)
          expand_small_group<DSM>(x, n, e.v, lane, wib);
        }
        if (nb) expand_slices<DSM>(x, p.big + (L % kCounterRing) * p.cap, nb, gwarp, nw, lane);
      }
      unsigned long long* pl = (prof && L - p.L0 < 64) ? prof + 8 + 4 * (L - p.L0) : nullptr;
      if (p.prof && lane == 0) atomicMax(&s.tm[2], gtimer());
      wstamp(x, 5, lane);
      if (x.mail_cap > 0) {
        // candidates delivered: every sender tells every owner how many it
        // wrote, the cluster barrier (release / acquire: the remote stores are
        // visible), then each CTA claims what it received
        __syncthreads();
        if (tid < (int)x.csize) {
          st_dsm32(s.rincnt[tid] + 4u * x.rank, (uint32_t)min(s.out_cnt[tid], x.mail_cap));
          s.out_cnt[tid] = 0;
        }
        cl_sync();
        wstamp(x, 3, lane);
        accept_mail(x, slice, lane, wib);
        wstamp(x, 4, lane);
      }
      // this CTA's counts, added into every CTA's totals of level L+1
      unsigned long long d = x.disc, e = x.edges;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        d += __shfl_xor_sync(kF, d, o);
        e += __shfl_xor_sync(kF, e, o);
      }
      if (lane == 0) {
        s.red[0][wib] = d;
        s.red[1][wib] = e;
      }
      __syncthreads();  // (also: this CTA's queue reads and stagings are complete)
      push_staged(x, lane, wib);
      wstamp(x, 6, lane);
      if (wib == 0) {
        d = lane < kCW ? s.red[0][lane] : 0ull;
        e = lane < kCW ? s.red[1][lane] : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          d += __shfl_xor_sync(kF, d, o);
          e += __shfl_xor_sync(kF, e, o);
        }
        const int ns1 = (ts + 1) % 3;
        unsigned long long r = 0;
        if (lane < (int)x.csize) {
          const uint32_t a = mapa(tot_base, (uint32_t)lane) + (uint32_t)(ns1 * 16);
          r = atom_add_dsm64(a, d) + atom_add_dsm64(a + 8, e);  // (returned: performed before the barrier)
        }
        if (__any_sync(kF, r == ~0ull) && lane == 0) s.tm[3] = r;  // (consume)
      }
      if (tid == 0) s.qcnt[cur] = 0;  // the consumed queue becomes level L+1's output
      // the totals this CTA read after the last barrier (slot L % 3) are next
      // added into in level L+2, after the next barrier
      if (tid < 2) s.tot[ts][tid] = 0ull;
      if (pl) {
        pl[0] = s.tm[0];  // last warp's loads back
        pl[1] = s.tm[1];  // last warp's claims back
        pl[2] = s.tm[2];  // last warp done
        s.tm[0] = s.tm[1] = s.tm[2] = 0;
      }
      cl_level_sync();
      wstamp(x, 7, lane);
      const unsigned long long td = s.tot[(ts + 1) % 3][0], te = s.tot[(ts + 1) % 3][1];
      if (pl) pl[3] = gtimer();
      if (x.rank == 0 && tid == 0)
        p.layers[L - p.L0] = lbfs_layer{(int64_t)in_disc, (int64_t)in_edges, (int64_t)td};
      ++L;
      in_disc = td;
      in_edges = te;
      if (td == 0) {
        done = true;
        break;
      }
      if (!cluster_takes(td, te, p.exit_edges, p.exit_hub_edges) || L - p.L0 >= p.max_levels) break;
    }
  }
  // ---- exit: the frontier of level L in the host's queue format (slot L % 3)
  Counters* outc = p.ring + L % kCounterRing;
  if (L > p.L0) {
    const int cur = (int)(L & 1);
    if (x.rank == 0 && tid == 0) {
      // slot L%3 is rebuilt here, slot (L+1)%3 must be zero for the host's next level
      Counters z{};
      z.discovered = in_disc;
      z.edges = in_edges;
      *outc = z;
      p.ring[(L + 1) % kCounterRing] = Counters{};
    }
    cl_sync();
    if (!done) {
      // small entries: records, then this CTA's range of the list from the
      // prefix of the CTAs' queue counts
      int64_t before = 0, total = 0;
      const uint32_t qa = (uint32_t)__cvta_generic_to_shared(&s.qcnt[cur]);
      for (uint32_t r = 0; r < x.csize; ++r) {
        const int64_t cnt = (int64_t)ld_dsm32(mapa(qa, r));
        if (r < x.rank) before += cnt;
        total += cnt;
      }
      const int32_t ns = s.qcnt[cur];
      int32_t* out_small = p.out_small[cur];
      for (int32_t i = tid; i < ns; i += kCT) {
        const QEntry e = qget(x, cur, i);
        write_record<DSM>(p, e, (int32_t)L);
        out_small[before + i] = e.v;
      }
      if (x.rank == 0 && tid == 0) outc->bin[kBinSmall] = (unsigned long long)total;
      // rows of degree >= 32 -> host slice items of <= qchunk edges
      const int64_t nb = (int64_t)__ldcg(p.big_cnt + L % kCounterRing);
      const CtaItem* bl = p.big + (L % kCounterRing) * p.cap;
      // (a bitmap-mode next level takes kChunk-edge slices, a queue-mode one qchunk)
      // a queue-mode level is a latency chain per 128-element window: cut the
      // items so that every warp of the full grid gets about one (>= 128 edges)
      const int fair = (int)min((unsigned long long)p.qchunk,
                                max(128ull, (in_edges / (unsigned long long)max(p.exit_warps, 1) + 127ull) & ~127ull));
      const int chunk = in_edges >= p.bitmap_min_edges ? kChunk : (p.exit_warps > 0 ? fair : p.qchunk);
      for (int64_t j0 = ((int64_t)x.rank * kCW + wib) * 32; j0 < nb; j0 += (int64_t)kCT * x.csize) {
        const int64_t j = j0 + lane;
        CtaItem it{0, 0, 0};
        if (j < nb) it = bl[j];
        const int items = j < nb ? slice_items(it.start, it.len, chunk) : 0;
        int incl = items;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(kF, incl, o);
          if (lane >= o) incl += t;
        }
        unsigned long long b = 0;
        if (lane == 31 && incl) b = atomicAdd(&outc->bin[kBinCta], (unsigned long long)incl);
        b = __shfl_sync(kF, b, 31) + (unsigned long long)(incl - items);
        for (int q = 0; q < 32; ++q) {  // the warp writes entry q's slices together
          const int nq = __shfl_sync(kF, items, q);
          const unsigned long long bq = __shfl_sync(kF, b, q);
          const int64_t sq = __shfl_sync(kF, it.start, q);
          const int32_t lq = __shfl_sync(kF, it.len, q), uq = __shfl_sync(kF, it.u, q);
          for (int k = lane; k < nq; k += 32)
            p.out_cta[cur][bq + k] = slice_item(sq, lq, chunk, k, uq);
        }
      }
    }
    cl_sync();  // (release: every store of the loop and the exit is performed)
  }
  if (prof) prof[2] = gtimer();
  if (L == p.L0 && x.rank == 0 && tid == 0) p.ring[(L + 1) % kCounterRing] = Counters{};  // the next level's slot
  if (x.rank == 0 && tid == 0 && p.mail) {
    Counters m = ld_counters_cg(outc);
    m.pad[0] = (unsigned long long)L;
    volatile unsigned long long* dst = reinterpret_cast<volatile unsigned long long*>(p.mail);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&m);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(Counters) / 8); ++i) dst[i] = src[i];
    reinterpret_cast<volatile unsigned long long*>(p.seq)[1] = gtimer() - t_start;  // ns inside this launch
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(p.seq) = p.seq_value;
  }
}

template __global__ void k_cluster_levels<true>(const __grid_constant__ ClusterArgs p);
template __global__ void k_cluster_levels<false>(const __grid_constant__ ClusterArgs p);

size_t cluster_static_smem() { return sizeof(ClusterSmem); }

}  // namespace lbfs
