// Weight/KV streaming engine shared by every cfb kernel.
//
// One producer warp (warp kNumConsumerWarps) streams a CTA's whole schedule of
// contiguous global rows into a ring of shared-memory slots with
// cp.async.bulk (TMA bulk copies) completing on per-slot mbarriers.  Each
// consumer warp owns `spw` private slots, so a slot is consumed by exactly
// one warp and no CTA-wide barrier is needed to recycle it.  Producer lane w
// feeds consumer warp w: the eight sub-rings refill independently (no
// head-of-line blocking behind a slow warp) and eight threads issue copies.
//
// A schedule is a list of Phases.  Weights and the KV cache never depend on
// the activations, so the producer runs ahead across phase boundaries (and
// across the DSMEM collectives the consumers wait on in between): the next
// phase's bytes are already in flight while the cluster exchanges partials.
#pragma once
#include "ptx.cuh"

namespace cfb {

constexpr int kNumConsumerWarps = 8;
constexpr int kThreads = (kNumConsumerWarps + 1) * 32;
constexpr int kConsumerThreads = kNumConsumerWarps * 32;
constexpr int kMaxSlotsPerWarp = 3;
constexpr int kNumSlots = kNumConsumerWarps * kMaxSlotsPerWarp;  // barrier storage
constexpr int kSlotBytes = 8192;
__host__ __device__ constexpr int ring_bytes(int spw) { return kNumConsumerWarps * spw * kSlotBytes; }
constexpr uint32_t kConsumerBar = 1;  // named barrier id for consumer-only sync

__device__ __forceinline__ void consumer_sync() { named_bar_sync(kConsumerBar, kConsumerThreads); }

// A phase streams `n_units` contiguous units of `unit_bytes` each from src0.
//   rows mode  (tiles == false): a unit is one K-major row (KV-cache rows,
//              W_out^T rows); paired phases carry the same rows of src0 and
//              src1 in the two halves of a slot (K and V).
//   tiles mode (tiles == true):  a unit is a 4-row tile of a row-tiled weight
//              matrix, [chunk][4 rows][16 B] (see gemv.cuh); a tile larger
//              than a slot is split into column pieces.
// Items (<= one slot) are dealt round-robin: item i goes to consumer warp i % 8
// (or all to one warp: warp_phase).
struct Phase {
  const char* src0;
  const char* src1;
  int n_units;
  int unit_bytes;
  int per_item;     // units per item (pieces == 1)
  int pieces;       // pieces per unit (> 1 only in tiles mode)
  int piece_bytes;
  int n_items;
  bool tiles;
  int warp;         // >= 0: every item goes to this consumer warp (warp-affine phase)
};
// A phase whose rows may live in a paged pool (rows mode only; pages == nullptr:
// contiguous).  Unit u is logical row row0 + u of 128-row pages; page g starts
// pages[g] * pstride bytes past src0/src1.  A separate type, so the kernels
// that never page keep the plain Phase (and its stack footprint).
constexpr int kPageRows = 128;
struct PagedPhase : Phase {
  const int* pages;
  int row0;
  long long pstride;
};

__device__ __forceinline__ Phase make_phase(const void* src0, const void* src1, int n_units,
                                            int unit_bytes, bool tiles = false) {
  Phase p;
  p.src0 = static_cast<const char*>(src0);
  p.src1 = static_cast<const char*>(src1);
  p.n_units = n_units < 0 ? 0 : n_units;
  p.unit_bytes = unit_bytes;
  p.tiles = tiles;
  p.warp = -1;
  const int cap = src1 ? kSlotBytes / 2 : kSlotBytes;
  if (unit_bytes <= cap) {
    p.per_item = cap / unit_bytes;
    p.pieces = 1;
    p.piece_bytes = unit_bytes;
    p.n_items = (p.n_units + p.per_item - 1) / p.per_item;
  } else {  // tiles mode only (checked on the host)
    p.per_item = 1;
    p.pieces = (unit_bytes + cap - 1) / cap;
    p.piece_bytes = cap;
    p.n_items = p.n_units * p.pieces;
  }
  return p;
}

struct Item {
  int unit0;   // first unit (row or tile)
  int nunits;  // units in this item (1 for pieces)
  int piece;   // piece index within the unit
  int byte0;   // byte offset of the piece within its unit
  int bytes;   // bytes per source
};

// Paged rows phase: the same units as `p`, unit u read from logical row
// row0 + u of the page pool (src0/src1 = the pool base of this head's rows);
// pages == nullptr keeps `p` contiguous.
__device__ __forceinline__ PagedPhase paged_phase(const Phase& p, const int* pages = nullptr, int row0 = 0,
                                                  long long pstride = 0) {
  PagedPhase q;
  static_cast<Phase&>(q) = p;
  q.pages = pages;
  q.row0 = row0;
  q.pstride = pstride;
  return q;
}

// Warp-affine phase: all items of the phase go to consumer warp `warp` (the
// warp then owns everything the phase produces, e.g. a block of output rows).
__device__ __forceinline__ Phase warp_phase(Phase p, int warp) {
  p.warp = warp;
  return p;
}

__device__ __forceinline__ int items_for_warp(const Phase& p, int w) {
  if (p.warp >= 0) return p.warp == w ? p.n_items : 0;
  return p.n_items > w ? (p.n_items - w + kNumConsumerWarps - 1) / kNumConsumerWarps : 0;
}

__device__ __forceinline__ Item item_of(const Phase& p, int w, int j) {
  const int i = p.warp >= 0 ? j : j * kNumConsumerWarps + w;
  Item it;
  if (p.pieces == 1) {
    it.unit0 = i * p.per_item;
    it.nunits = min(p.per_item, p.n_units - it.unit0);
    it.piece = 0;
    it.byte0 = 0;
    it.bytes = it.nunits * p.unit_bytes;
  } else {
    it.unit0 = i / p.pieces;
    it.nunits = 1;
    it.piece = i % p.pieces;
    it.byte0 = it.piece * p.piece_bytes;
    it.bytes = min(p.piece_bytes, p.unit_bytes - it.byte0);
  }
  return it;
}

struct Ring {
  char* slots;
  uint64_t* full;
  uint64_t* empty;
  int spw;        // slots per consumer warp
  int sleep_max;  // producer idle back-off cap (ns)
  __device__ __forceinline__ char* slot(int s) const { return slots + s * kSlotBytes; }
};

__device__ __forceinline__ void ring_init(const Ring& r) {
  for (int s = 0; s < kNumSlots; ++s) {
    mbar_init(&r.full[s], 1);
    mbar_init(&r.empty[s], 1);
  }
}

__device__ __forceinline__ void issue_item(const Phase& p, const Item& it, const Ring& r, int s,
                                           uint64_t policy) {
  const size_t off = static_cast<size_t>(it.unit0) * p.unit_bytes + it.byte0;
  mbar_arrive_expect_tx(&r.full[s], p.src1 ? 2u * it.bytes : static_cast<uint32_t>(it.bytes));
  bulk_g2s(r.slot(s), p.src0 + off, it.bytes, &r.full[s], policy);
  if (p.src1) bulk_g2s(r.slot(s) + kSlotBytes / 2, p.src1 + off, it.bytes, &r.full[s], policy);
}

// Paged rows: `pga` / `pgb` are the page ids of the item's first row and of the
// next page (an item of <= 16 rows spans at most two 128-row pages).
__device__ __forceinline__ void issue_item_paged(const PagedPhase& p, const Item& it, const Ring& r, int s,
                                                 uint64_t policy, int pga, int pgb) {
  mbar_arrive_expect_tx(&r.full[s], p.src1 ? 2u * it.bytes : static_cast<uint32_t>(it.bytes));
  const int r0 = p.row0 + it.unit0;
  const int n0 = min(it.nunits, kPageRows - (r0 & (kPageRows - 1)));
  const size_t o0 = (size_t)pga * p.pstride + (size_t)(r0 & (kPageRows - 1)) * p.unit_bytes;
  const int b0 = n0 * p.unit_bytes;
  bulk_g2s(r.slot(s), p.src0 + o0, b0, &r.full[s], policy);
  if (p.src1) bulk_g2s(r.slot(s) + kSlotBytes / 2, p.src1 + o0, b0, &r.full[s], policy);
  if (n0 < it.nunits) {
    const size_t o1 = (size_t)pgb * p.pstride;
    const int b1 = it.bytes - b0;
    bulk_g2s(r.slot(s) + b0, p.src0 + o1, b1, &r.full[s], policy);
    if (p.src1) bulk_g2s(r.slot(s) + kSlotBytes / 2 + b0, p.src1 + o1, b1, &r.full[s], policy);
  }
}

// Producer warp: lane w < kNumConsumerWarps feeds consumer warp w through
// its sub-ring, walking the phases in order.  `c` (per lane) counts the
// items issued so far, so a schedule may be produced in several calls (e.g.
// weights first, then - after a PDL wait - activation-dependent KV rows).  The loop is warp-uniform and
// only probes slots with the non-blocking test_wait, so one lane waiting for
// a busy slot never stalls the others (a blocking try_wait in divergent
// lanes would serialise the warp).
template <int NP>
__device__ __forceinline__ void produce_all(const Phase (&P)[NP], const Ring& r, int lane,
                                            uint64_t policy, int& c) {
  const int w = lane;
  int ph = 0, j = 0;
  bool done = w >= kNumConsumerWarps;
  int nap = 32;
  while (true) {
    bool issued = false;
    if (!done) {
      while (ph < NP && j >= items_for_warp(P[ph], w)) {
        ++ph;
        j = 0;
      }
      if (ph == NP) {
        done = true;
      } else {
        const int s = w * r.spw + (c % r.spw);
        if (mbar_test(&r.empty[s], ((c / r.spw) & 1) ^ 1)) {
          issue_item(P[ph], item_of(P[ph], w, j), r, s, policy);
          ++c;
          ++j;
          issued = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    // idle: exponential back-off, so a producer waiting on full sub-rings does
    // not steal issue slots from the consumer warps sharing its SM sub-partition
    if (__any_sync(0xffffffffu, issued)) {
      nap = 32;
    } else {
      __nanosleep(nap);
      nap = min(2 * nap, r.sleep_max);
    }
  }
}
// Same walk over `np` phases produced on the fly by gen(k) (no phase array:
// a long schedule indexed dynamically would live in local memory).
template <class Gen>
__device__ __forceinline__ void produce_gen(int np, Gen&& gen, const Ring& r, int lane, uint64_t policy,
                                            int& c) {
  const int w = lane;
  int ph = 0, j = 0;
  Phase cur = gen(0);
  bool done = w >= kNumConsumerWarps || np == 0;
  int nap = 32;
  while (true) {
    bool issued = false;
    if (!done) {
      while (ph < np && j >= items_for_warp(cur, w)) {
        ++ph;
        j = 0;
        if (ph < np) cur = gen(ph);
      }
      if (ph == np) {
        done = true;
      } else {
        const int s = w * r.spw + (c % r.spw);
        if (mbar_test(&r.empty[s], ((c / r.spw) & 1) ^ 1)) {
          issue_item(cur, item_of(cur, w, j), r, s, policy);
          ++c;
          ++j;
          issued = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (__any_sync(0xffffffffu, issued)) {
      nap = 32;
    } else {
      __nanosleep(nap);
      nap = min(2 * nap, r.sleep_max);
    }
  }
}

// produce_gen for a schedule whose phases may read paged rows (gen returns
// PagedPhase).  The page ids of the CTA's rows are held in the producer
// warp's registers - lane l keeps page p0 + 32 k + l in pg[k] (loaded once per
// launch: the rows of a CTA's segment sit on the same pages in every layer and
// head) - and read with shuffles in the convergent part of every loop trip, so
// no bulk copy waits on a dependent global load of the block table.
constexpr int kPageRegs = 4;  // <= 128 pages per CTA segment
template <class Gen>
__device__ __forceinline__ void produce_gen_paged(int np, Gen&& gen, const Ring& r, int lane, uint64_t policy,
                                                  int& c, const int (&pg)[kPageRegs], int p0) {
  const int w = lane;
  int ph = 0, j = 0;
  PagedPhase cur = gen(0);
  bool done = w >= kNumConsumerWarps || np == 0;
  int nap = 32;
  while (true) {
    bool issued = false, cand = false;
    Item it{};
    int rel = 0;
    if (!done) {
      while (ph < np && j >= items_for_warp(cur, w)) {
        ++ph;
        j = 0;
        if (ph < np) cur = gen(ph);
      }
      if (ph == np) {
        done = true;
      } else {
        cand = true;
        it = item_of(cur, w, j);
        if (cur.pages) rel = (cur.row0 + it.unit0) / kPageRows - p0;
      }
    }
    // pages of this item (rel, rel + 1) and of the lane's next item, 128 rows
    // further (rel + 1, rel + 2); every lane: convergent shuffles
    int pga = 0, pgb = 0, pgc = 0;
#pragma unroll
    for (int k = 0; k < kPageRegs; ++k) {
      const int va = __shfl_sync(0xffffffffu, pg[k], rel & 31);
      const int vb = __shfl_sync(0xffffffffu, pg[k], (rel + 1) & 31);
      const int vc = __shfl_sync(0xffffffffu, pg[k], (rel + 2) & 31);
      if ((rel >> 5) == k) pga = va;
      if (((rel + 1) >> 5) == k) pgb = vb;
      if (((rel + 2) >> 5) == k) pgc = vc;
    }
    if (cand) {
      const int s = w * r.spw + (c % r.spw);
      if (mbar_test(&r.empty[s], ((c / r.spw) & 1) ^ 1)) {
        if (cur.pages)
          issue_item_paged(cur, it, r, s, policy, pga, pgb);
        else
          issue_item(cur, it, r, s, policy);
        ++c;
        ++j;
        issued = true;
        // paged rows: a producer that fell behind refills two slots per trip
        // (the paged trip is longer); the lane's next item of the phase sits
        // one page further (rows + 128)
        if (cur.pages && j < items_for_warp(cur, w)) {
          const int s2 = w * r.spw + (c % r.spw);
          const Item it2 = item_of(cur, w, j);
          if ((cur.row0 + it2.unit0) / kPageRows - p0 == rel + 1 &&
              mbar_test(&r.empty[s2], ((c / r.spw) & 1) ^ 1)) {
            issue_item_paged(cur, it2, r, s2, policy, pgb, pgc);
            ++c;
            ++j;
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (__any_sync(0xffffffffu, issued)) {
      nap = 32;
    } else {
      __nanosleep(nap);
      nap = min(2 * nap, r.sleep_max);
    }
  }
}

template <int NP>
__device__ __forceinline__ void produce_all(const Phase (&P)[NP], const Ring& r, int lane,
                                            uint64_t policy) {
  int c = 0;
  produce_all(P, r, lane, policy, c);
}

// Consumer side: warp `w` walks its items; f(item, slot_ptr) runs warp-wide.
template <class F>
__device__ __forceinline__ void consume_phase(const Phase& p, const Ring& r, int w, int lane,
                                              int& cnt, F&& f) {
  const int n = items_for_warp(p, w);
  for (int j = 0; j < n; ++j) {
    const Item it = item_of(p, w, j);
    const int c = cnt++;
    const int s = w * r.spw + (c % r.spw);
    mbar_wait(&r.full[s], (c / r.spw) & 1);
    f(it, r.slot(s));
    __syncwarp();
    if (lane == 0) mbar_arrive(&r.empty[s]);
  }
}

// Load `n` consecutive elements of type T starting at p (16-byte aligned
// when n*sizeof(T) >= 16) into floats.
template <typename T, int n>
__device__ __forceinline__ void load_elems(const T* p, float* out) {
  constexpr int bytes = n * static_cast<int>(sizeof(T));
  if constexpr (bytes >= 16) {
#pragma unroll
    for (int i = 0; i < bytes / 16; ++i) {
      const uint4 v = lds128(reinterpret_cast<const char*>(p) + 16 * i);
      Elem<T>::unpack(v, out + i * Elem<T>::kPerVec);
    }
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) out[i] = Elem<T>::to_f(p[i]);
  }
}

}  // namespace cfb
