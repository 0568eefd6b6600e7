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

// `n_rows` rows of `row_bytes` each, contiguous from src0.  When src1 is set
// ("paired"), item k carries the same rows of src0 and src1 in the two halves
// of a slot (K and V cache rows).  Rows that do not fit a slot are split into
// pieces that all go to the same consumer warp, in order.
struct Phase {
  const char* src0;
  const char* src1;
  int n_rows;
  int row_bytes;
  int rows_per_item;
  int pieces;
  int piece_bytes;
};

__device__ __forceinline__ Phase make_phase(const void* src0, const void* src1, int n_rows,
                                            int row_bytes) {
  Phase p;
  p.src0 = static_cast<const char*>(src0);
  p.src1 = static_cast<const char*>(src1);
  p.n_rows = n_rows < 0 ? 0 : n_rows;
  p.row_bytes = row_bytes;
  const int cap = src1 ? kSlotBytes / 2 : kSlotBytes;
  if (row_bytes <= cap) {
    p.rows_per_item = cap / row_bytes;
    p.pieces = 1;
    p.piece_bytes = row_bytes;
  } else {  // paired phases never need pieces (row <= 4 KB checked on host)
    p.rows_per_item = 1;
    p.pieces = (row_bytes + cap - 1) / cap;
    p.piece_bytes = cap;
  }
  return p;
}

struct Item {
  int row0;     // first row
  int nrows;    // rows in this item (1 for pieces)
  int piece;    // piece index within the row
  int byte0;    // byte offset of the piece within its row
  int bytes;    // bytes per source
};

__device__ __forceinline__ int items_for_warp(const Phase& p, int w) {
  if (p.pieces == 1) {
    const int n_items = (p.n_rows + p.rows_per_item - 1) / p.rows_per_item;
    return n_items > w ? (n_items - w + kNumConsumerWarps - 1) / kNumConsumerWarps : 0;
  }
  const int rows_w = p.n_rows > w ? (p.n_rows - w + kNumConsumerWarps - 1) / kNumConsumerWarps : 0;
  return rows_w * p.pieces;
}

__device__ __forceinline__ Item item_of(const Phase& p, int w, int j) {
  Item it;
  if (p.pieces == 1) {
    const int i = j * kNumConsumerWarps + w;
    it.row0 = i * p.rows_per_item;
    it.nrows = min(p.rows_per_item, p.n_rows - it.row0);
    it.piece = 0;
    it.byte0 = 0;
    it.bytes = it.nrows * p.row_bytes;
  } else {
    it.row0 = (j / p.pieces) * kNumConsumerWarps + w;
    it.nrows = 1;
    it.piece = j % p.pieces;
    it.byte0 = it.piece * p.piece_bytes;
    it.bytes = min(p.piece_bytes, p.row_bytes - it.byte0);
  }
  return it;
}

struct Ring {
  char* slots;
  uint64_t* full;
  uint64_t* empty;
  int spw;  // slots per consumer warp
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
  const size_t off = static_cast<size_t>(it.row0) * p.row_bytes + it.byte0;
  mbar_arrive_expect_tx(&r.full[s], p.src1 ? 2u * it.bytes : static_cast<uint32_t>(it.bytes));
  bulk_g2s(r.slot(s), p.src0 + off, it.bytes, &r.full[s], policy);
  if (p.src1) bulk_g2s(r.slot(s) + kSlotBytes / 2, p.src1 + off, it.bytes, &r.full[s], policy);
}

// Producer warp: lane w < kNumConsumerWarps feeds consumer warp w through
// its sub-ring, walking the phases in order.  The loop is warp-uniform and
// only probes slots with the non-blocking test_wait, so one lane waiting for
// a busy slot never stalls the others (a blocking try_wait in divergent
// lanes would serialise the warp).
template <int NP>
__device__ __forceinline__ void produce_all(const Phase (&P)[NP], const Ring& r, int lane,
                                            uint64_t policy) {
  const int w = lane;
  int ph = 0, j = 0, c = 0;
  bool done = w >= kNumConsumerWarps;
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
    if (!__any_sync(0xffffffffu, issued)) __nanosleep(32);
  }
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
