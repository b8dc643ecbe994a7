// gc_kernels.cu -- the B200 (sm_100a) decode path and the C ABI of include/gc.h.
//
// Hot path of gc_decode_dgaps:
//   1. k_index  (subsystem (a)): control-space tiles of 2048
//      words parse every control word, run a device-wide segmented exclusive scan
//      (block scan + decoupled look-back, segmented by list) of (quads, data
//      lane-bits, exception bytes), and write one Entry per output tile: where the
//      quad containing output position t*kT starts in the control, data and
//      exception streams.
//   2. k_decode (subsystems (b)-(d), a3-a6): output-space tiles of 4096 ints.  A
//      tile stages its control words, data vectors and exceptions into shared
//      memory with 1-D bulk async copies (TMA engine), re-parses its control words
//      from the Entry (block scans), expands groups into per-quad descriptors,
//      unpacks one quad per thread-slot with shift/mask over the four vertical
//      lanes (the paper's high-first split for values that cross a word), patches
//      Group-PFD exceptions in shared memory, runs the segmented d-gap inclusive
//      scan (thread-serial + block + decoupled look-back across tiles) and writes
//      the tile with coalesced 128-bit stores.
#include <cuda.h>  // CUtensorMap (the decode's TMA tile stores)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "gc.h"
#include "gc_codecs.cuh"
#include "gc_device.cuh"

namespace gcd {

struct Dev {
  uint64_t n_lists;
  const uint32_t* list_n;
  const uint64_t* ctrl_off;
  const uint64_t* data_off;
  const uint64_t* exc_off;
  const uint64_t* out_off;
  const uint32_t* ctrl_words;
  uint64_t n_ctrl_words;
  const uint4* data;
  uint64_t data_vectors;
  const uint8_t* exc;
  uint64_t exc_bytes;
  uint64_t total_out;
  uint32_t n_tiles_a, n_tiles_b;
  uint32_t wa;            // control words per index tile (kWA, or kWASmall for small batches)
  WsHeader* hdr;
  TileA* tiles_a;
  uint64_t* tiles_b;
  Entry* entries;
  uint32_t* first_list;   // [n_tiles_a] 1 + owner list of the first word of control tile a
  // skip pointers (gc_build_skip: k_index writes them; gc_decode_range reads them)
  const uint32_t* docids;         // the batch's d-gap decode (the blocks' carries)
  uint64_t* skip_off;             // [n_lists + 1]
  gc_skip_entry* skip;            // [skip_off[n_lists]]
};


// Per-list view used by the group walks of the index kernel.
struct ListCur {
  uint64_t l;        // list index
  uint64_t n, Q;     // ints, quads
  uint64_t dbase;    // data_off * 32 (lane bits)
  uint64_t dlim, elim;  // data_off[l+1]*32, exc_off[l+1]
  __device__ void load(const Dev& D, uint64_t li) {
    l = li;
    n = D.list_n[li];
    Q = (n + 3) >> 2;
    dbase = D.data_off[li] * 32ull;
    dlim = D.data_off[li + 1] * 32ull;
    elim = D.exc_off ? D.exc_off[li + 1] : 0ull;
  }
};

// Largest l in [lo, hi) with off[l] <= key (assumes off[lo] <= key).
__device__ __forceinline__ uint64_t find_list(const uint64_t* off, uint64_t lo, uint64_t hi,
                                              uint64_t key) {
  uint64_t a = lo, b = hi;
  while (b - a > 1) {
    uint64_t m = (a + b) >> 1;
    if (off[m] <= key)
      a = m;
    else
      b = m;
  }
  return a;
}

__device__ __forceinline__ void report(uint32_t* s_err, uint32_t bits) {
  if (bits) atomicOr(s_err, bits);
}

// =====================================================================================
// k_lists: one thread per list.  Directory consistency (out_off must be the exclusive
// scan of list_n, offsets monotone and inside the streams, every non-empty list owns at
// least one control word) and the control-tile map: first_list[a] = 1 + the list owning
// control word a*wa (control areas are contiguous and 4-byte aligned).
// =====================================================================================
__global__ void __launch_bounds__(kThreads) k_lists(Dev D) {
  uint32_t err = 0;
  for (uint64_t l = (uint64_t)blockIdx.x * kThreads + threadIdx.x; l < D.n_lists;
       l += (uint64_t)gridDim.x * kThreads) {
    const uint64_t n = D.list_n[l];
    const uint64_t c0 = D.ctrl_off[l], c1 = D.ctrl_off[l + 1];
    const uint64_t d0 = D.data_off[l], d1 = D.data_off[l + 1];
    const uint64_t o0 = D.out_off[l], o1 = D.out_off[l + 1];
    bool bad = (o1 != o0 + n) || (c1 < c0) || (d1 < d0) || ((c0 | c1) & 3) ||
               (c1 > 4 * D.n_ctrl_words) || (d1 > D.data_vectors) || (o1 > D.total_out) ||
               (n > 0 && c1 == c0);
    if (D.exc_off) {
      const uint64_t e0 = D.exc_off[l], e1 = D.exc_off[l + 1];
      bad = bad || (e1 < e0) || (e1 > D.exc_bytes);
    }
    if (l == 0) bad = bad || (o0 != 0) || (c0 != 0);
    if (l + 1 == D.n_lists) bad = bad || (o1 != D.total_out);
    if (bad) {
      err |= GC_DEV_TRUNCATED;
      continue;
    }
    const uint64_t w0 = c0 >> 2, w1 = c1 >> 2;
    const uint32_t sh = D.wa == kWA ? 11u : 8u;  // log2 of the tile size (no 64-bit division)
    static_assert(kWA == 2048u && kWASmall == 256u, "tile sizes");
    for (uint64_t a = (w0 + D.wa - 1) >> sh; (a << sh) < w1 && a < D.n_tiles_a; a++)
      D.first_list[a] = (uint32_t)(l + 1);
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if ((threadIdx.x & 31) == 0 && err) atomicOr(&D.hdr->status, err);
}

// =====================================================================================
// k_index (subsystem (a)): device-wide segmented scan over the control stream.
// Control-space tiles of kWA words, 8 per thread.  Each word is parsed on its own into
// (raw quads, data lane-bits, exception bytes); a block scan segmented at list starts
// plus a decoupled look-back across tiles give every word its exact position in its
// list.  The word holding the quadruple of output int t*kT writes Entry[t]; the last
// word of every list (and any word a cheap test finds suspicious) is walked group by
// group to check the list's bounds and the group codes.
// =====================================================================================

// The group walk of one control word gw (word widx of list l, its groups starting at
// quad q0, data lane-bit d0, exception byte e0): group codes, and every group of the list
// inside the list's data / exception range.  Returns status bits.  Out of line: k_index
// calls it from the walk queue and, when the queue is full, in place.
struct WalkArgs {  // (by value: a kernel parameter passed by reference would be copied to the stack)
  const uint32_t* ctrl_words;
  const uint32_t* list_n;
  const uint64_t* data_off;
  const uint64_t* exc_off;
};
template <class C>
__device__ __noinline__ uint32_t index_walk_word(WalkArgs A, uint64_t gw, uint32_t widx, uint64_t l,
                                                 uint64_t q0, uint64_t d0, uint64_t e0) {
  uint32_t err = 0;
  const uint32_t w = A.ctrl_words[gw];
  const uint32_t pv = (C::kNeedsPrev && widx > 0) ? A.ctrl_words[gw - 1] : 0u;
  const uint64_t Q = (A.list_n[l] + 3ull) >> 2;
  const uint64_t dbase = A.data_off[l] * 32ull, dlim = A.data_off[l + 1] * 32ull;
  const uint64_t elim = A.exc_off ? A.exc_off[l + 1] : 0ull;
  const WCtx c{w, pv, widx, Q, 0u};
  word_walk<C>(c, [&](const Grp& g) {
    const uint64_t gq = q0 + g.q0;
    if (gq >= Q) return;
    if (g.err) err |= g.err;
    if (g.nq == 0) return;
    const uint64_t gdata = d0 + (int64_t)g.d0;
    const uint64_t gexc = e0 + g.e0;
    if (gdata < dbase || gdata + g.dlen > dlim) err |= GC_DEV_TRUNCATED;
    if (C::kExc && gexc + g.elen > elim) err |= GC_DEV_TRUNCATED;
  });
  return err;
}

#ifndef GC_INDEX_MINB
#define GC_INDEX_MINB 4
#endif
// SKIP: also write the skip entries (gc_build_skip); the decode path's instantiation has
// none of that code (it cost the decode's index stage ~10% in registers and issue).
template <class C, uint32_t CA, bool SKIP>
__global__ void __launch_bounds__(kThreads, GC_INDEX_MINB) k_index(Dev D) {
  constexpr uint32_t WA = CA * kThreads;  // control words per tile (== D.wa)
  constexpr uint32_t kLTA = WA + 2;       // list table entries (the lists of one tile)
  __shared__ uint32_t s_cw[kLTA + 1];           // first word of list la+i, relative to w0 (wraps)
  __shared__ uint32_t s_n[kLTA];                // ints of list la+i
  __shared__ unsigned long long s_o[kLTA];      // out_off of list la+i
  __shared__ Seg4 s_scr[kWarps];
  __shared__ uint32_t s_tile, s_err, s_nq, s_nl, s_nw, s_lastli, s_pq;
  __shared__ unsigned long long s_la, s_pd, s_pe;
  constexpr uint32_t kQueue = 3 * kThreads / 2;  // words needing a group walk (list ends, suspicious)
  __shared__ uint32_t s_qw[kQueue], s_qi[kQueue], s_qq[kQueue];
  __shared__ unsigned long long s_qd[kQueue], s_qe[C::kExc ? kQueue : 1];
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    const uint32_t tile = atomicAdd(&D.hdr->counter_a, 1u);
    s_tile = tile;
    s_err = 0;
    s_nq = 0;
    s_lastli = 0;
    const uint64_t w0 = (uint64_t)tile * WA;
    const uint64_t cend = D.n_lists ? mn64(D.ctrl_off[D.n_lists] >> 2, D.n_ctrl_words) : 0;
    uint64_t nw = cend > w0 ? mn64(WA, cend - w0) : 0;
    uint64_t la = 0, nl = 0;
    if (nw) {
      const uint32_t f = D.first_list[tile];
      if (f == 0) {
        s_err = GC_DEV_TRUNCATED;  // the directory does not cover this word
        nw = 0;
      } else {
        la = f - 1;
        uint64_t lb = D.n_lists - 1;
        if (tile + 1 < D.n_tiles_a && D.first_list[tile + 1]) lb = D.first_list[tile + 1] - 1;
        nl = lb >= la ? lb - la + 1 : 0;
        if (!nl) nw = 0;
      }
    }
    s_la = la;
    s_nl = (uint32_t)mn64(nl, 0xFFFFFFFFull);
    s_nw = (uint32_t)nw;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t w0 = (uint64_t)tile * WA;
  const uint32_t nw = s_nw, nl = s_nl;
  const uint64_t la = s_la;
  const bool big = nl > kLTA;  // (runs of empty lists) look the table up in global memory
  if (!big) {
    for (uint32_t i = tid; i <= nl && nw; i += kThreads) {
      s_cw[i] = (uint32_t)((D.ctrl_off[la + i] >> 2) - w0);
      if (i < nl) {
        s_n[i] = D.list_n[la + i];
        s_o[i] = D.out_off[la + i];
      }
    }
  }
  __syncthreads();
  auto cw_at = [&](uint32_t i) -> uint32_t {
    return big ? (uint32_t)((D.ctrl_off[la + i] >> 2) - w0) : s_cw[i];
  };
  auto n_at = [&](uint32_t i) -> uint32_t { return big ? D.list_n[la + i] : s_n[i]; };
  auto o_at = [&](uint32_t i) -> uint64_t { return big ? D.out_off[la + i] : s_o[i]; };

  // ---- words of this thread (8 consecutive, two 128-bit loads)
  const uint32_t r0 = tid * CA;
  const uint32_t myn = r0 < nw ? min(CA, nw - r0) : 0u;
  uint32_t wv[CA];
  if constexpr (CA == 8) {
    if (myn == CA) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(D.ctrl_words + w0 + r0));
      const uint4 y = __ldg(reinterpret_cast<const uint4*>(D.ctrl_words + w0 + r0) + 1);
      wv[0] = x.x; wv[1] = x.y; wv[2] = x.z; wv[3] = x.w;
      wv[4] = y.x; wv[5] = y.y; wv[6] = y.z; wv[7] = y.w;
    } else {
#pragma unroll
      for (uint32_t k = 0; k < CA; k++) wv[k] = k < myn ? D.ctrl_words[w0 + r0 + k] : 0u;
    }
  } else {
#pragma unroll
    for (uint32_t k = 0; k < CA; k++) wv[k] = k < myn ? D.ctrl_words[w0 + r0 + k] : 0u;
  }
  uint32_t pw = __shfl_up_sync(0xffffffffu, wv[CA - 1], 1);
  if (lane == 0) pw = (C::kNeedsPrev && myn && w0 + r0 > 0) ? D.ctrl_words[w0 + r0 - 1] : 0u;

  uint32_t li = 0;
  if (myn) {  // the last table entry whose first word is <= r0 (entry 0 is the owner of w0)
    uint32_t a = 0, b = nl;
    while (b - a > 1) {
      const uint32_t m = (a + b) >> 1;
      if (cw_at(m) <= r0) a = m;
      else b = m;
    }
    li = a;
  }
  // pass 1: per-word aggregates, segmented at list starts
  Seg4 agg{0, 0, 0, 0};
  WAgg wa_[CA];
  uint32_t wli[CA];
  // the current list's first word and length and the next list's first word, reloaded only
  // when a word crosses into the next list (a thread's 8 words mostly share one list)
  uint32_t cur_cw = 0, cur_n = 0, next_cw = 0xFFFFFFFFu;
  if (myn) {
    cur_cw = cw_at(li);
    cur_n = n_at(li);
    next_cw = li + 1 < nl ? cw_at(li + 1) : 0xFFFFFFFFu;
  }
#pragma unroll
  for (uint32_t k = 0; k < CA; k++) {
    wa_[k] = WAgg{0, 0, 0};
    wli[k] = li;
    if (k < myn) {
      const uint32_t wr = r0 + k;
      if (next_cw <= wr) {
        do {
          li++;
          cur_cw = next_cw;
          next_cw = li + 1 < nl ? cw_at(li + 1) : 0xFFFFFFFFu;
        } while (next_cw <= wr);
        cur_n = n_at(li);
      }
      wli[k] = li;
      const uint32_t widx = wr - cur_cw;
      const WCtx c{wv[k], k ? wv[k - 1] : pw, widx, (cur_n + 3ull) >> 2, 0u};
      const WAgg a = word_agg<C>(c);
      wa_[k] = a;
      agg = widx == 0 ? Seg4{1u, a.q, a.d, a.e} : Seg4{agg.f, agg.q + a.q, agg.d + a.d, agg.e + a.e};
    }
  }
  if (myn && r0 + myn == nw) s_lastli = wli[myn - 1];
  Seg4 total;
  const Seg4 excl = block_excl_seg4<C::kExc>(agg, s_scr, &total);

  // ---- decoupled look-back across control tiles (warp 0, 32 predecessors per round
  // trip); values are absolute
  if (tid < 32) {
    TileA* me = D.tiles_a + tile;
    const bool first_reset = nw == 0 || cw_at(0) == 0;
    if (tid == 0) {
      uint64_t bd = 0, be = 0;  // absolute base of the tile's last segment (if it starts here)
      if (total.f) {
        const uint64_t l = la + s_lastli;
        bd = D.data_off[l] * 32ull;
        be = D.exc_off ? D.exc_off[l] : 0ull;
      }
      uint64_t w0, w1;
      if (total.f || nw == 0) {
        tilea_pack(total.q, bd + total.d, be + total.e, w0, w1);
        st_relaxed_u64(&me->i1, w1);
        st_relaxed_u64(&me->i0, w0);
      } else {
        tilea_pack(total.q, total.d, total.e, w0, w1);
        st_relaxed_u64(&me->a1, w1);
        st_relaxed_u64(&me->a0, w0);
      }
    }
    uint32_t pq = 0;
    uint64_t pd = 0, pe = 0;
    if (!first_reset) {
      lookback_tilea(D.tiles_a, tile, pq, pd, pe);
      if (tid == 0 && !total.f) {
        uint64_t w0, w1;
        tilea_pack(pq + total.q, pd + total.d, pe + total.e, w0, w1);
        st_relaxed_u64(&me->i1, w1);
        st_relaxed_u64(&me->i0, w0);
      }
    }
    if (tid == 0) {
      s_pq = pq;
      s_pd = pd;
      s_pe = pe;
    }
  }
  __syncthreads();

  // ---- pass 2: absolute positions per word; tile Entries; queue words to walk
  uint32_t err = 0;
  // group walk of one word (out of line: one copy of the codec's walk in the kernel)
  auto walk_word = [&](uint32_t wr, uint32_t i, uint64_t q0, uint64_t d0, uint64_t e0) {
    GC_CHECK(w0 + wr < D.n_ctrl_words);
    err |= index_walk_word<C>(WalkArgs{D.ctrl_words, D.list_n, D.data_off, D.exc_off}, w0 + wr,
                              wr - cw_at(i), la + i, q0, d0, e0);
  };
  uint32_t cq = 0;
  uint64_t cd = 0, ce = 0;
  if (myn) {
    if (excl.f) {  // the list of my first word started inside this tile
      const uint64_t l = la + wli[0];
      cq = excl.q;
      cd = D.data_off[l] * 32ull + excl.d;
      ce = (D.exc_off ? D.exc_off[l] : 0ull) + excl.e;
    } else {
      cq = s_pq + excl.q;
      cd = s_pd + excl.d;
      ce = s_pe + excl.e;
    }
  }
  // the current list's values, reloaded only when the list changes (a thread's 8 words
  // mostly belong to one list)
  uint32_t ci = ~0u, c_cw = 0, c_cwn = 0, c_n = 0;
  uint64_t c_o = 0;
#pragma unroll
  for (uint32_t k = 0; k < CA; k++) {
    if (k >= myn) break;
    const uint32_t wr = r0 + k;
    const uint32_t i = wli[k];
    const uint64_t l = la + i;
    if (i != ci) {
      ci = i;
      c_cw = cw_at(i);
      c_cwn = cw_at(i + 1);
      c_n = n_at(i);
      c_o = o_at(i);
    }
    const uint32_t widx = wr - c_cw;
    const WAgg a = wa_[k];
    if (widx == 0) {
      cq = 0;
      cd = D.data_off[l] * 32ull;
      ce = D.exc_off ? D.exc_off[l] : 0ull;
    }
    const uint32_t n = c_n;
    const uint64_t Q = (n + 3ull) >> 2;
    const uint64_t qa = cq, qb = mn64((uint64_t)cq + a.q, Q);
    if (qb > qa) {
      const uint64_t o = c_o;
      const uint64_t lo = o + 4 * qa, hi = o + mn64(4 * qb, n);
      const uint64_t t = (lo + kT - 1) / kT;
      if (t * kT < hi && t < D.n_tiles_b) {
        Entry e;
        e.l = (uint32_t)l;
        e.k = (uint32_t)((t * kT - o) >> 2);
        e.wq = cq;
        e.valid = 1;
        e.w = w0 + wr;
        e.wd = cd;
        e.we = ce;
        e.wd_end = cd + a.d;
        e.we_end = ce + a.e;
        e.pad = 0;
        GC_CHECK(t < D.n_tiles_b);
        D.entries[t] = e;
      }
    }
    if (SKIP && n > 0) {
      // skip pointers (§7.5): this word owns the first quad 128b of blocks b
      // with 128b in [cq, cq + a.q), b < ceil(n / 512)
      const uint64_t nblk = (n + GC_SKIP_DIST - 1) / GC_SKIP_DIST;
      for (uint64_t blk = (cq + 127) / 128; blk < nblk && 128 * blk < (uint64_t)cq + a.q; blk++) {
        const uint64_t e = D.skip_off[l] + blk;
        GC_CHECK(e < D.skip_off[l + 1]);
        gc_skip_entry s;
        s.data_bits = cd - D.data_off[l] * 32ull;
        s.word = widx;
        s.quads = cq;
        s.exc_bytes = (uint32_t)(ce - (D.exc_off ? D.exc_off[l] : 0ull));
        s.docid = blk ? D.docids[c_o + GC_SKIP_DIST * blk - 1] : 0u;
        s.pad[0] = s.pad[1] = 0;
        D.skip[e] = s;
      }
    }
    const bool last = c_cwn == wr + 1;
    const WCtx c{wv[k], k ? wv[k - 1] : pw, widx, Q, 0u};
    if (last && (uint64_t)cq + a.q < Q) err |= GC_DEV_TRUNCATED;  // control ends before Q quads
    if (last || C::suspect(c)) {
      // compact the words that need a group walk so the walks run lane-dense
      const uint32_t slot = atomicAdd(&s_nq, 1u);
      if (slot < kQueue) {
        s_qw[slot] = wr;
        s_qi[slot] = i;
        s_qq[slot] = cq;
        s_qd[slot] = cd;
        if (C::kExc) s_qe[slot] = ce;
      } else {
        walk_word(wr, i, cq, cd, ce);  // queue full: walk in place
      }
    }
    cq += a.q;
    cd += a.d;
    ce += a.e;
  }
  __syncthreads();
  const uint32_t nq = min(s_nq, kQueue);
  for (uint32_t x = tid; x < nq; x += kThreads)
    walk_word(s_qw[x], s_qi[x], s_qq[x], s_qd[x], C::kExc ? (uint64_t)s_qe[x] : 0ull);
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0) report(&s_err, err);
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(&D.hdr->status, s_err);
}

#include "gc_decode.cuh"
#include "gc_skip.cuh"

// =====================================================================================
// checksum (verification only, G7)
// =====================================================================================
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_checksum(const uint32_t* __restrict__ list_n, const uint64_t* __restrict__ out_off,
                           uint64_t n_lists, const uint32_t* __restrict__ out, uint64_t total,
                           uint64_t list_base, unsigned long long* sums) {
  const uint64_t per = 1024;
  uint64_t g0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * per;
  unsigned long long h = 0, s = 0, cnt = 0;
  if (g0 < total) {
    uint64_t l = find_list(out_off, 0, n_lists, g0);
    while (l + 1 < n_lists && out_off[l + 1] <= g0) l++;
    uint64_t g1 = mn64(total, g0 + per);
    for (uint64_t g = g0; g < g1; g++) {
      while (out_off[l + 1] <= g) l++;
      uint64_t i = g - out_off[l];
      uint64_t d = out[g];
      h += mix64((((l + list_base) << 32) | i) ^ (d * 0x9E3779B97F4A7C15ull));
      s += d;
    }
  }
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_lists;
       l += (uint64_t)gridDim.x * blockDim.x)
    cnt += list_n[l];
  for (int o = 16; o > 0; o >>= 1) {
    h += __shfl_xor_sync(0xffffffffu, h, o);
    s += __shfl_xor_sync(0xffffffffu, s, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sums + 0, h);
    atomicAdd(sums + 1, s);
    atomicAdd(sums + 2, cnt);
  }
}

}  // namespace gcd

// =====================================================================================
// host side
// =====================================================================================
using namespace gcd;

namespace {

// ------------------------------------------------------------------ Variable Byte
// The short-list fallback of P:L640 §7.5 (P §2.3: 7-bit groups, least significant first,
// MSB = 1 on an int's last byte).  Bytes after a list's n ints (the 4-byte padding of the
// list's area) are ignored.
// Short lists (n < kVbShort, the fallback's case): one thread per list, a serial byte loop
// (staging a warp's 32 lists in shared memory first measured slower).
constexpr uint32_t kVbShort = 64;
// The directory checks of k_lists for one Variable Byte list (that path runs no k_lists):
// out_off is the exclusive scan of list_n and inside the output, the control range is
// ordered and inside the batch.  A list that fails is flagged GC_DEV_TRUNCATED and skipped.
__device__ __forceinline__ bool vb_list_ok(const Dev& D, uint64_t l, uint32_t n) {
  const uint64_t c0 = D.ctrl_off[l], c1 = D.ctrl_off[l + 1];
  const uint64_t o0 = D.out_off[l], o1 = D.out_off[l + 1];
  bool ok = c1 >= c0 && c1 <= 4 * D.n_ctrl_words && o1 == o0 + n && o1 <= D.total_out;
  if (l == 0) ok = ok && o0 == 0 && c0 == 0;
  if (l + 1 == D.n_lists) ok = ok && o1 == D.total_out;
  return ok;
}
template <bool DGAPS>
__global__ void __launch_bounds__(256) k_varbyte_short(Dev D, uint32_t* __restrict__ out) {
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(D.ctrl_words);
  uint32_t err = 0, long_seen = 0;
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < D.n_lists;
       l += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n = D.list_n[l];
    if (!vb_list_ok(D, l, n)) {
      err |= GC_DEV_TRUNCATED;
      continue;
    }
    if (n >= kVbShort) {
      if (D.ctrl_off[l + 1] - D.ctrl_off[l] < n) err |= GC_DEV_TRUNCATED;
      else long_seen = 1u;
      continue;
    }
    if (n == 0) continue;
    const uint64_t c0 = D.ctrl_off[l], c1 = D.ctrl_off[l + 1], o0 = D.out_off[l];
    uint64_t p = c0;
    uint32_t acc = 0;
    for (uint32_t i = 0; i < n; i++) {
      uint32_t v = 0, k = 0;
      for (;;) {
        if (p >= c1) {
          err |= GC_DEV_TRUNCATED;
          break;
        }
        if (k == 5) {
          err |= GC_DEV_BAD_LD;
          break;
        }
        GC_CHECK(p < 4 * D.n_ctrl_words);
        const uint32_t b = bytes[p++];
        v |= (b & 127u) << (7 * k);
        k++;
        if (b & 128u) break;
      }
      acc = DGAPS ? acc + v : v;
      GC_CHECK(o0 + i < D.total_out);
      out[o0 + i] = acc;
    }
  }
  if (err) atomicOr(&D.hdr->status, err);
  if (__any_sync(0xffffffffu, long_seen) && (threadIdx.x & 31) == 0) D.hdr->vb_long = 1u;
}
// Long lists (n >= kVbShort) in parallel: byte-space tiles of kVbTB bytes (one TileA slot
// each: the index kernel's control tiles have the same size, so the workspace layout is
// shared), one CTA per tile, claimed in order.  Each thread holds 32 consecutive bytes; an
// int ends at a byte with MSB 1 (P §2.3).  A block scan segmented at long-list starts of
// (ints ended, their sum) and a decoupled look-back across tiles give every int its index in
// its list and its d-gap prefix.  Bytes of short lists (k_varbyte_short's) and the
// padding after a list's n ints are skipped.
constexpr uint32_t kVbTB = 4 * kWA;     // bytes per tile (8192): 32 per thread
constexpr uint32_t kVbL = 136;          // long lists touching a tile: <= 8192 / 64 + 2

template <bool DGAPS>
__global__ void __launch_bounds__(256) k_varbyte_tiles(Dev D, uint32_t* __restrict__ out) {
  __shared__ uint32_t s_tile, s_cnt, s_pq, s_pd, s_err;
  __shared__ unsigned long long s_la, s_lb;
  __shared__ int32_t s_rs[kVbL];            // list start relative to the tile (>= -8)
  __shared__ uint32_t s_st[kVbL], s_en[kVbL];  // its bytes in the tile: [st, en)
  __shared__ uint32_t s_n[kVbL], s_fl[kVbL];   // ints; 1: starts in the tile, 2: ends in it
  __shared__ unsigned long long s_o[kVbL];
  __shared__ uint32_t s_wc[8], s_pw[8][2];
  __shared__ Seg4 s_scr[8];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(D.ctrl_words);
  const uint64_t nbytes = mn64(D.ctrl_off[D.n_lists], 4ull * D.n_ctrl_words);
  // (stream order: k_varbyte_short has finished; without a long list nothing is left to do)
  if (*reinterpret_cast<volatile const uint32_t*>(&D.hdr->vb_long) == 0) return;
  if (tid == 0) {
    s_tile = atomicAdd(&D.hdr->counter_a, 1u);
    s_cnt = 0;
    s_err = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t B0 = (uint64_t)tile * kVbTB;
  if (warp == 0) {  // lists la..lb overlap [B0, B0 + kVbTB)
    uint64_t la = 1, lb = 0;
    if (B0 < nbytes) {
      la = warp_find(D.ctrl_off, 0, D.n_lists, B0);
      lb = warp_find(D.ctrl_off, la, D.n_lists, B0 + kVbTB - 1);
    }
    if (lane == 0) {
      s_la = la;
      s_lb = lb;
    }
  }
  __syncthreads();
  const uint64_t la = s_la, lb = s_lb;
  // the long lists of the tile, in list order (block compaction, rounds of 256 lists)
  for (uint64_t r = la; r <= lb && lb >= la; r += 256) {
    const uint64_t l = r + tid;
    bool keep = false;
    uint32_t n = 0;
    uint64_t c0 = 0, c1 = 0;
    if (l <= lb) {
      n = D.list_n[l];
      if (n >= kVbShort && vb_list_ok(D, l, n)) {
        c0 = D.ctrl_off[l];
        c1 = D.ctrl_off[l + 1];
        // (a list with fewer bytes than ints is flagged by k_varbyte_short and skipped: every
        // kept list has >= 64 bytes, so at most kVbL of them touch a tile)
        keep = c1 - c0 >= n && c0 < B0 + kVbTB && c1 > B0;
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_wc[warp] = __popc(m);
    __syncthreads();
    uint32_t before = s_cnt;
    for (uint32_t x = 0; x < warp; x++) before += s_wc[x];
    if (keep) {
      const uint32_t k = before + __popc(m & ((1u << lane) - 1u));
      GC_CHECK(k < kVbL);
      if (k < kVbL) {
        const int64_t rs = (int64_t)c0 - (int64_t)B0;
        s_rs[k] = (int32_t)(rs < -8 ? -8 : rs);
        s_st[k] = c0 > B0 ? (uint32_t)(c0 - B0) : 0u;
        s_en[k] = (uint32_t)(mn64(c1, B0 + kVbTB) - B0);
        s_n[k] = n;
        s_fl[k] = (c0 >= B0 ? 1u : 0u) | (c1 <= B0 + kVbTB ? 2u : 0u);
        s_o[k] = D.out_off[l];
      }
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t t = s_cnt;
      for (uint32_t x = 0; x < 8; x++) t += s_wc[x];
      if (t > kVbL) s_err |= GC_DEV_TRUNCATED;  // (cannot happen with a consistent directory)
      s_cnt = min(t, kVbL);
    }
    __syncthreads();
  }
  const uint32_t cnt = s_cnt;
  if (cnt == 0) {  // no long list here: an empty inclusive prefix (no list continues through)
    if (tid == 0) {
      uint64_t v0, v1;
      tilea_pack(0, 0, 0, v0, v1);
      st_relaxed_u64(&D.tiles_a[tile].i1, v1);
      st_relaxed_u64(&D.tiles_a[tile].i0, v0);
      if (s_err) atomicOr(&D.hdr->status, s_err);
    }
    return;
  }
  // my 32 bytes (8 words) and the 8 bytes before them
  const uint32_t p0 = 32 * tid;
  const uint64_t g0 = B0 + p0;
  uint32_t w[8];
  if (g0 + 32 <= 4ull * D.n_ctrl_words) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(bytes + g0));
    const uint4 y = __ldg(reinterpret_cast<const uint4*>(bytes + g0) + 1);
    w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
    w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; i++) w[i] = g0 + 4 * i + 4 <= 4ull * D.n_ctrl_words ? D.ctrl_words[g0 / 4 + i] : 0u;
  }
  if (lane == 31) {
    s_pw[warp][0] = w[6];
    s_pw[warp][1] = w[7];
  }
  uint32_t pw6 = __shfl_up_sync(0xffffffffu, w[6], 1), pw7 = __shfl_up_sync(0xffffffffu, w[7], 1);
  __syncthreads();
  if (lane == 0) {
    if (warp) {
      pw6 = s_pw[warp - 1][0];
      pw7 = s_pw[warp - 1][1];
    } else {
      pw6 = B0 >= 8 ? D.ctrl_words[B0 / 4 - 2] : 0u;
      pw7 = B0 >= 8 ? D.ctrl_words[B0 / 4 - 1] : 0u;
    }
  }
  auto byte_at = [&](uint32_t i) -> uint32_t { return (w[i >> 2] >> (8 * (i & 3))) & 0xFFu; };
  // the table entry of my first byte: the last list starting at or before it
  uint32_t k0 = 0;
  {
    uint32_t a = 0, b = cnt;
    while (b - a > 1) {
      const uint32_t m = (a + b) >> 1;
      if (s_st[m] <= p0) a = m;
      else b = m;
    }
    k0 = a;
  }
  const bool in0 = cnt > 0 && s_st[k0] <= p0 && p0 < s_en[k0];
  // the open int at my first byte: its bytes among the 8 before me (in its list, after the
  // last byte with MSB 1)
  uint32_t cur0 = 0, nb0 = 0;
  if (in0) {
    const uint64_t pv = ((uint64_t)pw7 << 32) | pw6;  // bytes p0-8 .. p0-1
    uint32_t j = 0;
    while (j < 8) {
      const int32_t q = (int32_t)p0 - (int32_t)j - 1;
      const uint32_t b = (uint32_t)(pv >> (8 * (7 - j))) & 0xFFu;
      if (q < s_rs[k0] || (b & 128u)) break;
      j++;
    }
    nb0 = j;
    for (uint32_t t = 0; t < min(j, 5u); t++)
      cur0 |= ((uint32_t)(pv >> (8 * (8 - j + t))) & 127u) << (7 * t);
  }
  uint32_t err = 0;
  // pass 1: (list start seen, ints ended, their sum) of my bytes
  Seg4 agg{0u, 0u, 0u, 0u};
  {
    uint32_t k = k0, cur = cur0, nb = nb0;
#pragma unroll
    for (uint32_t i = 0; i < 32; i++) {
      const uint32_t p = p0 + i;
      while (k < cnt && p >= s_en[k]) k++;
      if (k >= cnt || p < s_st[k]) {
        cur = nb = 0;
        continue;
      }
      if (p == s_st[k] && (s_fl[k] & 1u)) {
        agg = Seg4{1u, 0u, 0u, 0u};
        cur = nb = 0;
      }
      const uint32_t b = byte_at(i);
      if (nb < 5) cur |= (b & 127u) << (7 * nb);
      nb++;
      if (b & 128u) {
        if (nb > 5) err |= GC_DEV_BAD_LD;
        agg.q += 1;
        agg.d += cur;
        cur = nb = 0;
      }
    }
  }
  Seg4 total;
  const Seg4 excl = block_excl_seg4<false, 8>(agg, s_scr, &total);
  // the carry into the tile: only if its first bytes continue a long list
  const bool need_carry = cnt > 0 && s_rs[0] < 0 && s_st[0] == 0 && s_en[0] > 0;
  if (warp == 0) {
    TileA* me = D.tiles_a + tile;
    uint64_t v0, v1;
    if (!need_carry || total.f) {
      tilea_pack(total.q, total.d, 0, v0, v1);
      if (lane == 0) {
        st_relaxed_u64(&me->i1, v1);
        st_relaxed_u64(&me->i0, v0);
      }
    } else {
      tilea_pack(total.q, total.d, 0, v0, v1);
      if (lane == 0) {
        st_relaxed_u64(&me->a1, v1);
        st_relaxed_u64(&me->a0, v0);
      }
    }
    uint32_t pq = 0;
    uint64_t pd = 0, pe = 0;
    if (need_carry) {
      lookback_tilea(D.tiles_a, tile, pq, pd, pe);
      if (lane == 0 && !total.f) {
        tilea_pack(pq + total.q, (uint32_t)(pd + total.d), 0, v0, v1);
        st_relaxed_u64(&me->i1, v1);
        st_relaxed_u64(&me->i0, v0);
      }
    }
    if (lane == 0) {
      s_pq = pq;
      s_pd = (uint32_t)pd;
    }
  }
  __syncthreads();
  // pass 2: every int ended in my bytes to its list position
  {
    uint32_t c = excl.f ? excl.q : s_pq + excl.q;
    uint32_t sum = excl.f ? excl.d : s_pd + excl.d;
    uint32_t k = k0, cur = cur0, nb = nb0;
#pragma unroll
    for (uint32_t i = 0; i < 32; i++) {
      const uint32_t p = p0 + i;
      while (k < cnt && p >= s_en[k]) k++;
      if (k >= cnt || p < s_st[k]) {
        cur = nb = 0;
        continue;
      }
      if (p == s_st[k] && (s_fl[k] & 1u)) {
        c = sum = 0;
        cur = nb = 0;
      }
      const uint32_t b = byte_at(i);
      if (nb < 5) cur |= (b & 127u) << (7 * nb);
      nb++;
      if (b & 128u) {
        sum += cur;
        if (c < s_n[k]) {
          GC_CHECK(s_o[k] + c < D.total_out);
          out[s_o[k] + c] = DGAPS ? sum : cur;
        }
        c++;
        cur = nb = 0;
      }
      if (p + 1 == s_en[k] && (s_fl[k] & 2u) && c < s_n[k]) err |= GC_DEV_TRUNCATED;
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(&s_err, err);
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(&D.hdr->status, s_err);
}

gc_status launch_varbyte(const Dev& D, uint32_t* out, bool dgaps, cudaStream_t st, int stages,
                         int n_sm, bool short_only = false) {
  if (!(stages & GC_STAGE_DECODE)) return GC_OK;
  const uint64_t sblocks = mn64((D.n_lists + 255) / 256, (uint64_t)n_sm * 16);
  // byte tiles over the whole stream (tiles without a long list return at once); a
  // workspace-resetting caller gives them zeroed tickets and look-back slots
  const uint64_t tiles = (4ull * D.n_ctrl_words + kVbTB - 1) / kVbTB;
  if (dgaps) {
    k_varbyte_short<true><<<(unsigned)mx64(sblocks, 1), 256, 0, st>>>(D, out);
    if (!short_only && tiles) k_varbyte_tiles<true><<<(unsigned)tiles, 256, 0, st>>>(D, out);
  } else {
    k_varbyte_short<false><<<(unsigned)mx64(sblocks, 1), 256, 0, st>>>(D, out);
    if (!short_only && tiles) k_varbyte_tiles<false><<<(unsigned)tiles, 256, 0, st>>>(D, out);
  }
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

struct WsLayout {
  uint64_t n_tiles_a, n_tiles_b, wa;
  uint64_t off_tiles_a, off_tiles_b, off_entries, off_first, bytes;
};

WsLayout ws_layout(const gc_batch* b) {
  WsLayout L;
  uint64_t words = b->ctrl_bytes / 4;
  L.wa = words < kSmallIndexWords ? kWASmall : kWA;
  // GC_INDEX_TILE_WORDS=256|2048 forces one index tile size (a test knob; the workspace size
  // and the decode must see the same setting)
  if (const char* e = getenv("GC_INDEX_TILE_WORDS")) {
    const uint64_t v = strtoull(e, nullptr, 10);
    if (v == kWASmall || v == kWA) L.wa = v;
  }
  L.n_tiles_a = (words + L.wa - 1) / L.wa;
  if (L.n_tiles_a == 0) L.n_tiles_a = 1;
  L.n_tiles_b = (b->total_out + kT - 1) / kT;
  L.off_tiles_a = sizeof(WsHeader);
  L.off_tiles_b = L.off_tiles_a + L.n_tiles_a * sizeof(TileA);
  L.off_entries = L.off_tiles_b + ((L.n_tiles_b * 8 + 255) & ~255ull);
  L.off_first = L.off_entries + L.n_tiles_b * sizeof(Entry);
  L.bytes = L.off_first + ((L.n_tiles_a * 4 + 255) & ~255ull);
  return L;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

gc_status check_codec(const gc_batch* b) {
  switch (b->codec) {
    case GC_VARBYTE:
    case GC_GROUP_SIMPLE:
    case GC_GROUP_AFOR:
      return b->variant == 0 ? GC_OK : GC_ERR_BAD_VARIANT;
    case GC_GROUP_SCHEME: {
      uint32_t kind = (b->variant >> 2) & 3u, cg = 1u << (b->variant & 3u);
      if (b->variant > 15 || kind > 2 || (kind == 2 && cg < 4)) return GC_ERR_BAD_VARIANT;
      return GC_OK;
    }
    case GC_GROUP_PFD:
      return (b->pfd_frame_quads == 32 || b->pfd_frame_quads == 128) && b->variant <= 1
                 ? GC_OK : GC_ERR_BAD_VARIANT;
    default:
      return GC_ERR_UNKNOWN_CODEC;
  }
}

gc_status check_batch(const gc_batch* b, bool device_ptrs) {
  if (!b) return GC_ERR_INVALID_ARGUMENT;
  gc_status s = check_codec(b);
  if (s != GC_OK) return s;
  if (!b->list_n && b->n_lists) return GC_ERR_INVALID_ARGUMENT;
  if (!b->ctrl_off || !b->data_off || !b->out_off) return GC_ERR_INVALID_ARGUMENT;
  if (b->codec == GC_GROUP_PFD && !b->exc_off) return GC_ERR_INVALID_ARGUMENT;
  if ((b->ctrl_bytes % 16) || (b->exc_bytes % 16)) return GC_ERR_INVALID_ARGUMENT;
  if (b->ctrl_bytes && (!b->ctrl || !aligned16(b->ctrl))) return GC_ERR_INVALID_ARGUMENT;
  if (b->data_vectors && (!b->data || !aligned16(b->data))) return GC_ERR_INVALID_ARGUMENT;
  if (b->exc_bytes && (!b->exc || !aligned16(b->exc))) return GC_ERR_INVALID_ARGUMENT;
  // (the index look-back packs lane-bit and exception-byte prefixes in 47 bits)
  if (b->data_vectors >= (1ull << 42) || b->exc_bytes >= (1ull << 47)) return GC_ERR_INVALID_ARGUMENT;
  if (b->total_out && !b->n_lists) return GC_ERR_INVALID_ARGUMENT;
  if (b->total_out > (1ull << 40) || b->n_lists > 0xFFFFFFF0ull) return GC_ERR_INVALID_ARGUMENT;
  (void)device_ptrs;
  return GC_OK;
}

// Per-device launch facts.  Nothing is cached across calls in process-wide statics: the
// device is the caller's current one, and the dynamic shared memory attribute (a
// per-device property of a kernel) is set on every launch -- both cost microseconds.
struct DevInfo {
  int dev, n_sm;
  uint64_t max_grid;  // GC_DECODE_MAX_GRID (tests: several tiles per CTA at small sizes), 0 = none
};
gc_status device_info(DevInfo* di) {
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&di->n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return GC_ERR_CUDA;
  di->dev = dev;
  const char* mg = getenv("GC_DECODE_MAX_GRID");
  di->max_grid = mg ? strtoull(mg, nullptr, 10) : 0;
  if (major != 10) return GC_ERR_UNSUPPORTED_DEVICE;
  return di->n_sm > 0 ? GC_OK : GC_ERR_CUDA;
}

template <class C>
gc_status launch_index(const Dev& D, cudaStream_t st, const DevInfo& di) {
  const uint64_t lb = (D.n_lists + kThreads - 1) / kThreads;
  k_lists<<<(unsigned)mn64(mx64(lb, 1), (uint64_t)di.n_sm * 8), kThreads, 0, st>>>(D);
  if (cudaGetLastError() != cudaSuccess) return GC_ERR_CUDA;
  const dim3 g((unsigned)D.n_tiles_a);
  if (D.skip) {
    if (D.wa == kWA) k_index<C, kCA, true><<<g, kThreads, 0, st>>>(D);
    else k_index<C, 1, true><<<g, kThreads, 0, st>>>(D);
  } else {
    if (D.wa == kWA) k_index<C, kCA, false><<<g, kThreads, 0, st>>>(D);
    else k_index<C, 1, false><<<g, kThreads, 0, st>>>(D);
  }
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).  The
// pointer is process-wide and device-independent; std::call_once makes the lookup reentrant.
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
  static std::once_flag once;
  static EncodeTiled fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}
// The decode output as a 2-D tensor {32 ints, total_out / 32 rows} with 8-row boxes and the
// staging window's 128-byte swizzle (gc_decode.cuh).  False (plain stores) when the output is
// not 16-byte aligned, shorter than a row, or the encoder is unavailable.
bool out_tensor_map(CUtensorMap* tm, uint32_t* out, uint64_t total_out) {
  memset(tm, 0, sizeof(*tm));
  const EncodeTiled enc = encode_tiled();
  const uint64_t rows = total_out / 32;
  if (!kTma || !enc || rows == 0 || ((uintptr_t)out & 15u) || rows > (1ull << 31)) return false;
  const cuuint64_t dims[2] = {32, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, kBoxC / 8};
  const cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k_decode over one batch, or (pair) over a docIDs batch D and a TFs batch *D1 together
template <class C>
gc_status launch_decode(const Dev& D, uint32_t* out, bool dgaps, cudaStream_t st, const DevInfo& di,
                        const Dev* D1 = nullptr, uint32_t* out1 = nullptr) {
  if (D.n_tiles_b == 0) return GC_OK;
  const uint32_t smem = DS<C>::bytes();
#ifdef GC_ABL_NODGAP
  dgaps = false;
#endif
  auto kern = D1 ? (dgaps ? k_decode<C, true, true> : k_decode<C, false, true>)
                 : (dgaps ? k_decode<C, true, false> : k_decode<C, false, false>);
  int per_sm = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDT, smem) != cudaSuccess)
    return GC_ERR_CUDA;
  if (per_sm < 1) return GC_ERR_CUDA;  // (cannot happen on sm_100: the kernel fits one SM)
  // tiles are assigned round-robin to a co-resident grid (the decoupled look-back waits on
  // earlier tiles, which must all be running): a cooperative launch guarantees residency
  const uint64_t nvt = D1 ? 2ull * D.n_tiles_b : D.n_tiles_b;
  uint64_t cap = (uint64_t)di.n_sm * per_sm;
  if (di.max_grid) cap = mn64(cap, di.max_grid);
  // a pair's CTAs take every grid-th virtual tile: an odd stride alternates each CTA between
  // docID tiles (d-gap scan, look-back) and TF tiles, where an even one would leave half the
  // grid on the cheaper TF tiles and the docIDs on the other half
  if (D1 && cap < nvt && (cap & 1) == 0 && cap > 1) cap--;
  const unsigned grid = (unsigned)mn64(nvt, cap);
  Dev Dv = D, Dv1 = D1 ? *D1 : D;
  uint32_t* o1 = D1 ? out1 : out;
  alignas(64) CUtensorMap tm0, tm1;
  uint32_t tma = out_tensor_map(&tm0, out, D.total_out) ? 1u : 0u;
  if (D1 && out_tensor_map(&tm1, out1, D1->total_out)) tma |= 2u;
  if (!D1) tm1 = tm0;
  void* args[] = {&Dv, &out, &Dv1, &o1, &tm0, &tm1, &tma};
  if (cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kDT), args, smem, st) !=
      cudaSuccess)
    return GC_ERR_CUDA;
  return GC_OK;
}

template <class C>
gc_status launch_codec(const Dev& D, uint32_t* out, bool dgaps, cudaStream_t st, int stages,
                       const DevInfo& di) {
  if (stages & GC_STAGE_INDEX) {
    const gc_status s = launch_index<C>(D, st, di);
    if (s != GC_OK) return s;
  }
  if (!(stages & GC_STAGE_DECODE)) return GC_OK;
  return launch_decode<C>(D, out, dgaps, st, di);
}

template <class T>
struct Tag {  // (a codec type as a value, for generic lambdas)
  using type = T;
};

// The kernels' view of a batch and its workspace.
Dev make_dev(const gc_batch* b, uint8_t* w, const WsLayout& L) {
  Dev D;
  D.n_lists = b->n_lists;
  D.list_n = b->list_n;
  D.ctrl_off = b->ctrl_off;
  D.data_off = b->data_off;
  D.exc_off = b->codec == GC_GROUP_PFD ? b->exc_off : nullptr;
  D.out_off = b->out_off;
  D.ctrl_words = (const uint32_t*)b->ctrl;
  D.n_ctrl_words = b->ctrl_bytes / 4;
  D.data = (const uint4*)b->data;
  D.data_vectors = b->data_vectors;
  D.exc = b->exc;
  D.exc_bytes = b->exc_bytes;
  D.total_out = b->total_out;
  D.n_tiles_a = (uint32_t)L.n_tiles_a;
  D.wa = (uint32_t)L.wa;
  D.n_tiles_b = (uint32_t)L.n_tiles_b;
  D.hdr = (WsHeader*)w;
  D.tiles_a = (TileA*)(w + L.off_tiles_a);
  D.tiles_b = (uint64_t*)(w + L.off_tiles_b);
  D.entries = (Entry*)(w + L.off_entries);
  D.first_list = (uint32_t*)(w + L.off_first);
  D.docids = nullptr;
  D.skip_off = nullptr;
  D.skip = nullptr;
  return D;
}

// What one call does: a decode (its stages), the skip-table build, or a range decode.
enum JobKind { JOB_DECODE, JOB_SKIP, JOB_RANGE };
struct Job {
  JobKind kind;
  bool dgaps;
  int stages;
  uint64_t first, last;  // JOB_RANGE: output ints [first, last)
};

template <class C>
gc_status run_codec(const Dev& D, uint32_t* out, const Job& J, cudaStream_t st, const DevInfo& di) {
  if (J.kind == JOB_DECODE) return launch_codec<C>(D, out, J.dgaps, st, J.stages, di);
  if (J.kind == JOB_SKIP) {
    // the control-stream scan with skip emission: k_index knows every word's list
    // prefixes; the entry offsets come first
    k_skip_off<<<1, kSkipT, 0, st>>>(D);
    if (cudaGetLastError() != cudaSuccess) return GC_ERR_CUDA;
    return launch_codec<C>(D, out, true, st, GC_STAGE_INDEX, di);
  }
  // JOB_RANGE: the covering entries, then one warp per 512-int block
  unsigned long long* eb = reinterpret_cast<unsigned long long*>(D.hdr->prof);
  k_range_bounds<<<1, 32, 0, st>>>(D, J.first, J.last, eb);
  if (cudaGetLastError() != cudaSuccess) return GC_ERR_CUDA;
  const uint64_t blocks = (J.last - J.first) / GC_SKIP_DIST + 2 * 32;  // (a bound of the count)
  const unsigned grid = (unsigned)mn64((blocks + kRangeW - 1) / kRangeW + 1, (uint64_t)di.n_sm * 16);
  if (J.dgaps) k_range<C, true><<<grid, 32 * kRangeW, 0, st>>>(D, out, J.first, J.last, eb);
  else k_range<C, false><<<grid, 32 * kRangeW, 0, st>>>(D, out, J.first, J.last, eb);
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

// (the workspace's header is all a range decode uses: status and the entry bounds)
constexpr uint64_t kRangeWsBytes = sizeof(WsHeader);

gc_status decode_impl(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                      void* stream, const Job& J, const uint32_t* docids = nullptr,
                      const uint64_t* skip_off_in = nullptr, uint64_t* skip_off_out = nullptr,
                      gc_skip_entry* skip = nullptr) {
  gc_status s = check_batch(b, true);
  if (s != GC_OK) return s;
  if (!ws || !aligned16(ws) || (b->total_out && J.kind != JOB_SKIP && (!out || !aligned16(out))))
    return GC_ERR_INVALID_ARGUMENT;
  WsLayout L = ws_layout(b);
  if (ws_bytes < (J.kind == JOB_RANGE ? kRangeWsBytes : L.bytes)) return GC_ERR_WORKSPACE_TOO_SMALL;
  if (J.kind != JOB_DECODE && b->codec == GC_VARBYTE) return GC_ERR_UNKNOWN_CODEC;  // (no groups)
  DevInfo di;
  s = device_info(&di);
  if (s != GC_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* w = (uint8_t*)ws;
  // (a range decode's status word is reset by k_range_bounds, its first kernel: one stream
  // operation fewer on the random-access path; an empty range still gets the memset)
  const bool range_kernels = J.kind == JOB_RANGE && b->n_lists && b->total_out && J.last > J.first;
  const uint64_t reset = J.kind == JOB_RANGE ? kRangeWsBytes : L.bytes;
  if (!range_kernels && (J.kind != JOB_DECODE || (J.stages & GC_STAGE_RESET)) &&
      cudaMemsetAsync(ws, 0, reset, st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (J.kind == JOB_SKIP && b->n_lists == 0)
    return cudaMemsetAsync(skip_off_out, 0, 8, st) == cudaSuccess ? GC_OK : GC_ERR_CUDA;
  if (b->n_lists == 0 || b->total_out == 0 || (J.kind == JOB_RANGE && J.last <= J.first)) return GC_OK;
  Dev D = make_dev(b, w, L);
  D.docids = docids;
  D.skip_off = J.kind == JOB_SKIP ? skip_off_out : const_cast<uint64_t*>(skip_off_in);
  D.skip = skip;
  if (b->codec == GC_VARBYTE) return launch_varbyte(D, out, J.dgaps, st, J.stages, di.n_sm);
  switch (b->codec) {
    case GC_GROUP_SIMPLE:
      return run_codec<CodecGS>(D, out, J, st, di);
    case GC_GROUP_AFOR:
      return run_codec<CodecAFOR>(D, out, J, st, di);
    case GC_GROUP_PFD:
      if (b->variant == 1)  // SIMD-BP128: no exception stream
        return b->pfd_frame_quads == 32 ? run_codec<CodecPFD<32, false>>(D, out, J, st, di)
                                        : run_codec<CodecPFD<128, false>>(D, out, J, st, di);
      return b->pfd_frame_quads == 32 ? run_codec<CodecPFD<32>>(D, out, J, st, di)
                                      : run_codec<CodecPFD<128>>(D, out, J, st, di);
    default:
      break;
  }
  switch (b->variant) {
    case 0: return run_codec<CodecGscB<1>>(D, out, J, st, di);
    case 1: return run_codec<CodecGscB<2>>(D, out, J, st, di);
    case 2: return run_codec<CodecGscB<4>>(D, out, J, st, di);
    case 3: return run_codec<CodecGscB<8>>(D, out, J, st, di);
    case 4: return run_codec<CodecGscCU<1>>(D, out, J, st, di);
    case 5: return run_codec<CodecGscCU<2>>(D, out, J, st, di);
    case 6: return run_codec<CodecGscCU<4>>(D, out, J, st, di);
    case 7: return run_codec<CodecGscCU<8>>(D, out, J, st, di);
    case 10: return run_codec<CodecGscIU<4>>(D, out, J, st, di);
    case 11: return run_codec<CodecGscIU<8>>(D, out, J, st, di);
    default: return GC_ERR_BAD_VARIANT;
  }
}

}  // namespace

extern "C" {

int gc_abi_version(void) { return GC_ABI_VERSION; }

int gc_build_flags(void) {
  int f = 0;
#ifdef GC_CHECKED
  f |= GC_BUILD_CHECKED;
#endif
#ifdef GC_TIMING
  f |= GC_BUILD_TIMING;
#endif
  return f;
}

const char* gc_status_string(gc_status s) {
  switch (s) {
    case GC_OK: return "ok";
    case GC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case GC_ERR_UNKNOWN_CODEC: return "unknown codec";
    case GC_ERR_BAD_VARIANT: return "bad variant";
    case GC_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case GC_ERR_UNSUPPORTED_DEVICE: return "unsupported device (needs sm_100)";
    case GC_ERR_CUDA: return "CUDA error";
    case GC_ERR_NOT_INCREASING: return "list not strictly increasing";
    case GC_ERR_NOMEM: return "out of host memory";
  }
  return "unknown status";
}

gc_status gc_workspace_size(const gc_batch* b, uint64_t* bytes) {
  if (!b || !bytes) return GC_ERR_INVALID_ARGUMENT;
  *bytes = ws_layout(b).bytes;
  return GC_OK;
}

gc_status gc_decode(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes, void* stream) {
  return decode_impl(b, out, ws, ws_bytes, stream, Job{JOB_DECODE, false, GC_STAGE_ALL, 0, 0});
}

gc_status gc_decode_dgaps(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                          void* stream) {
  return decode_impl(b, out, ws, ws_bytes, stream, Job{JOB_DECODE, true, GC_STAGE_ALL, 0, 0});
}

gc_status gc_decode_stage(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                          void* stream, int dgaps, int stage_mask) {
  if (stage_mask & ~GC_STAGE_ALL) return GC_ERR_INVALID_ARGUMENT;
  return decode_impl(b, out, ws, ws_bytes, stream, Job{JOB_DECODE, dgaps != 0, stage_mask, 0, 0});
}

gc_status gc_skip_capacity(const gc_batch* b, uint64_t* entries) {
  if (!b || !entries) return GC_ERR_INVALID_ARGUMENT;
  *entries = b->total_out / GC_SKIP_DIST + b->n_lists;
  return GC_OK;
}

gc_status gc_build_skip(const gc_batch* b, const uint32_t* docids, uint64_t* skip_off,
                        gc_skip_entry* entries, void* ws, uint64_t ws_bytes, void* stream) {
  if (!b || !skip_off || (b->total_out && (!docids || !entries))) return GC_ERR_INVALID_ARGUMENT;
  return decode_impl(b, nullptr, ws, ws_bytes, stream, Job{JOB_SKIP, true, GC_STAGE_INDEX, 0, 0},
                     docids, nullptr, skip_off, entries);
}

gc_status gc_decode_range(const gc_batch* b, const uint64_t* skip_off,
                          const gc_skip_entry* entries, uint32_t* out, uint64_t first,
                          uint64_t count, int dgaps, void* ws, uint64_t ws_bytes, void* stream) {
  if (!b || first > b->total_out || count > b->total_out - first || (count && (!skip_off || !entries)))
    return GC_ERR_INVALID_ARGUMENT;
  return decode_impl(b, out, ws, ws_bytes, stream,
                     Job{JOB_RANGE, dgaps != 0, GC_STAGE_DECODE, first, first + count}, nullptr,
                     skip_off, nullptr, const_cast<gc_skip_entry*>(entries));
}

// ------------------------------------------------------------------ posting store
gc_status gc_posting_split(const uint32_t* list_n, uint64_t n_lists, uint32_t threshold,
                           uint64_t* long_ids, uint64_t* n_long, uint64_t* short_ids,
                           uint64_t* n_short, uint64_t* list_out_off, uint64_t* short_base) {
  if ((n_lists && (!list_n || !long_ids || !short_ids || !list_out_off)) || !n_long || !n_short ||
      !short_base)
    return GC_ERR_INVALID_ARGUMENT;
  uint64_t nl = 0, ns = 0, long_total = 0;
  for (uint64_t l = 0; l < n_lists; l++) {
    if (list_n[l] >= threshold) {
      long_ids[nl++] = l;
      list_out_off[l] = long_total;
      long_total += list_n[l];
    } else {
      short_ids[ns++] = l;
    }
  }
  const uint64_t base = (long_total + 3) & ~3ull;  // the short group starts 16-B aligned
  uint64_t off = base;
  for (uint64_t i = 0; i < ns; i++) {
    list_out_off[short_ids[i]] = off;
    off += list_n[short_ids[i]];
  }
  *n_long = nl;
  *n_short = ns;
  *short_base = base;
  return GC_OK;
}

gc_status gc_posting_gather(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists,
                            const uint64_t* ids, uint64_t n_ids, uint32_t* out,
                            uint32_t* out_list_n) {
  if ((n_ids && (!ids || !out_list_n)) || (n_lists && !list_n)) return GC_ERR_INVALID_ARGUMENT;
  // list starts, then each requested list copied in turn
  uint64_t* start = (uint64_t*)malloc((size_t)(n_lists + 1) * 8);
  if (!start) return GC_ERR_NOMEM;
  start[0] = 0;
  for (uint64_t l = 0; l < n_lists; l++) start[l + 1] = start[l] + list_n[l];
  uint64_t o = 0;
  gc_status st = GC_OK;
  for (uint64_t i = 0; i < n_ids; i++) {
    if (ids[i] >= n_lists) {
      st = GC_ERR_INVALID_ARGUMENT;
      break;
    }
    const uint32_t n = list_n[ids[i]];
    if (n && (!values || !out)) {
      st = GC_ERR_INVALID_ARGUMENT;
      break;
    }
    if (n) memcpy(out + o, values + start[ids[i]], (size_t)n * 4);
    out_list_n[i] = n;
    o += n;
  }
  free(start);
  return st;
}

static uint64_t store_tf_ws_off(const gc_posting_store* s) {
  return (ws_layout(&s->long_docs).bytes + 255) & ~255ull;
}

gc_status gc_posting_store_ws_size(const gc_posting_store* s, uint64_t* bytes) {
  if (!s || !bytes) return GC_ERR_INVALID_ARGUMENT;
  *bytes = store_tf_ws_off(s) + (s->long_tfs ? ws_layout(s->long_tfs).bytes : sizeof(WsHeader));
  return GC_OK;
}

gc_status gc_decode_posting_store(const gc_posting_store* s, uint32_t* docs, uint32_t* tfs,
                                  int dgaps, void* ws, uint64_t ws_bytes, void* stream) {
  if (!s || !ws || !aligned16(ws)) return GC_ERR_INVALID_ARGUMENT;
  uint64_t need = 0;
  gc_posting_store_ws_size(s, &need);
  if (ws_bytes < need) return GC_ERR_WORKSPACE_TOO_SMALL;
  const gc_batch* LD = &s->long_docs;
  const gc_batch* SD = &s->short_docs;
  const bool has_tf = s->long_tfs != nullptr;
  if (has_tf && (!tfs || !s->short_tfs)) return GC_ERR_INVALID_ARGUMENT;
  if (SD->codec != GC_VARBYTE || (has_tf && s->short_tfs->codec != GC_VARBYTE)) return GC_ERR_BAD_VARIANT;
  if ((s->short_base & 3) || s->short_base < LD->total_out) return GC_ERR_INVALID_ARGUMENT;
  if (has_tf && (s->long_tfs->codec != LD->codec || s->long_tfs->variant != LD->variant ||
                 s->long_tfs->pfd_frame_quads != LD->pfd_frame_quads ||
                 s->long_tfs->total_out != LD->total_out || s->long_tfs->n_lists != LD->n_lists))
    return GC_ERR_INVALID_ARGUMENT;
  for (const gc_batch* b : {LD, SD, s->long_tfs, s->short_tfs}) {
    if (!b) continue;
    gc_status st = check_batch(b, true);
    if (st != GC_OK) return st;
  }
  if (!docs || !aligned16(docs) || (has_tf && !aligned16(tfs))) return GC_ERR_INVALID_ARGUMENT;
  DevInfo di;
  gc_status st = device_info(&di);
  if (st != GC_OK) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  uint8_t* w0 = (uint8_t*)ws;
  uint8_t* w1 = w0 + store_tf_ws_off(s);
  const WsLayout L0 = ws_layout(LD);
  const WsLayout L1 = has_tf ? ws_layout(s->long_tfs) : WsLayout{};
  if (cudaMemsetAsync(w0, 0, L0.bytes, cs) != cudaSuccess ||
      cudaMemsetAsync(w1, 0, has_tf ? L1.bytes : sizeof(WsHeader), cs) != cudaSuccess)
    return GC_ERR_CUDA;
  Dev D0 = make_dev(LD, w0, L0);
  Dev D1 = has_tf ? make_dev(s->long_tfs, w1, L1) : D0;
  // the long group: both index stages, then one fused decode of docIDs (+ TFs)
  auto run_long = [&](auto codec_tag) -> gc_status {
    using C = typename decltype(codec_tag)::type;
    gc_status r = launch_index<C>(D0, cs, di);
    if (r == GC_OK && has_tf) r = launch_index<C>(D1, cs, di);
    if (r != GC_OK) return r;
    return launch_decode<C>(D0, docs, dgaps != 0, cs, di, has_tf ? &D1 : nullptr, tfs);
  };
  if (LD->n_lists && LD->total_out) {
    if (LD->codec == GC_VARBYTE) return GC_ERR_BAD_VARIANT;
    switch (LD->codec) {
      case GC_GROUP_SIMPLE: st = run_long(Tag<CodecGS>{}); break;
      case GC_GROUP_AFOR: st = run_long(Tag<CodecAFOR>{}); break;
      case GC_GROUP_PFD:
        if (LD->variant == 1)
          st = LD->pfd_frame_quads == 32 ? run_long(Tag<CodecPFD<32, false>>{})
                                         : run_long(Tag<CodecPFD<128, false>>{});
        else
          st = LD->pfd_frame_quads == 32 ? run_long(Tag<CodecPFD<32>>{})
                                         : run_long(Tag<CodecPFD<128>>{});
        break;
      default:
        switch (LD->variant) {
          case 0: st = run_long(Tag<CodecGscB<1>>{}); break;
          case 1: st = run_long(Tag<CodecGscB<2>>{}); break;
          case 2: st = run_long(Tag<CodecGscB<4>>{}); break;
          case 3: st = run_long(Tag<CodecGscB<8>>{}); break;
          case 4: st = run_long(Tag<CodecGscCU<1>>{}); break;
          case 5: st = run_long(Tag<CodecGscCU<2>>{}); break;
          case 6: st = run_long(Tag<CodecGscCU<4>>{}); break;
          case 7: st = run_long(Tag<CodecGscCU<8>>{}); break;
          case 10: st = run_long(Tag<CodecGscIU<4>>{}); break;
          case 11: st = run_long(Tag<CodecGscIU<8>>{}); break;
          default: st = GC_ERR_BAD_VARIANT;
        }
    }
    if (st != GC_OK) return st;
  }
  // the short group: Variable Byte, docIDs and TFs, from short_base (status: same headers)
  if (SD->n_lists && SD->total_out) {
    const WsLayout LS = ws_layout(SD);
    Dev DS = make_dev(SD, w0, LS);
    st = launch_varbyte(DS, docs + s->short_base, dgaps != 0, cs, GC_STAGE_DECODE, di.n_sm, true);
    if (st != GC_OK) return st;
    if (has_tf) {
      Dev DT = make_dev(s->short_tfs, w1, ws_layout(s->short_tfs));
      st = launch_varbyte(DT, tfs + s->short_base, false, cs, GC_STAGE_DECODE, di.n_sm, true);
    }
  }
  return st;
}

gc_status gc_posting_store_status(const gc_posting_store* s, const void* ws, uint32_t* host_bits,
                                  void* stream) {
  if (!s || !ws || !host_bits) return GC_ERR_INVALID_ARGUMENT;
  uint32_t a = 0, b = 0;
  gc_status st = gc_read_device_status(ws, &a, stream);
  if (st == GC_OK) st = gc_read_device_status((const uint8_t*)ws + store_tf_ws_off(s), &b, stream);
  *host_bits = a | b;
  return st;
}

gc_status gc_read_device_status(const void* ws, uint32_t* host_bits, void* stream) {
  if (!ws || !host_bits) return GC_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(host_bits, ws, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return GC_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

gc_status gc_checksum(const gc_batch* b, const uint32_t* out, uint64_t list_base,
                      uint64_t* dev_sum3, void* stream) {
  if (!b || !dev_sum3 || (b->total_out && !out)) return GC_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(dev_sum3, 0, 24, st) != cudaSuccess) return GC_ERR_CUDA;
  if (b->n_lists == 0) return GC_OK;
  uint64_t threads = (b->total_out + 1023) / 1024;
  uint64_t blocks = (mx64(threads, b->n_lists / 64 + 1) + 255) / 256;
  blocks = mn64(blocks, 1u << 20);
  k_checksum<<<(unsigned)blocks, 256, 0, st>>>(b->list_n, b->out_off, b->n_lists, out,
                                                 b->total_out, list_base,
                                                 (unsigned long long*)dev_sum3);
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

// --------------------------------------------------------------------------- host path
static uint64_t al256(uint64_t x) { return (x + 255) & ~255ull; }

gc_status gc_host_scratch_size(const gc_batch* hb, uint64_t* bytes) {
  if (!hb || !bytes) return GC_ERR_INVALID_ARGUMENT;
  uint64_t L = hb->n_lists;
  uint64_t s = al256(4 * L) + 4 * al256(8 * (L + 1)) + al256(hb->ctrl_bytes) +
               al256(16 * hb->data_vectors) + al256(hb->exc_bytes) + al256(4 * hb->total_out);
  s += ws_layout(hb).bytes;
  *bytes = s;
  return GC_OK;
}

gc_status gc_decode_host(const gc_batch* hb, uint32_t* host_out, int dgaps, void* dev_scratch,
                         uint64_t scratch_bytes, void* stream) {
  gc_status s = check_batch(hb, false);
  if (s != GC_OK) return s;
  uint64_t need = 0;
  gc_host_scratch_size(hb, &need);
  if (!dev_scratch || ((uintptr_t)dev_scratch & 255u) || scratch_bytes < need ||
      (hb->total_out && !host_out))
    return GC_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* p = (uint8_t*)dev_scratch;
  uint64_t L = hb->n_lists;
  gc_batch d = *hb;
  auto put = [&](const void* src, uint64_t bytes) -> void* {
    void* dst = p;
    p += al256(bytes);
    if (bytes && cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return nullptr;
    return dst;
  };
  d.list_n = (const uint32_t*)put(hb->list_n, 4 * L);
  d.ctrl_off = (const uint64_t*)put(hb->ctrl_off, 8 * (L + 1));
  d.data_off = (const uint64_t*)put(hb->data_off, 8 * (L + 1));
  d.exc_off = nullptr;
  if (hb->exc_off) d.exc_off = (const uint64_t*)put(hb->exc_off, 8 * (L + 1));
  else p += al256(8 * (L + 1));
  d.out_off = (const uint64_t*)put(hb->out_off, 8 * (L + 1));
  d.ctrl = (const uint8_t*)put(hb->ctrl, hb->ctrl_bytes);
  d.data = put(hb->data, 16 * hb->data_vectors);
  d.exc = hb->exc_bytes ? (const uint8_t*)put(hb->exc, hb->exc_bytes) : nullptr;
  if (!d.list_n || !d.ctrl_off || !d.data_off || !d.out_off || !d.ctrl || !d.data)
    return GC_ERR_CUDA;
  uint32_t* dout = (uint32_t*)p;
  p += al256(4 * hb->total_out);
  void* ws = p;
  uint64_t wsb = ws_layout(hb).bytes;
  s = decode_impl(&d, dout, ws, wsb, stream, Job{JOB_DECODE, dgaps != 0, GC_STAGE_ALL, 0, 0});
  if (s != GC_OK) return s;
  if (hb->total_out && cudaMemcpyAsync(host_out, dout, 4 * hb->total_out, cudaMemcpyDeviceToHost,
                                       st) != cudaSuccess)
    return GC_ERR_CUDA;
  return GC_OK;
}

}  // extern "C"
