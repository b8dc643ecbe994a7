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
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

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
  WsHeader* hdr;
  TileA* tiles_a;
  uint64_t* tiles_b;
  Entry* entries;
};

// Per-thread cursor over the lists of consecutive control words.
struct ListCur {
  uint64_t l;        // list index (n_lists = past the end)
  uint64_t cw_lo;    // first control word of the list
  uint64_t cw_hi;    // one past its last control word
  uint64_t n, Q;     // ints, quads
  uint64_t oo;       // out_off
  uint64_t dbase;    // data_off * 32 (lane bits)
  uint64_t ebase;    // exc_off
  uint64_t dlim, elim;  // data_off[l+1]*32, exc_off[l+1]
  __device__ void load(const Dev& D, uint64_t li) {
    l = li;
    if (li >= D.n_lists) {
      cw_lo = cw_hi = ~0ull;
      n = Q = 0;
      return;
    }
    cw_lo = D.ctrl_off[li] >> 2;
    cw_hi = D.ctrl_off[li + 1] >> 2;
    n = D.list_n[li];
    Q = (n + 3) >> 2;
    oo = D.out_off[li];
    dbase = D.data_off[li] * 32ull;
    dlim = D.data_off[li + 1] * 32ull;
    ebase = D.exc_off ? D.exc_off[li] : 0ull;
    elim = D.exc_off ? D.exc_off[li + 1] : 0ull;
  }
  // advance to the list owning control word w (skips lists without control words)
  __device__ void seek(const Dev& D, uint64_t w) {
    if (l < D.n_lists && w < cw_hi) return;
    uint64_t li = l;
    while (li < D.n_lists && (D.ctrl_off[li + 1] >> 2) <= w) li++;
    load(D, li);
  }
};

// Largest l in [lo, hi) with ctrl_off[l] <= key (assumes ctrl_off[lo] <= key).
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
// k_validate: directory consistency (one pass over the lists, folded into the index
// grid).  out_off must be the exclusive scan of list_n, offsets monotone and inside the
// streams, every non-empty list must own at least one control word.
// =====================================================================================
__device__ void validate_lists(const Dev& D, uint32_t tile, uint32_t* s_err) {
  uint64_t per = (D.n_lists + D.n_tiles_a - 1) / D.n_tiles_a;
  uint64_t l0 = (uint64_t)tile * per, l1 = mn64(D.n_lists, l0 + per);
  uint32_t err = 0;
  for (uint64_t l = l0 + threadIdx.x; l < l1; l += kThreads) {
    uint64_t n = D.list_n[l];
    uint64_t c0 = D.ctrl_off[l], c1 = D.ctrl_off[l + 1];
    uint64_t d0 = D.data_off[l], d1 = D.data_off[l + 1];
    uint64_t o0 = D.out_off[l], o1 = D.out_off[l + 1];
    bool bad = (o1 != o0 + n) || (c1 < c0) || (d1 < d0) || ((c0 | c1) & 3) ||
               (c1 > 4 * D.n_ctrl_words) || (d1 > D.data_vectors) || (o1 > D.total_out) ||
               (n > 0 && c1 == c0);
    if (D.exc_off) {
      uint64_t e0 = D.exc_off[l], e1 = D.exc_off[l + 1];
      bad = bad || (e1 < e0) || (e1 > D.exc_bytes);
    }
    if (l == 0) bad = bad || (o0 != 0) || (c0 != 0);
    if (l + 1 == D.n_lists) bad = bad || (o1 != D.total_out);
    if (bad) err |= GC_DEV_TRUNCATED;
  }
  report(s_err, err);
}

// =====================================================================================
// k_index (subsystem (a)): device-wide segmented scan over the control stream.
// =====================================================================================
constexpr uint32_t kLTA = kWA + 2;  // index-kernel list table entries (lists of one tile)

template <class C>
__global__ void __launch_bounds__(kThreads) k_index(Dev D) {
  __shared__ uint32_t s_w[kWA + 1];     // [0] = halo word (tile start - 1)
  __shared__ uint32_t s_cw[kLTA];       // first control word of each list, relative to w0
  __shared__ uint32_t s_q[kLTA];        // quads of each list
  __shared__ uint32_t s_jb[kLTA];       // first quad of the list holding a tile boundary
  __shared__ Seg3 s_scr[kWarps];
  __shared__ Seg3 s_prefix;
  __shared__ uint32_t s_tile, s_err, s_first_reset, s_nl, s_nq;
  __shared__ uint64_t s_la;
  constexpr uint32_t kQueue = 384;  // words needing a group walk (list ends, tile boundaries)
  __shared__ uint32_t s_qw[kQueue], s_qq[kQueue];
  __shared__ uint64_t s_qd[kQueue], s_qe[C::kExc ? kQueue : 1];
  const int tid = threadIdx.x;
  if (tid == 0) {
    const uint32_t tile = atomicAdd(&D.hdr->counter_a, 1u);
    s_tile = tile;
    s_err = 0;
    s_nq = 0;
    const uint64_t w0 = (uint64_t)tile * kWA;
    const uint64_t nw = D.n_ctrl_words > w0 ? mn64(kWA, D.n_ctrl_words - w0) : 0;
    // lists owning words [w0, w0+nw): la = owner of w0, lb = owner of the last word
    uint64_t la = D.n_lists, lb = D.n_lists;
    if (nw) {
      la = find_list(D.ctrl_off, 0, D.n_lists + 1, 4 * w0);
      lb = find_list(D.ctrl_off, la, D.n_lists + 1, 4 * (w0 + nw - 1));
    }
    s_la = la;
    s_nl = la < D.n_lists ? (uint32_t)(mn64(lb, D.n_lists - 1) - la + 1) : 0u;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  validate_lists(D, tile, &s_err);
  const uint64_t w0 = (uint64_t)tile * kWA;
  const uint64_t nw = D.n_ctrl_words > w0 ? mn64(kWA, D.n_ctrl_words - w0) : 0;
  const uint64_t la = s_la;
  const uint32_t nl = s_nl;
  for (uint32_t i = tid; i <= nw; i += kThreads) {
    int64_t gw = (int64_t)w0 - 1 + (int64_t)i;
    s_w[i] = (gw >= 0 && (uint64_t)gw < D.n_ctrl_words) ? D.ctrl_words[gw] : 0u;
  }
  for (uint32_t i = tid; i <= nl; i += kThreads) {
    const uint64_t l = la + i;
    s_cw[i] = (uint32_t)((D.ctrl_off[l] >> 2) - w0);  // may wrap for the first list
    if (i < nl) {
      const uint32_t n = D.list_n[l];
      const uint64_t oo = D.out_off[l];
      const uint64_t tb = (oo + kT - 1) / kT * kT;  // first tile boundary at or after oo
      s_q[i] = (n + 3) >> 2;
      s_jb[i] = tb < oo + n ? (uint32_t)((tb - oo) >> 2) : 0xFFFFFFFFu;
    }
  }
  __syncthreads();

  const uint64_t my0 = w0 + (uint64_t)tid * kCA;
  const uint32_t myn = my0 < w0 + nw ? (uint32_t)mn64(kCA, w0 + nw - my0) : 0u;
  uint32_t li0 = 0;
  if (myn && nl) {
    const uint32_t key = (uint32_t)(my0 - w0);
    uint32_t a = 0, b = nl;
    while (b - a > 1) {
      const uint32_t m = (a + b) >> 1;
      if (s_cw[m] <= key) a = m;
      else b = m;
    }
    li0 = a;
  }
  const uint32_t mynl = nl ? myn : 0u;

  // pass 1: per-word aggregates, segmented at list starts
  Seg3 agg{0, 0, 0, 0};
  WAgg wa_[kCA];
  uint32_t wli[kCA];
  {
    uint32_t li = li0;
    for (uint32_t k = 0; k < kCA; k++) {
      if (k >= mynl) break;
      const uint32_t wr = (uint32_t)(my0 + k - w0);
      while (li + 1 < nl && s_cw[li + 1] <= wr) li++;
      wli[k] = li;
      const uint32_t widx = wr - s_cw[li];
      WCtx c{s_w[wr + 1], s_w[wr], widx, s_q[li], 0u};
      const WAgg a = word_agg<C>(c);
      wa_[k] = a;
      if (widx == 0) {
        const uint64_t l = la + li;
        agg = Seg3{1u, a.q, D.data_off[l] * 32ull + a.d, (D.exc_off ? D.exc_off[l] : 0ull) + a.e};
      } else {
        agg = Seg3{agg.f, agg.q + a.q, agg.d + a.d, agg.e + a.e};
      }
    }
  }
  if (tid == 0) s_first_reset = (mynl && s_cw[li0] == (uint32_t)(my0 - w0)) ? 1u : 0u;
  Seg3 total;
  Seg3 excl = block_excl_seg3(agg, s_scr, &total);

  // decoupled look-back across control tiles (thread 0)
  if (tid == 0) {
    TileA* me = D.tiles_a + tile;
    if (total.f) {
      me->iq = total.q;
      me->id = total.d;
      me->ie = total.e;
      fence_gpu();
      st_relaxed_u32(&me->flag, kFlagIncl);
    } else {
      me->aq = total.q;
      me->ad = total.d;
      me->ae = total.e;
      fence_gpu();
      st_relaxed_u32(&me->flag, kFlagAgg);
    }
    Seg3 pre{0, 0, 0, 0};
    if (!s_first_reset) {
      int64_t p = (int64_t)tile - 1;
      while (p >= 0) {
        TileA* t = D.tiles_a + p;
        uint32_t f = ld_relaxed_u32(&t->flag);
        while (f == 0) {
          __nanosleep(100);
          f = ld_relaxed_u32(&t->flag);
        }
        fence_gpu();
        if (f == kFlagIncl) {
          Seg3 v{1u, ld_relaxed_u32(&t->iq), ld_relaxed_u64(&t->id), ld_relaxed_u64(&t->ie)};
          pre = seg3_op(v, pre);
          break;
        }
        Seg3 v{0u, ld_relaxed_u32(&t->aq), ld_relaxed_u64(&t->ad), ld_relaxed_u64(&t->ae)};
        pre = seg3_op(v, pre);
        p--;
      }
      if (!total.f) {
        Seg3 inc = seg3_op(pre, total);
        me->iq = inc.q;
        me->id = inc.d;
        me->ie = inc.e;
        fence_gpu();
        st_relaxed_u32(&me->flag, kFlagIncl);
      }
    }
    s_prefix = pre;
  }
  __syncthreads();

  // pass 2: per word, only where needed (a tile boundary falls in it, it is the list's
  // last word, or a cheap test says it may be malformed), walk the groups: write the tile
  // Entries and check the groups' bounds
  uint32_t err = 0;
  auto walk_word = [&](uint64_t w, uint32_t li, const WCtx& c, const Seg3& SW) {
    ListCur L;
    L.load(D, la + li);
    word_walk<C>(c, [&](const Grp& g) {
      uint64_t gq = (uint64_t)SW.q + g.q0;
      if (gq < L.Q && g.err) err |= g.err;
      if (gq >= L.Q || g.nq == 0) return;
      uint64_t ge = mn64(gq + g.nq, L.Q);
      uint64_t gdata = SW.d + (int64_t)g.d0;
      uint64_t gexc = SW.e + g.e0;
      if (gdata < L.dbase || gdata + g.dlen > L.dlim) err |= GC_DEV_TRUNCATED;
      if (C::kExc && gexc + g.elen > L.elim) err |= GC_DEV_TRUNCATED;
      uint64_t lo_int = L.oo + 4 * gq;
      uint64_t hi_int = L.oo + mn64(4 * ge, L.n);
      uint64_t t = (lo_int + kT - 1) / kT;
      if (t * kT < hi_int && t < D.n_tiles_b) {
        uint64_t j = (t * kT - L.oo) >> 2;
        Entry e;
        e.l = (uint32_t)L.l;
        e.j = (uint32_t)j;
        e.wq = SW.q;
        e.valid = 1;
        e.gword = w;
        e.wd = SW.d;
        e.we = SW.e;
        e.dbeg = gdata;
        e.ebeg = gexc;
        e.cend = w + 1;
        if (j > gq) {  // the boundary splits a multi-quad group
          e.dend = gdata + 32ull * (((j - gq) * g.step + 31) / 32);
          e.eend = gexc + g.elen;
        } else {
          e.dend = gdata;
          e.eend = gexc;
        }
        D.entries[t] = e;
      }
    });
  };
  Seg3 S = seg3_op(s_prefix, excl);
  for (uint32_t k = 0; k < kCA; k++) {
    if (k >= mynl) break;
    const uint64_t w = my0 + k;
    const uint32_t wr = (uint32_t)(w - w0);
    const uint32_t li = wli[k];
    const uint32_t widx = wr - s_cw[li];
    const uint32_t Q = s_q[li];
    const WCtx c{s_w[wr + 1], s_w[wr], widx, Q, 0u};
    const WAgg a = wa_[k];
    if (widx == 0) {
      const uint64_t l = la + li;
      S = Seg3{1u, 0u, D.data_off[l] * 32ull, D.exc_off ? D.exc_off[l] : 0ull};
    }
    const Seg3 SW = S;
    S.q += a.q;
    S.d += a.d;
    S.e += a.e;
    const bool last = li + 1 < nl ? s_cw[li + 1] == wr + 1
                                  : (uint64_t)(D.ctrl_off[la + li + 1] >> 2) == w + 1;
    if (last && S.q < Q) err |= GC_DEV_TRUNCATED;  // the control ends before Q quads
    const uint32_t qa = SW.q, qb = min(SW.q + a.q, Q);
    const uint32_t jb0 = s_jb[li];
    bool boundary = false;
    if (qb > qa && qb > jb0) {
      const uint32_t kk = qa > jb0 ? (qa - jb0 + (kT / 4) - 1) / (kT / 4) : 0u;
      boundary = jb0 + kk * (kT / 4) < qb;
    }
    if (!(boundary || last || C::suspect(c))) continue;
    // compact the words that need a group walk into a queue so the walks run lane-dense
    const uint32_t slot = atomicAdd(&s_nq, 1u);
    if (slot < kQueue) {
      s_qw[slot] = wr | (li << 16);
      s_qq[slot] = SW.q;
      s_qd[slot] = SW.d;
      if (C::kExc) s_qe[slot] = SW.e;
    } else {
      walk_word(w, li, c, SW);  // queue full: walk in place
    }
  }
  __syncthreads();
  const uint32_t nq = min(s_nq, kQueue);
  for (uint32_t i = tid; i < nq; i += kThreads) {
    const uint32_t wr = s_qw[i] & 0xFFFFu, li = s_qw[i] >> 16;
    const Seg3 SW{0u, s_qq[i], s_qd[i], C::kExc ? s_qe[i] : 0ull};
    const WCtx c{s_w[wr + 1], s_w[wr], wr - s_cw[li], s_q[li], 0u};
    walk_word(w0 + wr, li, c, SW);
  }
  report(&s_err, err);
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(&D.hdr->status, s_err);
}

#include "gc_decode.cuh"

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

struct WsLayout {
  uint64_t n_tiles_a, n_tiles_b;
  uint64_t off_tiles_a, off_tiles_b, off_entries, bytes;
};

WsLayout ws_layout(const gc_batch* b) {
  WsLayout L;
  uint64_t words = b->ctrl_bytes / 4;
  L.n_tiles_a = (words + kWA - 1) / kWA;
  if (L.n_tiles_a == 0) L.n_tiles_a = 1;
  L.n_tiles_b = (b->total_out + kT - 1) / kT;
  L.off_tiles_a = sizeof(WsHeader);
  L.off_tiles_b = L.off_tiles_a + L.n_tiles_a * sizeof(TileA);
  L.off_entries = L.off_tiles_b + ((L.n_tiles_b * 8 + 255) & ~255ull);
  L.bytes = L.off_entries + L.n_tiles_b * sizeof(Entry);
  return L;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

gc_status check_codec(const gc_batch* b) {
  switch (b->codec) {
    case GC_GROUP_SIMPLE:
    case GC_GROUP_AFOR:
      return b->variant == 0 ? GC_OK : GC_ERR_BAD_VARIANT;
    case GC_GROUP_SCHEME: {
      uint32_t kind = (b->variant >> 2) & 3u, cg = 1u << (b->variant & 3u);
      if (b->variant > 15 || kind > 2 || (kind == 2 && cg < 4)) return GC_ERR_BAD_VARIANT;
      return GC_OK;
    }
    case GC_GROUP_PFD:
      return (b->pfd_frame_quads == 32 || b->pfd_frame_quads == 128) ? GC_OK : GC_ERR_BAD_VARIANT;
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
  if (b->total_out && !b->n_lists) return GC_ERR_INVALID_ARGUMENT;
  if (b->total_out > (1ull << 40) || b->n_lists > 0xFFFFFFF0ull) return GC_ERR_INVALID_ARGUMENT;
  (void)device_ptrs;
  return GC_OK;
}

gc_status check_device() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0;
    cudaDeviceProp prop;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
      return GC_ERR_CUDA;
    ok = prop.major == 10 ? 1 : 0;
  }
  return ok ? GC_OK : GC_ERR_UNSUPPORTED_DEVICE;
}

template <class C>
gc_status launch_codec(const Dev& D, uint32_t* out, bool dgaps, cudaStream_t st, int stages) {
  if (stages & GC_STAGE_INDEX) {
    k_index<C><<<(unsigned)D.n_tiles_a, kThreads, 0, st>>>(D);
    if (cudaGetLastError() != cudaSuccess) return GC_ERR_CUDA;
  }
  if (D.n_tiles_b == 0 || !(stages & GC_STAGE_DECODE)) return GC_OK;
  constexpr int kWPC = C::kExc ? 7 : 8;  // warps per CTA (shared memory: 2 CTAs per SM)
  const uint32_t smem = kWPC * WarpSmem::bytes(C::kExc);
  static bool attr_set[2] = {false, false};
  static int n_sm = 0;
  auto kern = dgaps ? k_decode<C, true, kWPC> : k_decode<C, false, kWPC>;
  if (!attr_set[dgaps]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return GC_ERR_CUDA;
    attr_set[dgaps] = true;
  }
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  // persistent: enough CTAs to fill every SM, never more warps than tiles
  const uint64_t want = (D.n_tiles_b + kWPC - 1) / kWPC;
  const unsigned grid = (unsigned)mn64(want, (uint64_t)n_sm * 2);
  kern<<<grid, 32 * kWPC, smem, st>>>(D, out);
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

gc_status decode_impl(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                      void* stream, bool dgaps, int stages = GC_STAGE_ALL) {
  gc_status s = check_batch(b, true);
  if (s != GC_OK) return s;
  if (!ws || !aligned16(ws) || (b->total_out && (!out || !aligned16(out))))
    return GC_ERR_INVALID_ARGUMENT;
  WsLayout L = ws_layout(b);
  if (ws_bytes < L.bytes) return GC_ERR_WORKSPACE_TOO_SMALL;
  s = check_device();
  if (s != GC_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* w = (uint8_t*)ws;
  if ((stages & GC_STAGE_RESET) && cudaMemsetAsync(ws, 0, L.bytes, st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (b->n_lists == 0 || b->total_out == 0) return GC_OK;
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
  D.n_tiles_b = (uint32_t)L.n_tiles_b;
  D.hdr = (WsHeader*)w;
  D.tiles_a = (TileA*)(w + L.off_tiles_a);
  D.tiles_b = (uint64_t*)(w + L.off_tiles_b);
  D.entries = (Entry*)(w + L.off_entries);
  switch (b->codec) {
    case GC_GROUP_SIMPLE:
      return launch_codec<CodecGS>(D, out, dgaps, st, stages);
    case GC_GROUP_AFOR:
      return launch_codec<CodecAFOR>(D, out, dgaps, st, stages);
    case GC_GROUP_PFD:
      return b->pfd_frame_quads == 32 ? launch_codec<CodecPFD<32>>(D, out, dgaps, st, stages)
                                      : launch_codec<CodecPFD<128>>(D, out, dgaps, st, stages);
    default:
      break;
  }
  switch (b->variant) {
    case 0: return launch_codec<CodecGscB<1>>(D, out, dgaps, st, stages);
    case 1: return launch_codec<CodecGscB<2>>(D, out, dgaps, st, stages);
    case 2: return launch_codec<CodecGscB<4>>(D, out, dgaps, st, stages);
    case 3: return launch_codec<CodecGscB<8>>(D, out, dgaps, st, stages);
    case 4: return launch_codec<CodecGscCU<1>>(D, out, dgaps, st, stages);
    case 5: return launch_codec<CodecGscCU<2>>(D, out, dgaps, st, stages);
    case 6: return launch_codec<CodecGscCU<4>>(D, out, dgaps, st, stages);
    case 7: return launch_codec<CodecGscCU<8>>(D, out, dgaps, st, stages);
    case 10: return launch_codec<CodecGscIU<4>>(D, out, dgaps, st, stages);
    case 11: return launch_codec<CodecGscIU<8>>(D, out, dgaps, st, stages);
    default: return GC_ERR_BAD_VARIANT;
  }
}

}  // namespace

extern "C" {

int gc_abi_version(void) { return GC_ABI_VERSION; }

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
  return decode_impl(b, out, ws, ws_bytes, stream, false);
}

gc_status gc_decode_dgaps(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                          void* stream) {
  return decode_impl(b, out, ws, ws_bytes, stream, true);
}

gc_status gc_decode_stage(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                          void* stream, int dgaps, int stage_mask) {
  if (stage_mask & ~GC_STAGE_ALL) return GC_ERR_INVALID_ARGUMENT;
  return decode_impl(b, out, ws, ws_bytes, stream, dgaps != 0, stage_mask);
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
  s = decode_impl(&d, dout, ws, wsb, stream, dgaps != 0);
  if (s != GC_OK) return s;
  if (hb->total_out && cudaMemcpyAsync(host_out, dout, 4 * hb->total_out, cudaMemcpyDeviceToHost,
                                       st) != cudaSuccess)
    return GC_ERR_CUDA;
  return GC_OK;
}

}  // extern "C"
