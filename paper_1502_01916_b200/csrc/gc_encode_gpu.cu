// gc_encode_gpu.cu -- GPU encoder of the frame codecs: Group-PFD and SIMD-BP128 (PFD
// variant 1), SURVEY §8(f) rank 1 ("Group-PFD (per frame)").  The bytes are identical to
// the oracle's / the host encoder's (tests/test_gpu_encoder.py), DESIGN §3.5:
//   * frame = F quads (4F ints, the tail frame q < F quads, A33), 4-way vertical layout;
//   * b = smallest b in 1..32 with #{quads of the frame with width(quad max) > b} * den <=
//     num * q (P:L404 Step 2, A28); SIMD-BP128: the width of the frame's largest int
//     (zeta = 0);
//   * exceptions = every int of the frame wider than b, ascending position p = 4j+k (A29);
//     stored at the smallest of 8/16/32 bits holding the frame's largest one (A30);
//   * control: {b, wcode, count16 LE} per frame (A31); exception stream: count positions
//     (u8, u16 LE when 4F > 256) then count values (LE); data: the low b bits of all 4q ints,
//     high-first split (A3), a fresh vector per frame;
//   * batch: lists in order, per-list control padded to 4 bytes (a frame header is 4),
//     totals of the control and exception streams padded to 16 bytes.
//
// One warp per frame: lane j holds quad j (F = 32) or quads j, j+32, j+64, j+96 (F = 128).
// Pass 1 (k_fr_plan) writes each frame's (b, wcode, count, vectors, exception bytes);
// device-wide exclusive scans over frames give every frame's data vector and exception
// byte offsets (and so the directory); pass 2 (k_fr_write) packs the frame's data in shared
// memory with atomicOr and writes header, vectors and exception records.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "gc.h"

namespace gce {

constexpr uint32_t kWarpsPerBlock = 8;

__device__ __forceinline__ uint32_t width_of(uint32_t x) { return x ? 32u - __clz(x) : 1u; }
__device__ __forceinline__ uint32_t low_bits(uint32_t v, uint32_t b) {
  return b >= 32u ? v : (v & ((1u << b) - 1u));
}

struct Dir {
  const uint32_t* values;  // docIDs when delta, else the ints to store
  const uint32_t* list_n;
  uint64_t n_lists;
  int delta;
  uint32_t F, zn, zd, bp128;
  uint64_t* out_off;     // [L+1]
  uint64_t* frame_off;   // [L+1] first frame of each list
  uint64_t n_frames;
  uint32_t* rec;         // [n_frames][4]: b | wcode<<8 | count<<16 ; vectors ; exc bytes ; -
  uint64_t* vec_off;     // [n_frames+1] exclusive scan of vectors
  uint64_t* exb_off;     // [n_frames+1] exclusive scan of exception bytes
};

// ------------------------------------------------------------------ device-wide u64 scan
// Exclusive scan of a[0..n) into s[0..n] (s[n] = total): per-block sums, one block scans
// them, then every block scans its elements from its offset.
constexpr uint32_t kScanT = 256, kScanPer = 8, kScanB = kScanT * kScanPer;

__device__ __forceinline__ uint64_t block_excl_u64(uint64_t v, uint64_t* scr, uint64_t* tot) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += n;
  }
  if (lane == 31) scr[warp] = inc;
  __syncthreads();
  uint64_t w = lane < kScanT / 32 ? scr[lane] : 0ull;
#pragma unroll
  for (int o = 1; o < (int)(kScanT / 32); o <<= 1) {
    const uint64_t n = __shfl_up_sync(0xffffffffu, w, o);
    if (lane >= (uint32_t)o) w += n;
  }
  const uint64_t wpre = warp ? __shfl_sync(0xffffffffu, w, warp - 1) : 0ull;
  *tot = __shfl_sync(0xffffffffu, w, kScanT / 32 - 1);
  __syncthreads();
  return wpre + inc - v;
}

template <class Get>
__global__ void __launch_bounds__(kScanT) k_scan_sums(Get get, uint64_t n, uint64_t* sums) {
  __shared__ uint64_t scr[kScanT / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanB + threadIdx.x * kScanPer;
  uint64_t t = 0;
  for (uint32_t k = 0; k < kScanPer; k++)
    if (base + k < n) t += get(base + k);
  uint64_t tot;
  block_excl_u64(t, scr, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(kScanT) k_scan_top(uint64_t* sums, uint64_t nb) {
  __shared__ uint64_t scr[kScanT / 32];
  uint64_t carry = 0;
  for (uint64_t c0 = 0; c0 < nb; c0 += kScanT) {
    const uint64_t i = c0 + threadIdx.x;
    const uint64_t v = i < nb ? sums[i] : 0ull;
    uint64_t tot;
    const uint64_t ex = block_excl_u64(v, scr, &tot);
    if (i < nb) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}
template <class Get>
__global__ void __launch_bounds__(kScanT) k_scan_apply(Get get, uint64_t n, const uint64_t* sums,
                                                       uint64_t* s) {
  __shared__ uint64_t scr[kScanT / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanB + threadIdx.x * kScanPer;
  uint64_t v[kScanPer], t = 0;
  for (uint32_t k = 0; k < kScanPer; k++) {
    v[k] = base + k < n ? get(base + k) : 0ull;
    t += v[k];
  }
  uint64_t tot;
  uint64_t run = sums[blockIdx.x] + block_excl_u64(t, scr, &tot);
  for (uint32_t k = 0; k < kScanPer; k++) {
    if (base + k < n) s[base + k] = run;
    run += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) s[n] = sums[gridDim.x];
}

template <class Get>
cudaError_t scan_u64(Get get, uint64_t n, uint64_t* s, uint64_t* sums, cudaStream_t st) {
  const uint64_t nb = n ? (n + kScanB - 1) / kScanB : 1;
  k_scan_sums<<<(unsigned)nb, kScanT, 0, st>>>(get, n, sums);
  k_scan_top<<<1, kScanT, 0, st>>>(sums, nb);
  k_scan_apply<<<(unsigned)nb, kScanT, 0, st>>>(get, n, sums, s);
  return cudaGetLastError();
}

struct GetListN {
  const uint32_t* p;
  __device__ uint64_t operator()(uint64_t i) const { return p[i]; }
};
struct GetFrames {
  const uint32_t* list_n;
  uint32_t F;
  __device__ uint64_t operator()(uint64_t i) const {
    const uint64_t Q = (list_n[i] + 3ull) >> 2;
    return (Q + F - 1) / F;
  }
};
struct GetRec {
  const uint32_t* rec;
  uint32_t field;
  __device__ uint64_t operator()(uint64_t i) const { return rec[4 * i + field]; }
};

// ------------------------------------------------------------------ frames
struct FrameCtx {
  uint64_t l, e0;   // list, first element of the frame
  uint32_t n, q;    // ints of the list, quads of the frame
  uint32_t k;       // frame index within the list
};
__device__ __forceinline__ FrameCtx frame_ctx(const Dir& D, uint64_t f) {
  uint64_t a = 0, b = D.n_lists;  // the last list whose first frame is <= f (non-empty)
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (D.frame_off[m] <= f) a = m;
    else b = m;
  }
  FrameCtx c;
  c.l = a;
  c.n = D.list_n[a];
  c.k = (uint32_t)(f - D.frame_off[a]);
  const uint64_t Q = (c.n + 3ull) >> 2;
  c.q = (uint32_t)((Q - (uint64_t)c.k * D.F) < D.F ? (Q - (uint64_t)c.k * D.F) : D.F);
  c.e0 = D.out_off[a] + 4ull * D.F * c.k;
  return c;
}
// the 4 ints of quad j of the frame (zeros past the list's end; d-gaps if delta)
__device__ __forceinline__ void load_quad(const Dir& D, const FrameCtx& c, uint32_t j, uint32_t* v) {
  const uint64_t p0 = 4ull * D.F * c.k + 4ull * j;  // position in the list
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const uint64_t p = p0 + t;
    uint32_t x = 0;
    if (p < c.n) {
      x = D.values[c.e0 + 4ull * j + t];
      if (D.delta && p > 0) x -= D.values[c.e0 + 4ull * j + t - 1];
    }
    v[t] = x;
  }
}

// pass 1: (b, wcode, count, vectors, exception bytes) of every frame
__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_fr_plan(Dir D) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t f = (uint64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (f >= D.n_frames) return;
  const FrameCtx c = frame_ctx(D, f);
  const uint32_t R = D.F / 32;  // quads per lane
  uint32_t qw[4], qv[4][4];
  uint32_t maxw = 0;
  for (uint32_t r = 0; r < R; r++) {
    const uint32_t j = 32 * r + lane;
    qw[r] = 0;
    if (j < c.q) {
      load_quad(D, c, j, qv[r]);
      qw[r] = width_of(qv[r][0] | qv[r][1] | qv[r][2] | qv[r][3]);  // width of the quad max (A9)
      maxw = max(maxw, qw[r]);
    }
  }
  maxw = __reduce_max_sync(0xffffffffu, maxw);
  uint32_t b = maxw ? maxw : 1u;
  if (!D.bp128) {  // P:L404 Step 2: the smallest b whose exceptional quads are within zeta
    for (uint32_t cb = 1; cb <= 32; cb++) {
      uint32_t cnt = 0;
      for (uint32_t r = 0; r < R; r++) cnt += __popc(__ballot_sync(0xffffffffu, qw[r] > cb));
      if ((uint64_t)cnt * D.zd <= (uint64_t)D.zn * c.q) {
        b = cb;
        break;
      }
    }
  }
  // exceptions: ints wider than b (A29), and the largest of them (A30)
  uint32_t cnt = 0, mx = 0;
  for (uint32_t r = 0; r < R; r++) {
    const uint32_t j = 32 * r + lane;
    if (j < c.q)
      for (int t = 0; t < 4; t++)
        if (width_of(qv[r][t]) > b) {
          cnt++;
          mx = max(mx, qv[r][t]);
        }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  mx = __reduce_max_sync(0xffffffffu, mx);
  const uint32_t wc = cnt ? (mx <= 0xFFu ? 1u : (mx <= 0xFFFFu ? 2u : 3u)) : 0u;
  const uint32_t wb = wc == 1 ? 1u : (wc == 2 ? 2u : (wc == 3 ? 4u : 0u));
  const uint32_t pb = 4 * D.F <= 256 ? 1u : 2u;
  if (lane == 0) {
    uint32_t* rr = D.rec + 4 * f;
    rr[0] = b | (wc << 8) | (cnt << 16);
    rr[1] = (c.q * b + 31u) / 32u;
    rr[2] = cnt * (pb + wb);
    rr[3] = 0;
  }
}

// pass 2: header, data vectors, exception records of every frame
__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_fr_write(Dir D, uint8_t* ctrl, uint4* data,
                                                                  uint8_t* exc) {
  __shared__ uint32_t s_pack[kWarpsPerBlock][4 * 32 + 4];  // a frame's lane streams (<= 32 words
                                                            // per lane at F = 32)
  const uint32_t lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint64_t f = (uint64_t)blockIdx.x * kWarpsPerBlock + wi;
  if (f >= D.n_frames) return;
  const FrameCtx c = frame_ctx(D, f);
  const uint32_t* rr = D.rec + 4 * f;
  const uint32_t h = rr[0], nvec = rr[1];
  const uint32_t b = h & 0xFFu, wc = (h >> 8) & 0xFFu, cnt = h >> 16;
  const uint32_t wb = wc == 1 ? 1u : (wc == 2 ? 2u : (wc == 3 ? 4u : 0u));
  const uint32_t pb = 4 * D.F <= 256 ? 1u : 2u;
  if (lane == 0) *reinterpret_cast<uint32_t*>(ctrl + 4 * f) = h;  // {b, wcode, count16 LE}
  uint32_t* pk = s_pack[wi];
  const uint64_t vbase = D.vec_off[f];
  uint8_t* ex = exc + D.exb_off[f];
  const uint32_t R = D.F / 32;
  uint32_t xoff = 0;  // exceptions of earlier rounds
  // data: the frame's vectors, packed in shared memory a round of 32 quads at a time (a
  // round's lane streams are 32*b bits = b words, starting at word b*r)
  for (uint32_t r = 0; r < R; r++) {
    for (uint32_t w = lane; w < 4 * 32 + 4; w += 32) pk[w] = 0;
    __syncwarp();
    const uint32_t j = 32 * r + lane;
    uint32_t v[4] = {0, 0, 0, 0};
    if (j < c.q) load_quad(D, c, j, v);
    // this round's quad lane at bit (j - 32r)*b of the round's stream (fresh words)
    const uint32_t pos = lane * b, m = pos >> 5, off = pos & 31u, rem = 32u - off;
    if (j < c.q) {
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const uint32_t x = low_bits(v[t], b);
        if (b <= rem) {
          atomicOr(&pk[4 * m + t], x << off);
        } else {  // high part at the top of word m, low part at the bottom of word m+1 (A3)
          const uint32_t lo = b - rem;
          atomicOr(&pk[4 * m + t], (x >> lo) << off);
          atomicOr(&pk[4 * (m + 1) + t], low_bits(x, lo));
        }
      }
    }
    __syncwarp();
    // the round covers vectors [b*r, b*r + b) of the frame (the last one may be partial)
    const uint32_t v0 = b * r, v1 = min(nvec, b * r + b);
    for (uint32_t m2 = v0 + lane; m2 < v1; m2 += 32) {
      const uint32_t mm = m2 - v0;
      data[vbase + m2] = make_uint4(pk[4 * mm], pk[4 * mm + 1], pk[4 * mm + 2], pk[4 * mm + 3]);
    }
    // exceptions of this round, in ascending position p = 4j + t
    uint32_t mine = 0;
    if (j < c.q)
      for (int t = 0; t < 4; t++) mine += width_of(v[t]) > b ? 1u : 0u;
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += n;
    }
    uint32_t rank = xoff + incl - mine;
    if (j < c.q)
      for (int t = 0; t < 4; t++)
        if (width_of(v[t]) > b) {
          const uint32_t p = 4 * j + t;
          ex[rank * pb] = (uint8_t)(p & 0xFFu);
          if (pb == 2) ex[rank * pb + 1] = (uint8_t)(p >> 8);
          for (uint32_t y = 0; y < wb; y++) ex[cnt * pb + rank * wb + y] = (uint8_t)(v[t] >> (8 * y));
          rank++;
        }
    xoff += __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
  }
}

// directory from the scans: ctrl = 4 bytes per frame, data / exceptions from the frame scans
__global__ void k_fr_dir(Dir D, uint64_t* ctrl_off, uint64_t* data_off, uint64_t* exc_off) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l > D.n_lists) return;
  const uint64_t f = D.frame_off[l];
  ctrl_off[l] = 4 * f;
  data_off[l] = D.vec_off[f];
  exc_off[l] = D.exb_off[f];
}

// ------------------------------------------------------------------ Group-Scheme (B, CU)
// Binary and complete-unary LD (A12-A18).  Per quad: u = ceil(width(quad max) /
// CG) (Eq. 1 with the outer ceiling, A12), BW = CG*u (Eq. 2).  Global exclusive scans over
// all quads of BW (and, for CU, of the code length u) give every quad's offsets: a list's
// base is the scan at its first quad and its sizes are differences of the scan, so no
// segmented scan is needed.  Binary fields sit at closed-form places (A18); unary codes
// (u-1 ones then a 0, MSB-first in address order, A15/A16) and the data bits (high-first
// split, A3) are OR-ed into the zeroed streams.
struct Gsc {
  const uint32_t* values;
  const uint32_t* list_n;
  uint64_t n_lists;
  int delta;
  uint32_t cg, kind;       // CG, 0 binary / 1 complete unary
  uint64_t* out_off;       // [L+1]
  uint64_t* quad_off;      // [L+1] first quad of each list
  uint64_t n_quads;
  uint8_t* u;              // [n_quads] units per quad
  uint64_t* bw_off;        // [n_quads+1] exclusive scan of BW (lane bits)
  uint64_t* cu_off;        // [n_quads+1] exclusive scan of u (CU control bits)
  uint32_t* lstart;        // [n_quads] lists starting at each quad (list ids >= 1)
  uint64_t* lid;           // [n_quads+1] exclusive scan of lstart: lid[g+1] = list of quad g
};
struct GetStarts {
  const uint32_t* p;
  __device__ uint64_t operator()(uint64_t i) const { return p[i]; }
};
// lstart[quad_off[l]] += 1 for every list l >= 1 (empty lists share their successor's start),
// so the inclusive scan at quad g counts the lists starting at or before g: g's list
__global__ void k_gsc_lstart(Gsc G) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (l >= G.n_lists) return;
  const uint64_t q = G.quad_off[l];
  if (q < G.n_quads) atomicAdd(&G.lstart[q], 1u);
}
struct GetQuads {
  const uint32_t* list_n;
  __device__ uint64_t operator()(uint64_t i) const { return (list_n[i] + 3ull) >> 2; }
};
struct GetBW {
  const uint8_t* u;
  uint32_t cg;
  __device__ uint64_t operator()(uint64_t i) const { return (uint64_t)cg * u[i]; }
};
struct GetU {
  const uint8_t* u;
  __device__ uint64_t operator()(uint64_t i) const { return u[i]; }
};
// the list of quad g (lid: the scan of the list-start counts, k_gsc_lstart)
__device__ __forceinline__ uint64_t quad_list(const Gsc& G, uint64_t g) {
  return g < G.n_quads ? G.lid[g + 1] : 0;
}
__device__ __forceinline__ void gsc_quad(const Gsc& G, uint64_t l, uint64_t j, uint32_t* v) {
  const uint32_t n = G.list_n[l];
  const uint64_t e = G.out_off[l] + 4 * j;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const uint64_t p = 4 * j + t;
    uint32_t x = 0;
    if (p < n) {
      x = G.values[e + t];
      if (G.delta && p > 0) x -= G.values[e + t - 1];  // d-gaps
    }
    v[t] = x;
  }
}
__global__ void k_gsc_units(Gsc G) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t l = quad_list(G, g);
  if (g >= G.n_quads) return;
  uint32_t v[4];
  gsc_quad(G, l, g - G.quad_off[l], v);
  const uint32_t w = width_of(v[0] | v[1] | v[2] | v[3]);  // width of the quad max (A9)
  G.u[g] = (uint8_t)((w + G.cg - 1) / G.cg);               // A12
}
// per list: control bytes (4-byte padded) and data vectors
__global__ void k_gsc_sizes(Gsc G, uint64_t* cb, uint64_t* vecs) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= G.n_lists) return;
  const uint64_t qs = G.quad_off[l], qe = G.quad_off[l + 1], Q = qe - qs;
  uint64_t bytes;
  if (G.kind == 1) {
    bytes = (G.cu_off[qe] - G.cu_off[qs] + 7) / 8;
  } else {  // A18: CG 1 three 5-bit fields per 16-bit unit, CG 2/4 two per byte, CG 8 four
    bytes = G.cg == 1 ? 2 * ((Q + 2) / 3) : (G.cg == 8 ? (Q + 3) / 4 : (Q + 1) / 2);
  }
  if (G.kind != 2) cb[l] = 4 * ((bytes + 3) / 4);  // (IU: k_iu_chain)
  vecs[l] = (G.bw_off[qe] - G.bw_off[qs] + 31) / 32;
}
// incomplete unary (A17): a code never crosses a byte -- if it does not fit in the rest of
// the current byte, that rest is filled with 1s and the code starts the next byte; the last
// byte is filled with 1s too.  The placement is a sequential state per list (bits used in
// the current byte, 0..7), so lists are cut into chunks of kIuChunk quads: every chunk's
// bit advance for each of the 8 entry states (in parallel), one thread per list chains its
// chunks, then every chunk places its codes from its entry position (cu_off[g] = the code's
// bit position within the list's control area).
constexpr uint32_t kIuChunk = 256;
struct GetIuChunks {
  const uint64_t* quad_off;
  __device__ uint64_t operator()(uint64_t i) const {
    return (quad_off[i + 1] - quad_off[i] + kIuChunk - 1) / kIuChunk;
  }
};
__device__ __forceinline__ uint64_t iu_walk(const Gsc& G, uint64_t g0, uint64_t g1, uint64_t p,
                                            uint64_t* pos) {
  for (uint64_t g = g0; g < g1; g++) {
    const uint32_t u = G.u[g], used = (uint32_t)(p & 7);
    if (used != 0 && used + u > 8) p = (p + 7) & ~7ull;
    if (pos) pos[g] = p;
    p += u;
  }
  return p;
}
struct IuChunk {
  const uint64_t* ch_off;  // [L+1] first chunk of each list
  uint64_t n_chunks;
  uint32_t* adv;           // [n_chunks][8] bit advance from entry state s
  uint64_t* start;         // [n_chunks] entry position (bits from the list's start)
};
__device__ __forceinline__ uint64_t list_of_chunk(const Gsc& G, const IuChunk& K, uint64_t c) {
  uint64_t a = 0, b = G.n_lists;
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (K.ch_off[m] <= c) a = m;
    else b = m;
  }
  return a;
}
__global__ void k_iu_adv(Gsc G, IuChunk K) {  // thread = (chunk, entry state)
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 8 * K.n_chunks) return;
  const uint64_t c = t >> 3;
  const uint32_t st = (uint32_t)(t & 7);
  const uint64_t l = list_of_chunk(G, K, c);
  const uint64_t g0 = G.quad_off[l] + (c - K.ch_off[l]) * kIuChunk;
  const uint64_t g1 = min(g0 + kIuChunk, G.quad_off[l + 1]);
  K.adv[t] = (uint32_t)(iu_walk(G, g0, g1, st, nullptr) - st);
}
__global__ void k_iu_chain(Gsc G, IuChunk K, uint64_t* cb) {  // thread = list
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= G.n_lists) return;
  uint64_t p = 0;
  for (uint64_t c = K.ch_off[l]; c < K.ch_off[l + 1]; c++) {
    K.start[c] = p;
    p += K.adv[8 * c + (p & 7)];
  }
  const uint64_t bytes = (p + 7) / 8;
  cb[l] = 4 * ((bytes + 3) / 4);
}
__global__ void k_iu_place(Gsc G, IuChunk K) {  // thread = chunk
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K.n_chunks) return;
  const uint64_t l = list_of_chunk(G, K, c);
  const uint64_t g0 = G.quad_off[l] + (c - K.ch_off[l]) * kIuChunk;
  const uint64_t g1 = min(g0 + kIuChunk, G.quad_off[l + 1]);
  iu_walk(G, g0, g1, K.start[c], G.cu_off);
}
__device__ __forceinline__ void or_byte_bits(uint8_t* base, uint64_t byte, uint32_t bits) {
  // OR `bits` (8 bits) into the byte at `byte` through its aligned 32-bit word
  if (!bits) return;
  uint32_t* w = reinterpret_cast<uint32_t*>(base + (byte & ~3ull));
  atomicOr(w, bits << (8 * (uint32_t)(byte & 3)));
}
// one quad's control: its binary field (A18) or its unary code (+ IU padding 1s)
__device__ __forceinline__ void gsc_ctrl(const Gsc& G, uint64_t g, uint64_t l, const uint64_t* ctrl_off,
                                         uint8_t* ctrl) {
  const uint64_t qs = G.quad_off[l], j = g - qs;
  const uint32_t u = G.u[g];
  // control
  const uint64_t cbase = ctrl_off[l];
  if (G.kind >= 1) {  // (u-1) ones then a 0, MSB-first in address order
    const uint64_t c = G.kind == 1 ? G.cu_off[g] - G.cu_off[qs] : G.cu_off[g];
    auto ones = [&](uint64_t from, uint64_t to) {  // stream bits [from, to) set, a byte at a time
      for (uint64_t i = from; i < to;) {
        const uint64_t byte = i >> 3;
        const uint64_t e = to - 8 * byte;
        const uint32_t b0 = (uint32_t)(i & 7), b1 = e < 8 ? (uint32_t)e : 8u;
        or_byte_bits(ctrl, cbase + byte, ((0xFFu >> b0) & ~(0xFFu >> b1)) & 0xFFu);
        i = 8 * byte + b1;
      }
    };
    ones(c, c + u - 1);
    if (G.kind == 2) {  // IU: the 1s that fill the byte up to the next code (or its end)
      const uint64_t end = c + u;
      const uint64_t next = g + 1 < G.quad_off[l + 1] ? G.cu_off[g + 1] : (end + 7) & ~7ull;
      ones(end, next);
    }
  } else {
    const uint32_t f = u - 1;  // A13: binary stores u - 1
    uint64_t byte;
    uint32_t sh;
    if (G.cg == 1) { byte = 2 * (j / 3); sh = 5 * (uint32_t)(j % 3); }
    else if (G.cg == 2) { byte = j / 2; sh = 4 * (uint32_t)(j % 2); }
    else if (G.cg == 4) { byte = j / 2; sh = 3 * (uint32_t)(j % 2); }
    else { byte = j / 4; sh = 2 * (uint32_t)(j % 4); }
    const uint64_t a = cbase + byte;  // (a 16-bit unit never crosses its aligned word)
    atomicOr(reinterpret_cast<uint32_t*>(ctrl + (a & ~3ull)), f << (sh + 8 * (uint32_t)(a & 3)));
  }
}

constexpr uint32_t kGscSpan = 72;  // data words a warp's 32 quads can touch (<= 65)
__global__ void __launch_bounds__(256) k_gsc_write(Gsc G, const uint64_t* ctrl_off,
                                                   const uint64_t* data_off, uint8_t* ctrl,
                                                   uint32_t* data) {
  __shared__ uint32_t s_pack[8][4 * kGscSpan];
  const uint32_t lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = g < G.n_quads;
  const uint64_t lw = quad_list(G, g);
  uint64_t pos = 0;
  uint32_t bw = 0, v[4] = {0, 0, 0, 0};
  if (act) {
    const uint64_t l = lw, qs = G.quad_off[l];
    bw = G.cg * G.u[g];
    gsc_quad(G, l, g - qs, v);
    pos = data_off[l] * 32 + (G.bw_off[g] - G.bw_off[qs]);
    gsc_ctrl(G, g, l, ctrl_off, ctrl);
  }
  // data: the warp's 32 quads are consecutive in the data stream; pack them in shared
  // memory, store the interior words, OR only the two end words a neighbour may share
  if (__all_sync(0xffffffffu, !act)) return;
  uint64_t m_lo = act ? (pos >> 5) : ~0ull, m_hi = act ? ((pos + bw - 1) >> 5) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m_lo = min(m_lo, (uint64_t)__shfl_xor_sync(0xffffffffu, m_lo, o));
    m_hi = max(m_hi, (uint64_t)__shfl_xor_sync(0xffffffffu, m_hi, o));
  }
  uint32_t* pk = s_pack[wi];
  const uint64_t span = m_hi - m_lo + 1;
  if (span > kGscSpan) {  // (cannot happen for 32 quads; kept for safety) -- OR directly
    if (act) {
      const uint64_t m = pos >> 5;
      const uint32_t off = (uint32_t)(pos & 31), rem = 32u - off;
      for (int t = 0; t < 4; t++) {
        const uint32_t x = low_bits(v[t], bw);
        if (bw <= rem) atomicOr(&data[4 * m + t], x << off);
        else {
          atomicOr(&data[4 * m + t], (x >> (bw - rem)) << off);
          atomicOr(&data[4 * (m + 1) + t], low_bits(x, bw - rem));
        }
      }
    }
    return;
  }
  for (uint32_t w = lane; w < 4 * span; w += 32) pk[w] = 0;
  __syncwarp();
  if (act) {
    const uint32_t m = (uint32_t)((pos >> 5) - m_lo), off = (uint32_t)(pos & 31), rem = 32u - off;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const uint32_t x = low_bits(v[t], bw);
      if (!x) continue;
      if (bw <= rem) {
        atomicOr(&pk[4 * m + t], x << off);
      } else {  // high part at the top of word m, low part at the bottom of word m+1 (A3)
        atomicOr(&pk[4 * m + t], (x >> (bw - rem)) << off);
        atomicOr(&pk[4 * (m + 1) + t], low_bits(x, bw - rem));
      }
    }
  }
  __syncwarp();
  for (uint32_t w = lane; w < 4 * span; w += 32) {
    const uint32_t word = w >> 2, x = pk[w];
    uint32_t* dst = &data[4 * (m_lo + word) + (w & 3)];
    if (word == 0 || word + 1 == span) {
      if (x) atomicOr(dst, x);
    } else {
      *dst = x;
    }
  }
}
struct WsLayout {
  uint64_t frame_off, rec, vec_off, exb_off, sums, bytes;
};
// the frame count is only known on the device: the workspace is sized for its upper bound
inline WsLayout ws_layout(uint64_t n_lists, uint64_t total, uint32_t F) {
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t nf = total / (4ull * F) + 2 * n_lists + 1;  // >= sum over lists of ceil(Q/F)
  const uint64_t nsum = (std::max(nf, n_lists) + 1) / kScanB + 2;
  WsLayout L;
  L.frame_off = 0;
  L.rec = L.frame_off + al(8 * (n_lists + 1));
  L.vec_off = L.rec + al(16 * nf);
  L.exb_off = L.vec_off + al(8 * (nf + 1));
  L.sums = L.exb_off + al(8 * (nf + 1));
  L.bytes = L.sums + al(8 * (nsum + 1));
  return L;
}

// ------------------------------------------------------------------ Group-AFOR
// P:L392 §6.1 with the readings A22-A25: the quad-max widths of a list padded with zero
// quads (width 1) to a multiple of 8; a backward DP over the 8-quad slots, frame lengths
// L tried in the order 32, 16, 8 and replaced only on strict improvement of
// 8 + 128*ceil(L*bw/32) + (cost of the rest); header byte = code(8/16/32 -> 0/1/2) |
// (bw-1) << 2; each frame's data starts a fresh vector.  Lists in parallel (one thread
// runs a list's DP over precomputed 8-quad block maxima), frames written by one warp each.
struct Afor {
  const uint32_t* values;
  const uint32_t* list_n;
  uint64_t n_lists;
  int delta;
  uint64_t* out_off;     // [L+1]
  uint64_t* blk_off;     // [L+1] first 8-quad block of each list
  uint64_t n_blocks;
  uint8_t* bmax;         // [n_blocks] max quad width of the block
  uint8_t* fstart;       // [n_blocks] L of the frame starting here, 0 if none
  uint8_t* fbw;          // [n_blocks] its bw
  uint32_t* fvec;        // [n_blocks] its first vector within the list
  uint32_t* fidx;        // [n_blocks] its index within the list
  uint64_t* cost;        // [n_blocks] DP cost of the list from this block on
  uint64_t* nf;          // [n_lists] frames of each list
  uint64_t* nv;          // [n_lists] vectors of each list
};
struct GetBlocks {
  const uint32_t* list_n;
  __device__ uint64_t operator()(uint64_t i) const {
    const uint64_t Q = (list_n[i] + 3ull) >> 2;
    return (Q + 7) / 8;
  }
};
__device__ __forceinline__ uint64_t list_of_block(const Afor& A, uint64_t g) {
  uint64_t a = 0, b = A.n_lists;
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (A.blk_off[m] <= g) a = m;
    else b = m;
  }
  return a;
}
__device__ __forceinline__ void afor_quad(const Afor& A, uint64_t l, uint64_t j, uint32_t* v) {
  const uint32_t n = A.list_n[l];
  const uint64_t e = A.out_off[l] + 4 * j;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const uint64_t p = 4 * j + t;
    uint32_t x = 0;
    if (p < n) {
      x = A.values[e + t];
      if (A.delta && p > 0) x -= A.values[e + t - 1];  // d-gaps
    }
    v[t] = x;
  }
}
__global__ void k_afor_bmax(Afor A) {  // one thread per 8-quad block
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= A.n_blocks) return;
  const uint64_t l = list_of_block(A, g), s = g - A.blk_off[l];
  uint32_t m = 1;
  for (uint32_t t = 0; t < 8; t++) {
    uint32_t v[4];
    afor_quad(A, l, 8 * s + t, v);  // (zero past the list: width 1, A25)
    m = max(m, width_of(v[0] | v[1] | v[2] | v[3]));
  }
  A.bmax[g] = (uint8_t)m;
}
__global__ void k_afor_dp(Afor A) {  // one thread per list
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= A.n_lists) return;
  const uint64_t b0 = A.blk_off[l], S = A.blk_off[l + 1] - b0;
  // the DP's dependency chain stays in registers: the costs of the next 4 slots (cost of the
  // rest past the list end = 0) and the block maxima of the next 3 slots slide with s, so a
  // step waits on no memory round trip (the costs went through global memory before: one L2
  // round trip per slot, 42.9 ms for config 4's longest lists)
  uint64_t c1 = 0, c2 = 0, c4a = 0, c4b = 0;  // cost[s+1], cost[s+2], cost[s+3], cost[s+4]
  uint32_t m1 = 0, m2 = 0, m3 = 0;            // bmax[s+1], bmax[s+2], bmax[s+3]
  for (int64_t s = (int64_t)S - 1; s >= 0; s--) {
    const uint32_t m0 = A.bmax[b0 + s];
    const uint64_t left = (uint64_t)S - (uint64_t)s;  // slots from s to the list end
    uint64_t best = ~0ull;
    uint8_t bl = 8;
    uint32_t bw = max(1u, m0), bbw = bw;
#pragma unroll
    for (uint32_t L = 8; L <= 32; L <<= 1) {  // bw of the first L quads from s
      if (L / 8 > left) break;
      if (L == 16) bw = max(bw, m1);
      if (L == 32) bw = max(bw, max(m2, m3));
      // candidates in the oracle's order 32, 16, 8: evaluate all, pick by that order below
      const uint64_t rest = L == 8 ? c1 : (L == 16 ? c2 : c4b);
      const uint64_t c = 8 + 128 * (((uint64_t)L * bw + 31) / 32) + rest;
      // strict improvement in the order 32, 16, 8 == the smallest cost, ties to the longest L
      if (c < best || (c == best && L > bl)) {
        best = c;
        bl = (uint8_t)L;
        bbw = bw;
      }
    }
    A.fstart[b0 + s] = bl;  // (the choice; turned into frame starts below)
    A.fbw[b0 + s] = (uint8_t)bbw;  // (its width: read back only where a frame starts)
    c4b = c4a;
    c4a = c2;
    c2 = c1;
    c1 = best;
    m3 = m2;
    m2 = m1;
    m1 = m0;
  }
  // forward: the frames, their bw, vector offsets and indices
  uint64_t f = 0, vec = 0;
  uint64_t s = 0;
  while (s < S) {
    const uint32_t L = A.fstart[b0 + s], bw = A.fbw[b0 + s];
    for (uint32_t k = 1; k < L / 8; k++) A.fstart[b0 + s + k] = 0;
    A.fvec[b0 + s] = (uint32_t)vec;
    A.fidx[b0 + s] = (uint32_t)f;
    vec += ((uint64_t)L * bw + 31) / 32;
    f++;
    s += L / 8;
  }
  A.nf[l] = 4 * ((f + 3) / 4);  // control bytes: one header per frame, padded to 4
  A.nv[l] = vec;
}
__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_afor_write(Afor A, const uint64_t* ctrl_off,
                                                                   const uint64_t* data_off,
                                                                   uint8_t* ctrl, uint4* data) {
  __shared__ uint32_t s_pack[kWarpsPerBlock][4 * 32 + 4];
  const uint32_t lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint64_t g = (uint64_t)blockIdx.x * kWarpsPerBlock + wi;
  if (g >= A.n_blocks) return;
  const uint32_t L = A.fstart[g];
  if (!L) return;  // (warp-uniform)
  const uint64_t l = list_of_block(A, g), s = g - A.blk_off[l];
  const uint32_t bw = A.fbw[g];
  if (lane == 0) {
    const uint32_t code = L == 8 ? 0u : (L == 16 ? 1u : 2u);
    ctrl[ctrl_off[l] + A.fidx[g]] = (uint8_t)(code | ((bw - 1) << 2));  // A22 header byte
  }
  uint32_t* pk = s_pack[wi];
  for (uint32_t w = lane; w < 4 * 32 + 4; w += 32) pk[w] = 0;
  __syncwarp();
  if (lane < L) {
    uint32_t v[4];
    afor_quad(A, l, 8 * s + lane, v);
    const uint32_t pos = lane * bw, m = pos >> 5, off = pos & 31u, rem = 32u - off;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const uint32_t x = low_bits(v[t], bw);
      if (bw <= rem) {
        atomicOr(&pk[4 * m + t], x << off);
      } else {
        const uint32_t lo = bw - rem;
        atomicOr(&pk[4 * m + t], (x >> lo) << off);
        atomicOr(&pk[4 * (m + 1) + t], low_bits(x, lo));
      }
    }
  }
  __syncwarp();
  const uint32_t nvec = (L * bw + 31) / 32;
  const uint64_t vb = data_off[l] + A.fvec[g];
  for (uint32_t m2 = lane; m2 < nvec; m2 += 32)
    data[vb + m2] = make_uint4(pk[4 * m2], pk[4 * m2 + 1], pk[4 * m2 + 2], pk[4 * m2 + 3]);
}
struct AforWs {
  uint64_t blk_off, bmax, fstart, fbw, fvec, fidx, cost, nf, nv, sums, bytes;
};
inline AforWs afor_ws_layout(uint64_t n_lists, uint64_t total) {
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t nb = total / 32 + n_lists + 1;  // >= sum over lists of ceil(ceil(n/4)/8)
  const uint64_t nsum = (std::max(nb, n_lists) + 1) / kScanB + 2;
  AforWs L;
  L.blk_off = 0;
  L.bmax = L.blk_off + al(8 * (n_lists + 1));
  L.fstart = L.bmax + al(nb);
  L.fbw = L.fstart + al(nb);
  L.fvec = L.fbw + al(nb);
  L.fidx = L.fvec + al(4 * nb);
  L.cost = L.fidx + al(4 * nb);
  L.nf = L.cost + al(8 * nb);
  L.nv = L.nf + al(8 * (n_lists + 1));
  L.sums = L.nv + al(8 * (n_lists + 1));
  L.bytes = L.sums + al(8 * (nsum + 1));
  return L;
}

// ------------------------------------------------------------------ Group-Simple
// Algorithm 1 is a greedy over a list's quad maxima.  Its step from any quad
// depends only on the quad maxima ahead, so every quad's step (selector, quads covered) is
// computed in parallel; one thread per list then follows the chain from quad 0 (one load
// per selector) and numbers the selectors; every selector start writes its nibble (low
// first, A6) and its 128-bit vector (int t of a component at [t*BW, (t+1)*BW), A7).
__constant__ uint32_t kGsNum[10] = {32, 16, 10, 8, 6, 5, 4, 3, 2, 1};
__constant__ uint32_t kGsBw[10] = {1, 2, 3, 4, 5, 6, 8, 10, 16, 32};
struct GsEnc {
  const uint32_t* values;
  const uint32_t* list_n;
  uint64_t n_lists;
  int delta;
  uint64_t* out_off;
  uint64_t* cb;        // [L+1] control bytes (4-padded), then the exclusive scan
  uint64_t* nv;        // [L+1] selectors = vectors, then the exclusive scan
  uint64_t* quad_off;  // [L+1] first quad of each list
  uint32_t* M;         // [quads] quad maxima, precomputed in parallel
  uint64_t n_quads;
};
__device__ __forceinline__ void gs_quad(const GsEnc& E, uint64_t e0, uint32_t n, uint64_t j,
                                        uint32_t* v) {
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const uint64_t p = 4 * j + t;
    uint32_t x = 0;
    if (p < n) {
      x = E.values[e0 + p];
      if (E.delta && p > 0) x -= E.values[e0 + p - 1];  // d-gaps
    }
    v[t] = x;
  }
}
__global__ void k_gs_qmax(GsEnc E) {  // one thread per quad
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= E.n_quads) return;
  uint64_t a = 0, b = E.n_lists;  // the last list whose first quad is <= g
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (E.quad_off[m] <= g) a = m;
    else b = m;
  }
  uint32_t v[4];
  gs_quad(E, E.out_off[a], E.list_n[a], g - E.quad_off[a], v);
  E.M[g] = max(max(v[0], v[1]), max(v[2], v[3]));
}
// one selector of Algorithm 1 at quad j with l quads left: (SEL i, quads covered)
__device__ __forceinline__ void gs_next(const uint32_t* M, uint64_t j, uint64_t l, uint32_t& sel,
                                        uint64_t& pos) {
  uint32_t i;
  for (i = 0; i <= 9; i++) {
    const uint64_t nn = kGsNum[i], mask = (1ull << kGsBw[i]) - 1;  // 64-bit mask (A8)
    const uint64_t lim = nn < l ? nn : l;
    pos = 0;
    while (pos < lim && (uint64_t)M[j + pos] <= mask) pos++;
    if (pos == nn || pos == l) break;
  }
  sel = i;
}
// the selector Algorithm 1 would emit if one started at quad g, and the quads it covers
// (every quad in parallel; only the chain from each list's quad 0 is used)
__global__ void k_gs_step(GsEnc E, uint8_t* sel, uint8_t* cov) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= E.n_quads) return;
  uint64_t a = 0, b = E.n_lists;
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (E.quad_off[m] <= g) a = m;
    else b = m;
  }
  const uint64_t q0 = E.quad_off[a], j = g - q0, Q = E.quad_off[a + 1] - q0;
  uint32_t s;
  uint64_t pos;
  gs_next(E.M + q0, j, Q - j, s, pos);
  sel[g] = (uint8_t)s;
  cov[g] = (uint8_t)pos;
}
// per list: follow the chain from quad 0 (one load per selector), number the selectors
__global__ void k_gs_chase(GsEnc E, const uint8_t* cov, uint32_t* idx) {
  const uint64_t li = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= E.n_lists) return;
  const uint64_t q0 = E.quad_off[li], Q = E.quad_off[li + 1] - q0;
  uint64_t j = 0, T = 0;
  while (j < Q) {
    idx[q0 + j] = (uint32_t)T++;
    j += cov[q0 + j];
  }
  E.cb[li] = 4 * (((T + 1) / 2 + 3) / 4);  // nibbles, low first (A6), padded to 4 bytes
  E.nv[li] = T;                            // one vector per selector
}
// every selector start: its nibble and its vector (int t of a component at t*BW, A7)
__global__ void k_gs_write(GsEnc E, const uint8_t* sel, const uint8_t* cov, const uint32_t* idx,
                           uint8_t* ctrl, uint4* data) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= E.n_quads || idx[g] == ~0u) return;
  uint64_t a = 0, b = E.n_lists;
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (E.quad_off[m] <= g) a = m;
    else b = m;
  }
  const uint32_t s = idx[g], SEL = sel[g], c = cov[g], BW = kGsBw[SEL];
  const uint64_t q0 = E.quad_off[a], e0 = E.out_off[a];
  const uint32_t n = E.list_n[a];
  uint32_t cmp[4] = {0, 0, 0, 0};
  for (uint32_t t = 0; t < c; t++) {
    uint32_t v[4];
    gs_quad(E, e0, n, g - q0 + t, v);
#pragma unroll
    for (int k = 0; k < 4; k++) cmp[k] |= v[k] << (t * BW);
  }
  data[E.nv[a] + s] = make_uint4(cmp[0], cmp[1], cmp[2], cmp[3]);
  const uint64_t byte = E.cb[a] + (s >> 1);
  atomicOr(reinterpret_cast<uint32_t*>(ctrl + (byte & ~3ull)),
           (SEL << (4 * (s & 1))) << (8 * (uint32_t)(byte & 3)));
}

// ------------------------------------------------------------------ Variable Byte
// P §2.3: an int takes ceil(width/7) bytes (width(0) = 1), 7-bit groups
// least significant first, MSB = 1 on the last.  One thread per int: a global exclusive
// scan of the byte lengths gives every int's position; per-list byte counts (differences of
// the scan) padded to 4 and scanned over the lists give the directory.
struct Vb {
  const uint32_t* values;
  const uint32_t* list_n;
  uint64_t n_lists, n;
  int delta;
  uint64_t* out_off;   // [L+1]
  uint8_t* len;        // [n] bytes per int
  uint64_t* pos;       // [n+1] exclusive scan of len
  uint64_t* cb;        // [L+1] control bytes per list (4-padded), then their scan
};
struct GetLen {
  const uint8_t* p;
  __device__ uint64_t operator()(uint64_t i) const { return p[i]; }
};
__device__ __forceinline__ uint64_t vb_list_of(const Vb& V, uint64_t i) {
  uint64_t a = 0, b = V.n_lists;  // the last list whose first int is <= i
  while (b - a > 1) {
    const uint64_t m = (a + b) >> 1;
    if (V.out_off[m] <= i) a = m;
    else b = m;
  }
  return a;
}
__device__ __forceinline__ uint32_t vb_value(const Vb& V, uint64_t i, uint64_t l) {
  uint32_t x = V.values[i];
  if (V.delta && i > V.out_off[l]) x -= V.values[i - 1];  // d-gaps
  return x;
}
__global__ void k_vb_len(Vb V) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V.n) return;
  const uint32_t x = vb_value(V, i, vb_list_of(V, i));
  V.len[i] = (uint8_t)((width_of(x) + 6) / 7);
}
__global__ void k_vb_sizes(Vb V) {
  const uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= V.n_lists) return;
  const uint64_t bytes = V.pos[V.out_off[l + 1]] - V.pos[V.out_off[l]];
  V.cb[l] = 4 * ((bytes + 3) / 4);
}
__global__ void k_vb_write(Vb V, const uint64_t* ctrl_off, uint8_t* ctrl) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V.n) return;
  const uint64_t l = vb_list_of(V, i);
  uint32_t x = vb_value(V, i, l);
  uint64_t p = ctrl_off[l] + (V.pos[i] - V.pos[V.out_off[l]]);
  const uint32_t k = V.len[i];
  for (uint32_t j = 0; j < k; j++, x >>= 7) ctrl[p + j] = (uint8_t)((x & 127u) | (j + 1 == k ? 128u : 0u));
}
struct VbWs {
  uint64_t len, pos, cb, sums, bytes;
};
inline VbWs vb_ws_layout(uint64_t n_lists, uint64_t total) {
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  VbWs L;
  L.len = 0;
  L.pos = al(total + 1);
  L.cb = L.pos + al(8 * (total + 1));
  L.sums = L.cb + al(8 * (n_lists + 1));
  L.bytes = L.sums + al(8 * ((std::max(total, n_lists) + 1) / kScanB + 3));
  return L;
}

struct GscWs {
  uint64_t quad_off, u, bw_off, cu_off, c_off, d_off, ch_off, adv, start, lstart, lid, sums, bytes;
};
inline GscWs gsc_ws_layout(uint64_t n_lists, uint64_t total) {
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t nq = total / 4 + n_lists + 1;  // >= sum over lists of ceil(n/4)
  const uint64_t nsum = (std::max(nq, n_lists) + 1) / kScanB + 2;
  GscWs L;
  L.quad_off = 0;
  L.u = L.quad_off + al(8 * (n_lists + 1));
  L.bw_off = L.u + al(nq);
  L.cu_off = L.bw_off + al(8 * (nq + 1));
  L.c_off = L.cu_off + al(8 * (nq + 1));
  L.d_off = L.c_off + al(8 * (n_lists + 1));
  const uint64_t nch = nq / kIuChunk + n_lists + 1;  // IU chunks
  L.ch_off = L.d_off + al(8 * (n_lists + 1));
  L.adv = L.ch_off + al(8 * (n_lists + 1));
  L.start = L.adv + al(32 * nch);
  L.lstart = L.start + al(8 * nch);
  L.lid = L.lstart + al(4 * nq);
  L.sums = L.lid + al(8 * (nq + 1));
  L.bytes = L.sums + al(8 * (nsum + 1));
  return L;
}
struct GetArr {
  const uint64_t* p;
  __device__ uint64_t operator()(uint64_t i) const { return p[i]; }
};
__global__ void k_copy_u64(const uint64_t* a, uint64_t* b, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

}  // namespace gce

using namespace gce;

namespace {
bool is_pfd(const gc_encode_params* p) {
  return p->codec == GC_GROUP_PFD && (p->pfd_frame_quads == 32 || p->pfd_frame_quads == 128) &&
         p->variant <= 1 && (p->variant == 1 || p->zeta_den > 0);
}
bool is_gsc(const gc_encode_params* p) {  // binary, complete unary, incomplete unary (CG 4/8)
  const uint32_t kind = (p->variant >> 2) & 3u, cg = 1u << (p->variant & 3u);
  return p->codec == GC_GROUP_SCHEME && p->variant <= 15 && kind <= 2 && !(kind == 2 && cg < 4);
}
bool is_afor(const gc_encode_params* p) { return p->codec == GC_GROUP_AFOR; }
bool is_gs(const gc_encode_params* p) { return p->codec == GC_GROUP_SIMPLE; }
bool is_vb(const gc_encode_params* p) { return p->codec == GC_VARBYTE; }
Vb make_vb(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists, uint64_t total,
           int delta, uint64_t* out_off, void* ws) {
  const VbWs L = vb_ws_layout(n_lists, total);
  uint8_t* w = (uint8_t*)ws;
  Vb V;
  V.values = values;
  V.list_n = list_n;
  V.n_lists = n_lists;
  V.n = total;
  V.delta = delta;
  V.out_off = out_off;
  V.len = w + L.len;
  V.pos = (uint64_t*)(w + L.pos);
  V.cb = (uint64_t*)(w + L.cb);
  return V;
}
gc_status refuse(const gc_encode_params* p) {
  if (!p) return GC_ERR_INVALID_ARGUMENT;
  if (p->codec != GC_GROUP_PFD && p->codec != GC_GROUP_SCHEME) return GC_ERR_UNKNOWN_CODEC;
  return GC_ERR_BAD_VARIANT;
}
struct GsWs {
  uint64_t cb, nv, quad_off, M, sel, cov, idx, sums, bytes;
};
inline GsWs gs_ws_layout(uint64_t n_lists, uint64_t total) {
  auto al = [](uint64_t x) { return (x + 255) & ~255ull; };
  const uint64_t nq = total / 4 + n_lists + 1;
  GsWs L;
  L.cb = 0;
  L.nv = al(8 * (n_lists + 1));
  L.quad_off = L.nv + al(8 * (n_lists + 1));
  L.M = L.quad_off + al(8 * (n_lists + 1));
  L.sel = L.M + al(4 * nq);
  L.cov = L.sel + al(nq);
  L.idx = L.cov + al(nq);
  L.sums = L.idx + al(4 * nq);
  L.bytes = L.sums + al(8 * ((n_lists + 1) / kScanB + 3));
  return L;
}
GsEnc make_gs(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists, int delta,
              uint64_t* out_off, void* ws, uint64_t total) {
  const GsWs L = gs_ws_layout(n_lists, total);
  GsEnc E;
  E.values = values;
  E.list_n = list_n;
  E.n_lists = n_lists;
  E.delta = delta;
  E.out_off = out_off;
  E.cb = (uint64_t*)((uint8_t*)ws + L.cb);
  E.nv = (uint64_t*)((uint8_t*)ws + L.nv);
  E.quad_off = (uint64_t*)((uint8_t*)ws + L.quad_off);
  E.M = (uint32_t*)((uint8_t*)ws + L.M);
  E.n_quads = 0;
  return E;
}
Afor make_afor(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists, int delta,
               uint64_t* out_off, void* ws, uint64_t total) {
  const AforWs L = afor_ws_layout(n_lists, total);
  uint8_t* w = (uint8_t*)ws;
  Afor A;
  A.values = values;
  A.list_n = list_n;
  A.n_lists = n_lists;
  A.delta = delta;
  A.out_off = out_off;
  A.blk_off = (uint64_t*)(w + L.blk_off);
  A.n_blocks = 0;
  A.bmax = w + L.bmax;
  A.fstart = w + L.fstart;
  A.fbw = w + L.fbw;
  A.fvec = (uint32_t*)(w + L.fvec);
  A.fidx = (uint32_t*)(w + L.fidx);
  A.cost = (uint64_t*)(w + L.cost);
  A.nf = (uint64_t*)(w + L.nf);
  A.nv = (uint64_t*)(w + L.nv);
  return A;
}
Gsc make_gsc(const gc_encode_params* p, const uint32_t* values, const uint32_t* list_n,
             uint64_t n_lists, int delta, uint64_t* out_off, void* ws, uint64_t total) {
  const GscWs L = gsc_ws_layout(n_lists, total);
  uint8_t* w = (uint8_t*)ws;
  Gsc G;
  G.values = values;
  G.list_n = list_n;
  G.n_lists = n_lists;
  G.delta = delta;
  G.cg = 1u << (p->variant & 3u);
  G.kind = (p->variant >> 2) & 3u;
  G.out_off = out_off;
  G.quad_off = (uint64_t*)(w + L.quad_off);
  G.n_quads = 0;
  G.u = w + L.u;
  G.bw_off = (uint64_t*)(w + L.bw_off);
  G.cu_off = (uint64_t*)(w + L.cu_off);
  G.lstart = (uint32_t*)(w + L.lstart);
  G.lid = (uint64_t*)(w + L.lid);
  return G;
}
Dir make_dir(const gc_encode_params* p, const uint32_t* values, const uint32_t* list_n,
             uint64_t n_lists, int delta, uint64_t* out_off, void* ws, uint64_t total) {
  const WsLayout L = ws_layout(n_lists, total, p->pfd_frame_quads);
  uint8_t* w = (uint8_t*)ws;
  Dir D;
  D.values = values;
  D.list_n = list_n;
  D.n_lists = n_lists;
  D.delta = delta;
  D.F = p->pfd_frame_quads;
  D.bp128 = p->variant == 1;
  D.zn = D.bp128 ? 0u : p->zeta_num;
  D.zd = D.bp128 ? 1u : p->zeta_den;
  D.out_off = out_off;
  D.frame_off = (uint64_t*)(w + L.frame_off);
  D.n_frames = 0;
  D.rec = (uint32_t*)(w + L.rec);
  D.vec_off = (uint64_t*)(w + L.vec_off);
  D.exb_off = (uint64_t*)(w + L.exb_off);
  return D;
}
}  // namespace

extern "C" {

gc_status gc_encode_device_ws_size(const gc_encode_params* p, uint64_t n_lists, uint64_t total_ints,
                                   uint64_t* bytes) {
  if (!p || !bytes) return GC_ERR_INVALID_ARGUMENT;
  if (is_pfd(p)) *bytes = ws_layout(n_lists, total_ints, p->pfd_frame_quads).bytes;
  else if (is_gsc(p)) *bytes = gsc_ws_layout(n_lists, total_ints).bytes;
  else if (is_afor(p)) *bytes = afor_ws_layout(n_lists, total_ints).bytes;
  else if (is_gs(p)) *bytes = gs_ws_layout(n_lists, total_ints).bytes;
  else if (is_vb(p)) *bytes = vb_ws_layout(n_lists, total_ints).bytes;
  else return refuse(p);
  return GC_OK;
}

static gc_status gsc_plan(const gc_encode_params* p, const uint32_t* values, const uint32_t* list_n,
                          uint64_t n_lists, uint64_t total_ints, int delta, uint64_t* ctrl_off,
                          uint64_t* data_off, uint64_t* exc_off, uint64_t* out_off, void* ws,
                          uint64_t* sizes, cudaStream_t st) {
  const GscWs L = gsc_ws_layout(n_lists, total_ints);
  Gsc G = make_gsc(p, values, list_n, n_lists, delta, out_off, ws, total_ints);
  uint8_t* w = (uint8_t*)ws;
  uint64_t* sums = (uint64_t*)(w + L.sums);
  uint64_t* c_off = (uint64_t*)(w + L.c_off);
  uint64_t* d_off = (uint64_t*)(w + L.d_off);
  if (scan_u64(GetListN{list_n}, n_lists, out_off, sums, st) != cudaSuccess ||
      scan_u64(GetQuads{list_n}, n_lists, G.quad_off, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  uint64_t nq = 0, tot = 0;
  if (cudaMemcpyAsync(&nq, G.quad_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&tot, out_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (tot != total_ints) return GC_ERR_INVALID_ARGUMENT;
  G.n_quads = nq;
  if (nq) {  // the list of every quad (no per-quad search)
    if (cudaMemsetAsync(G.lstart, 0, 4 * nq, st) != cudaSuccess) return GC_ERR_CUDA;
    if (n_lists > 1) k_gsc_lstart<<<(unsigned)((n_lists + 255) / 256), 256, 0, st>>>(G);
    if (scan_u64(GetStarts{G.lstart}, nq, G.lid, sums, st) != cudaSuccess) return GC_ERR_CUDA;
    k_gsc_units<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(G);
  }
  if (scan_u64(GetBW{G.u, G.cg}, nq, G.bw_off, sums, st) != cudaSuccess) return GC_ERR_CUDA;
  if (G.kind == 1 && scan_u64(GetU{G.u}, nq, G.cu_off, sums, st) != cudaSuccess) return GC_ERR_CUDA;
  if (G.kind == 2 && n_lists) {
    IuChunk K;
    K.ch_off = (uint64_t*)(w + L.ch_off);
    K.adv = (uint32_t*)(w + L.adv);
    K.start = (uint64_t*)(w + L.start);
    if (scan_u64(GetIuChunks{G.quad_off}, n_lists, const_cast<uint64_t*>(K.ch_off), sums, st) != cudaSuccess)
      return GC_ERR_CUDA;
    uint64_t nch = 0;
    if (cudaMemcpyAsync(&nch, K.ch_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return GC_ERR_CUDA;
    K.n_chunks = nch;
    if (nch) k_iu_adv<<<(unsigned)((8 * nch + 255) / 256), 256, 0, st>>>(G, K);
    k_iu_chain<<<(unsigned)((n_lists + 127) / 128), 128, 0, st>>>(G, K, c_off);
    if (nch) k_iu_place<<<(unsigned)((nch + 127) / 128), 128, 0, st>>>(G, K);
  }
  if (n_lists) k_gsc_sizes<<<(unsigned)((n_lists + 255) / 256), 256, 0, st>>>(G, c_off, d_off);
  // exclusive scans in place: the per-list sizes become the list offsets
  if (scan_u64(GetArr{c_off}, n_lists, c_off, sums, st) != cudaSuccess ||
      scan_u64(GetArr{d_off}, n_lists, d_off, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  const unsigned nb = (unsigned)((n_lists + 1 + 255) / 256);
  k_copy_u64<<<nb, 256, 0, st>>>(c_off, ctrl_off, n_lists + 1);
  k_copy_u64<<<nb, 256, 0, st>>>(d_off, data_off, n_lists + 1);
  if (cudaMemsetAsync(exc_off, 0, 8 * (n_lists + 1), st) != cudaSuccess) return GC_ERR_CUDA;
  uint64_t ct = 0, vt = 0;
  if (cudaMemcpyAsync(&ct, c_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&vt, d_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  sizes[0] = 16 * ((ct + 15) / 16);
  sizes[1] = vt;
  sizes[2] = 0;
  sizes[3] = nq;
  return GC_OK;
}

static gc_status vb_plan(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists,
                         uint64_t total_ints, int delta, uint64_t* ctrl_off, uint64_t* data_off,
                         uint64_t* exc_off, uint64_t* out_off, void* ws, uint64_t* sizes,
                         cudaStream_t st) {
  const VbWs L = vb_ws_layout(n_lists, total_ints);
  Vb V = make_vb(values, list_n, n_lists, total_ints, delta, out_off, ws);
  uint64_t* sums = (uint64_t*)((uint8_t*)ws + L.sums);
  if (scan_u64(GetListN{list_n}, n_lists, out_off, sums, st) != cudaSuccess) return GC_ERR_CUDA;
  uint64_t tot = 0;
  if (cudaMemcpyAsync(&tot, out_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (tot != total_ints) return GC_ERR_INVALID_ARGUMENT;
  if (total_ints) k_vb_len<<<(unsigned)((total_ints + 255) / 256), 256, 0, st>>>(V);
  if (scan_u64(GetLen{V.len}, total_ints, V.pos, sums, st) != cudaSuccess) return GC_ERR_CUDA;
  if (n_lists) k_vb_sizes<<<(unsigned)((n_lists + 255) / 256), 256, 0, st>>>(V);
  if (scan_u64(GetArr{V.cb}, n_lists, V.cb, sums, st) != cudaSuccess) return GC_ERR_CUDA;
  const unsigned nbl = (unsigned)((n_lists + 1 + 255) / 256);
  k_copy_u64<<<nbl, 256, 0, st>>>(V.cb, ctrl_off, n_lists + 1);
  if (cudaMemsetAsync(data_off, 0, 8 * (n_lists + 1), st) != cudaSuccess ||
      cudaMemsetAsync(exc_off, 0, 8 * (n_lists + 1), st) != cudaSuccess)
    return GC_ERR_CUDA;
  uint64_t ct = 0;
  if (cudaMemcpyAsync(&ct, V.cb + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  sizes[0] = 16 * ((ct + 15) / 16);
  sizes[1] = 0;
  sizes[2] = 0;
  sizes[3] = total_ints;
  return GC_OK;
}

static gc_status gs_plan(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists,
                         uint64_t total_ints, int delta, uint64_t* ctrl_off, uint64_t* data_off,
                         uint64_t* exc_off, uint64_t* out_off, void* ws, uint64_t* sizes,
                         cudaStream_t st) {
  const GsWs L = gs_ws_layout(n_lists, total_ints);
  GsEnc E = make_gs(values, list_n, n_lists, delta, out_off, ws, total_ints);
  uint64_t* sums = (uint64_t*)((uint8_t*)ws + L.sums);
  if (scan_u64(GetListN{list_n}, n_lists, out_off, sums, st) != cudaSuccess ||
      scan_u64(GetQuads{list_n}, n_lists, E.quad_off, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  uint64_t tot = 0, nq = 0;
  if (cudaMemcpyAsync(&tot, out_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&nq, E.quad_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (tot != total_ints) return GC_ERR_INVALID_ARGUMENT;
  E.n_quads = nq;
  uint8_t* w = (uint8_t*)ws;
  uint32_t* idx = (uint32_t*)(w + L.idx);
  if (nq) {
    k_gs_qmax<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(E);
    k_gs_step<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(E, w + L.sel, w + L.cov);
    if (cudaMemsetAsync(idx, 0xFF, 4 * nq, st) != cudaSuccess) return GC_ERR_CUDA;
  }
  if (n_lists) k_gs_chase<<<(unsigned)((n_lists + 127) / 128), 128, 0, st>>>(E, w + L.cov, idx);
  if (scan_u64(GetArr{E.cb}, n_lists, E.cb, sums, st) != cudaSuccess ||
      scan_u64(GetArr{E.nv}, n_lists, E.nv, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  const unsigned nbl = (unsigned)((n_lists + 1 + 255) / 256);
  k_copy_u64<<<nbl, 256, 0, st>>>(E.cb, ctrl_off, n_lists + 1);
  k_copy_u64<<<nbl, 256, 0, st>>>(E.nv, data_off, n_lists + 1);
  if (cudaMemsetAsync(exc_off, 0, 8 * (n_lists + 1), st) != cudaSuccess) return GC_ERR_CUDA;
  uint64_t ct = 0, vt = 0;
  if (cudaMemcpyAsync(&ct, E.cb + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&vt, E.nv + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  sizes[0] = 16 * ((ct + 15) / 16);
  sizes[1] = vt;
  sizes[2] = 0;
  sizes[3] = nq;
  return GC_OK;
}

static gc_status afor_plan(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists,
                           uint64_t total_ints, int delta, uint64_t* ctrl_off, uint64_t* data_off,
                           uint64_t* exc_off, uint64_t* out_off, void* ws, uint64_t* sizes,
                           cudaStream_t st) {
  const AforWs L = afor_ws_layout(n_lists, total_ints);
  Afor A = make_afor(values, list_n, n_lists, delta, out_off, ws, total_ints);
  uint64_t* sums = (uint64_t*)((uint8_t*)ws + L.sums);
  if (scan_u64(GetListN{list_n}, n_lists, out_off, sums, st) != cudaSuccess ||
      scan_u64(GetBlocks{list_n}, n_lists, A.blk_off, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  uint64_t nb = 0, tot = 0;
  if (cudaMemcpyAsync(&nb, A.blk_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&tot, out_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (tot != total_ints) return GC_ERR_INVALID_ARGUMENT;
  A.n_blocks = nb;
  if (nb) k_afor_bmax<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(A);
  if (n_lists) k_afor_dp<<<(unsigned)((n_lists + 127) / 128), 128, 0, st>>>(A);
  // the per-list sizes become the list offsets (exclusive scans in place)
  if (scan_u64(GetArr{A.nf}, n_lists, A.nf, sums, st) != cudaSuccess ||
      scan_u64(GetArr{A.nv}, n_lists, A.nv, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  const unsigned nbl = (unsigned)((n_lists + 1 + 255) / 256);
  k_copy_u64<<<nbl, 256, 0, st>>>(A.nf, ctrl_off, n_lists + 1);
  k_copy_u64<<<nbl, 256, 0, st>>>(A.nv, data_off, n_lists + 1);
  if (cudaMemsetAsync(exc_off, 0, 8 * (n_lists + 1), st) != cudaSuccess) return GC_ERR_CUDA;
  uint64_t ct = 0, vt = 0;
  if (cudaMemcpyAsync(&ct, A.nf + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&vt, A.nv + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  sizes[0] = 16 * ((ct + 15) / 16);
  sizes[1] = vt;
  sizes[2] = 0;
  sizes[3] = nb;
  return GC_OK;
}

gc_status gc_encode_device_plan(const gc_encode_params* p, const uint32_t* values,
                                const uint32_t* list_n, uint64_t n_lists, uint64_t total_ints,
                                int delta, uint64_t* ctrl_off, uint64_t* data_off,
                                uint64_t* exc_off, uint64_t* out_off, void* ws, uint64_t ws_bytes,
                                uint64_t* sizes, void* stream) {
  uint64_t need = 0;
  const gc_status s0 = gc_encode_device_ws_size(p, n_lists, total_ints, &need);
  if (s0 != GC_OK) return s0;
  if (!ws || !sizes || !ctrl_off || !data_off || !exc_off || !out_off ||
      (n_lists && !list_n) || (total_ints && !values))
    return GC_ERR_INVALID_ARGUMENT;
  if (ws_bytes < need) return GC_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = (cudaStream_t)stream;
  if (is_gsc(p))
    return gsc_plan(p, values, list_n, n_lists, total_ints, delta, ctrl_off, data_off, exc_off,
                    out_off, ws, sizes, st);
  if (is_afor(p))
    return afor_plan(values, list_n, n_lists, total_ints, delta, ctrl_off, data_off, exc_off,
                     out_off, ws, sizes, st);
  if (is_gs(p))
    return gs_plan(values, list_n, n_lists, total_ints, delta, ctrl_off, data_off, exc_off,
                   out_off, ws, sizes, st);
  if (is_vb(p))
    return vb_plan(values, list_n, n_lists, total_ints, delta, ctrl_off, data_off, exc_off,
                   out_off, ws, sizes, st);
  const WsLayout L = ws_layout(n_lists, total_ints, p->pfd_frame_quads);
  Dir D = make_dir(p, values, list_n, n_lists, delta, out_off, ws, total_ints);
  uint64_t* sums = (uint64_t*)((uint8_t*)ws + L.sums);
  // list offsets and first frames
  if (scan_u64(GetListN{list_n}, n_lists, out_off, sums, st) != cudaSuccess) return GC_ERR_CUDA;
  if (scan_u64(GetFrames{list_n, p->pfd_frame_quads}, n_lists, D.frame_off, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  uint64_t nf = 0, tot = 0;
  if (cudaMemcpyAsync(&nf, D.frame_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&tot, out_off + n_lists, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  if (tot != total_ints) return GC_ERR_INVALID_ARGUMENT;
  D.n_frames = nf;
  if (nf) {
    const uint64_t blocks = (nf + kWarpsPerBlock - 1) / kWarpsPerBlock;
    k_fr_plan<<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(D);
  }
  if (scan_u64(GetRec{D.rec, 1}, nf, D.vec_off, sums, st) != cudaSuccess ||
      scan_u64(GetRec{D.rec, 2}, nf, D.exb_off, sums, st) != cudaSuccess)
    return GC_ERR_CUDA;
  k_fr_dir<<<(unsigned)((n_lists + 1 + 255) / 256), 256, 0, st>>>(D, ctrl_off, data_off, exc_off);
  uint64_t vt = 0, et = 0;
  if (cudaMemcpyAsync(&vt, D.vec_off + nf, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&et, D.exb_off + nf, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return GC_ERR_CUDA;
  sizes[0] = 16 * ((4 * nf + 15) / 16);  // ctrl bytes
  sizes[1] = vt;                         // data vectors
  sizes[2] = 16 * ((et + 15) / 16);      // exception bytes
  sizes[3] = nf;                         // frames (for gc_encode_device_write)
  return GC_OK;
}

gc_status gc_encode_device_write(const gc_encode_params* p, const uint32_t* values,
                                 const uint32_t* list_n, uint64_t n_lists, uint64_t total_ints,
                                 int delta, const uint64_t* out_off, const uint64_t* sizes,
                                 uint8_t* ctrl, void* data, uint8_t* exc, void* ws,
                                 uint64_t ws_bytes, void* stream) {
  uint64_t need = 0;
  const gc_status s0 = gc_encode_device_ws_size(p, n_lists, total_ints, &need);
  if (s0 != GC_OK) return s0;
  if (!ws || ws_bytes < need) return GC_ERR_WORKSPACE_TOO_SMALL;
  if (!sizes || (sizes[0] && !ctrl) || (sizes[1] && !data) || (sizes[2] && !exc) ||
      ((uintptr_t)data & 15) || ((uintptr_t)ctrl & 3))
    return GC_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  // padding bytes of the control / exception streams are zero; the OR-packed ones start at 0
  if ((sizes[0] && cudaMemsetAsync(ctrl, 0, sizes[0], st) != cudaSuccess) ||
      (sizes[2] && cudaMemsetAsync(exc, 0, sizes[2], st) != cudaSuccess))
    return GC_ERR_CUDA;
  if (is_gsc(p)) {
    const GscWs L = gsc_ws_layout(n_lists, total_ints);
    Gsc G = make_gsc(p, values, list_n, n_lists, delta, const_cast<uint64_t*>(out_off), ws, total_ints);
    G.n_quads = sizes[3];
    if (sizes[1] && cudaMemsetAsync(data, 0, 16 * sizes[1], st) != cudaSuccess) return GC_ERR_CUDA;
    if (G.n_quads)
      k_gsc_write<<<(unsigned)((G.n_quads + 255) / 256), 256, 0, st>>>(
          G, (const uint64_t*)((uint8_t*)ws + L.c_off), (const uint64_t*)((uint8_t*)ws + L.d_off),
          ctrl, (uint32_t*)data);
    return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
  }
  if (is_vb(p)) {
    const VbWs L = vb_ws_layout(n_lists, total_ints);
    Vb V = make_vb(values, list_n, n_lists, total_ints, delta, const_cast<uint64_t*>(out_off), ws);
    if (total_ints)
      k_vb_write<<<(unsigned)((total_ints + 255) / 256), 256, 0, st>>>(
          V, (const uint64_t*)((uint8_t*)ws + L.cb), ctrl);
    return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
  }
  if (is_gs(p)) {
    const GsWs L = gs_ws_layout(n_lists, total_ints);
    GsEnc E = make_gs(values, list_n, n_lists, delta, const_cast<uint64_t*>(out_off), ws, total_ints);
    E.n_quads = sizes[3];
    uint8_t* w = (uint8_t*)ws;
    if (E.n_quads)
      k_gs_write<<<(unsigned)((E.n_quads + 255) / 256), 256, 0, st>>>(
          E, w + L.sel, w + L.cov, (const uint32_t*)(w + L.idx), ctrl, (uint4*)data);
    return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
  }
  if (is_afor(p)) {
    const AforWs L = afor_ws_layout(n_lists, total_ints);
    Afor A = make_afor(values, list_n, n_lists, delta, const_cast<uint64_t*>(out_off), ws, total_ints);
    A.n_blocks = sizes[3];
    if (A.n_blocks) {
      const uint64_t blocks = (A.n_blocks + kWarpsPerBlock - 1) / kWarpsPerBlock;
      k_afor_write<<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(
          A, (const uint64_t*)((uint8_t*)ws + L.nf), (const uint64_t*)((uint8_t*)ws + L.nv), ctrl,
          (uint4*)data);
    }
    return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
  }
  Dir D = make_dir(p, values, list_n, n_lists, delta, const_cast<uint64_t*>(out_off), ws, total_ints);
  D.n_frames = sizes[3];
  if (D.n_frames) {
    const uint64_t blocks = (D.n_frames + kWarpsPerBlock - 1) / kWarpsPerBlock;
    k_fr_write<<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(D, ctrl, (uint4*)data, exc);
  }
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

}  // extern "C"
