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

}  // namespace gce

using namespace gce;

namespace {
bool valid_gpu_params(const gc_encode_params* p) {
  return p && p->codec == GC_GROUP_PFD && (p->pfd_frame_quads == 32 || p->pfd_frame_quads == 128) &&
         p->variant <= 1 && (p->variant == 1 || p->zeta_den > 0);
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
  if (!valid_gpu_params(p) || !bytes) return p && p->codec != GC_GROUP_PFD ? GC_ERR_UNKNOWN_CODEC
                                                                           : GC_ERR_INVALID_ARGUMENT;
  *bytes = ws_layout(n_lists, total_ints, p->pfd_frame_quads).bytes;
  return GC_OK;
}

gc_status gc_encode_device_plan(const gc_encode_params* p, const uint32_t* values,
                                const uint32_t* list_n, uint64_t n_lists, uint64_t total_ints,
                                int delta, uint64_t* ctrl_off, uint64_t* data_off,
                                uint64_t* exc_off, uint64_t* out_off, void* ws, uint64_t ws_bytes,
                                uint64_t* sizes, void* stream) {
  if (!valid_gpu_params(p)) return p && p->codec != GC_GROUP_PFD ? GC_ERR_UNKNOWN_CODEC : GC_ERR_BAD_VARIANT;
  if (!ws || !sizes || !ctrl_off || !data_off || !exc_off || !out_off ||
      (n_lists && !list_n) || (total_ints && !values))
    return GC_ERR_INVALID_ARGUMENT;
  const WsLayout L = ws_layout(n_lists, total_ints, p->pfd_frame_quads);
  if (ws_bytes < L.bytes) return GC_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = (cudaStream_t)stream;
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
  if (!valid_gpu_params(p)) return p && p->codec != GC_GROUP_PFD ? GC_ERR_UNKNOWN_CODEC : GC_ERR_BAD_VARIANT;
  const WsLayout L = ws_layout(n_lists, total_ints, p->pfd_frame_quads);
  if (!ws || ws_bytes < L.bytes) return GC_ERR_WORKSPACE_TOO_SMALL;
  if (!sizes || (sizes[0] && !ctrl) || (sizes[1] && !data) || (sizes[2] && !exc) ||
      ((uintptr_t)data & 15) || ((uintptr_t)ctrl & 3))
    return GC_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  Dir D = make_dir(p, values, list_n, n_lists, delta, const_cast<uint64_t*>(out_off), ws, total_ints);
  D.n_frames = sizes[3];
  // padding bytes of the control / exception streams are zero
  if ((sizes[0] && cudaMemsetAsync(ctrl, 0, sizes[0], st) != cudaSuccess) ||
      (sizes[2] && cudaMemsetAsync(exc, 0, sizes[2], st) != cudaSuccess))
    return GC_ERR_CUDA;
  if (D.n_frames) {
    const uint64_t blocks = (D.n_frames + kWarpsPerBlock - 1) / kWarpsPerBlock;
    k_fr_write<<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(D, ctrl, (uint4*)data, exc);
  }
  return cudaGetLastError() == cudaSuccess ? GC_OK : GC_ERR_CUDA;
}

}  // extern "C"
