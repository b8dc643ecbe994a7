// gc_device.cuh -- shared sm_100a device helpers: tile geometry, PTX wrappers
// (bulk async copies, mbarriers, relaxed/acquire global accesses), block scans
// and the decoupled look-back used by the two decode kernels.
#pragma once
#include <cstdint>

#include "gc.h"

namespace gcd {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Index kernel (control-space tiles): 2048 control words, 8 per thread.
constexpr uint32_t kWA = 2048;
constexpr uint32_t kCA = kWA / kThreads;

// Decode kernel (output-space warp-tiles): warp-tile t owns the quadruples that contain
// the output positions [t*kT, (t+1)*kT).  One warp decodes one tile at a
// time with warp-shuffle scans only; warps are persistent.
constexpr uint32_t kT = 1024;
constexpr uint32_t kCBW = 4;                     // control words per lane per parse round
constexpr uint32_t kRoundWords = kCBW * 32;      // 128
constexpr uint32_t kQPL = 9;                     // quads per lane per unpack window
constexpr uint32_t kRQ = kQPL * 32;              // quads per unpack window (288)
constexpr uint32_t kLT = 32;                     // lists per list round (per-warp list table)
constexpr uint32_t kOutWords = kT + 8;           // staging window [t*kT-4, t*kT+kT+4)
constexpr uint32_t kOutChunks = 264;             // 16-B chunks incl. swizzle slack
constexpr uint32_t kCCap = 272;                  // staged control words (incl. halo)
constexpr uint32_t kDCap = 288;                  // staged data vectors (4.5 KiB)
constexpr uint32_t kECap = 768;                  // staged exception bytes

// Look-back flags.
constexpr uint32_t kFlagAgg = 1, kFlagIncl = 2;

struct Entry {          // tile boundary descriptor written by the index kernel (80 B)
  uint32_t l;           // list of the quad containing output position t*kT
  uint32_t j;           // its quad index within the list
  uint32_t wq;          // raw quads of the list owned by control words before gword
  uint32_t valid;
  uint64_t gword;       // global control word owning the group of quad j
  uint64_t wd;          // global data lane-bit position at the start of gword
  uint64_t we;          // global exception byte at the start of gword
  uint64_t dbeg;        // data lane-bit where the group of quad j starts
  uint64_t ebeg;        // exception byte where the group of quad j starts
  uint64_t cend;        // control words needed by the quads before (l, j): [.., cend)
  uint64_t dend;        // data lane-bits needed by the quads before (l, j): [.., dend)
  uint64_t eend;        // exception bytes needed by the quads before (l, j)
};

struct TileA {          // index-kernel look-back slot: aggregate and inclusive prefix
  uint32_t flag;        // kept in separate fields so a reader that saw flag X reads X's
  uint32_t aq;          // values, which were complete before X was published
  uint64_t ad, ae;
  uint32_t iq, pad;
  uint64_t id, ie;
};

struct WsHeader {
  uint32_t status;
  uint32_t counter_a;
  uint32_t counter_b;
  uint32_t pad[61];
};

__host__ __device__ __forceinline__ uint64_t mn64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t mx64(uint64_t a, uint64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t smin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t smax64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ uint32_t mn32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- memory helpers
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// mbarrier + 1-D bulk async copy (TMA engine, SASS UBLKCP) global -> shared.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ uint4 ldg_nc_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------- scans
// Segmented value: f = "a segment (list) starts inside"; (q, d, e) = sums since the
// last segment start.  a (+) b = b.f ? b : (a.f, a + b).
struct Seg3 {
  uint32_t f, q;
  uint64_t d, e;
};
__device__ __forceinline__ Seg3 seg3_op(const Seg3& a, const Seg3& b) {
  if (b.f) return b;
  Seg3 r;
  r.f = a.f;
  r.q = a.q + b.q;
  r.d = a.d + b.d;
  r.e = a.e + b.e;
  return r;
}
__device__ __forceinline__ Seg3 shfl_up(const Seg3& v, int delta) {
  Seg3 r;
  r.f = __shfl_up_sync(0xffffffffu, v.f, delta);
  r.q = __shfl_up_sync(0xffffffffu, v.q, delta);
  r.d = __shfl_up_sync(0xffffffffu, v.d, delta);
  r.e = __shfl_up_sync(0xffffffffu, v.e, delta);
  return r;
}

// Block-wide exclusive segmented scan; returns the exclusive prefix of this thread
// and (in *total) the block aggregate.  scratch: kWarps entries of shared memory.
__device__ __forceinline__ Seg3 block_excl_seg3(Seg3 v, Seg3* scratch, Seg3* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Seg3 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg3 n = shfl_up(inc, o);
    if (lane >= o) inc = seg3_op(n, inc);
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  Seg3 wpre = Seg3{0, 0, 0, 0};
  Seg3 tot = Seg3{0, 0, 0, 0};
#pragma unroll
  for (int w = 0; w < kWarps; w++) {
    if (w < warp) wpre = seg3_op(wpre, scratch[w]);
    tot = seg3_op(tot, scratch[w]);
  }
  Seg3 ex = shfl_up(inc, 1);
  if (lane == 0) ex = Seg3{0, 0, 0, 0};
  *total = tot;
  __syncthreads();
  return seg3_op(wpre, ex);
}

// Block-wide exclusive sum of u32.
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* scratch,
                                                   uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kWarps; w++) {
    uint32_t s = scratch[w];
    if (w < warp) wpre += s;
    tot += s;
  }
  *total = tot;
  __syncthreads();
  return wpre + inc - v;
}

// Segmented u32 (mod 2^32) value for the d-gap scan.
struct Seg1 {
  uint32_t f, v;
};
__device__ __forceinline__ Seg1 seg1_op(Seg1 a, Seg1 b) {
  return b.f ? b : Seg1{a.f, a.v + b.v};
}
__device__ __forceinline__ Seg1 block_excl_seg1(Seg1 x, Seg1* scratch, Seg1* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Seg1 inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg1 n;
    n.f = __shfl_up_sync(0xffffffffu, inc.f, o);
    n.v = __shfl_up_sync(0xffffffffu, inc.v, o);
    if (lane >= o) inc = seg1_op(n, inc);
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  Seg1 wpre{0, 0}, tot{0, 0};
#pragma unroll
  for (int w = 0; w < kWarps; w++) {
    Seg1 s = scratch[w];
    if (w < warp) wpre = seg1_op(wpre, s);
    tot = seg1_op(tot, s);
  }
  Seg1 ex;
  ex.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
  ex.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
  if (lane == 0) ex = Seg1{0, 0};
  *total = tot;
  __syncthreads();
  return seg1_op(wpre, ex);
}

// ---------------------------------------------------------------- decoupled look-back
// d-gap carry: one 64-bit word per tile, (flag << 32) | value.  Called by one full
// warp; returns the sum of the aggregates of the tiles before `tile` back to (and
// including) the nearest tile that published an inclusive prefix.  Lane i watches tile
// base-i; a window is usable as soon as every lane up to the nearest inclusive one has
// published (the older tiles of the window are not waited for).
__device__ __forceinline__ uint32_t lookback_u32(uint64_t* status, uint32_t tile) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t acc = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    uint64_t s = (uint64_t)kFlagIncl << 32;  // before tile 0: an empty inclusive prefix
    if (idx >= 0) s = ld_relaxed_u64(status + idx);
    while (true) {
      const uint32_t flag = (uint32_t)(s >> 32);
      const uint32_t valid = __ballot_sync(0xffffffffu, flag != 0);
      const uint32_t incl = __ballot_sync(0xffffffffu, flag == kFlagIncl);
      const uint32_t first = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;
      const uint32_t need = first == 31u ? 0xffffffffu : ((2u << first) - 1u);
      if ((valid & need) == need) break;
      if (!(valid & (1u << lane)) && (need & (1u << lane))) {
        __nanosleep(32);
        s = ld_relaxed_u64(status + idx);
      }
    }
    const uint32_t flag = (uint32_t)(s >> 32);
    const uint32_t incl = __ballot_sync(0xffffffffu, flag == kFlagIncl);
    uint32_t mine = (uint32_t)s;
    if (incl) {
      const uint32_t first = (uint32_t)(__ffs(incl) - 1);  // nearest inclusive predecessor
      if (lane > first) mine = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    acc += mine;
    if (incl) return acc;
    base -= 32;
  }
}

// Staging window swizzle: 16-B chunk c is stored at chunk c ^ ((c >> 3) & 7), which
// keeps both the blocked (16 consecutive ints per thread) and the striped (one chunk
// per thread) 128-bit accesses free of bank conflicts.
__device__ __forceinline__ uint32_t sw_chunk(uint32_t c) { return c ^ ((c >> 3) & 7u); }
__device__ __forceinline__ uint32_t sw_word(uint32_t x) {
  return (sw_chunk(x >> 2) << 2) | (x & 3u);
}

__device__ __forceinline__ uint32_t mask_bits(uint32_t b) {
  return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u);
}

}  // namespace gcd
