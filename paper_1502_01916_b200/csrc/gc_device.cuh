// gc_device.cuh -- shared sm_100a device helpers: tile geometry, PTX wrappers
// (bulk async copies, mbarriers, relaxed/acquire global accesses), block scans
// and the decoupled look-back used by the two decode kernels.
#pragma once
#include <cstdint>

#include "gc.h"

namespace gcd {

#ifndef GC_ITHREADS
#define GC_ITHREADS 256
#endif
#ifndef GC_WA
#define GC_WA 2048
#endif
constexpr int kThreads = GC_ITHREADS;  // index / list kernels
constexpr int kWarps = kThreads / 32;

// Index kernel (control-space tiles): 2048 control words, 8 per thread; batches of fewer
// than kSmallIndexWords words use 256-word tiles (1 per thread), so a small batch still
// spreads its control scan over many CTAs (latency, not throughput, bounds it).
constexpr uint32_t kWA = GC_WA;
constexpr uint32_t kCA = kWA / kThreads;
static_assert(kCA == 8, "the index kernel parses 8 control words per thread");
constexpr uint32_t kWASmall = kThreads;
#ifndef GC_SMALL_INDEX_WORDS
#define GC_SMALL_INDEX_WORDS (1u << 18)
#endif
constexpr uint64_t kSmallIndexWords = GC_SMALL_INDEX_WORDS;

// Decode kernel (output-space tiles): tile t owns the output ints
// [t*kT, (t+1)*kT) exactly; it decodes every quadruple that holds one of them.
// One CTA of kThreads threads decodes a tile; CTAs are persistent.
#ifndef GC_T_INTS
#define GC_T_INTS 8192
#endif
#ifndef GC_DT
#define GC_DT 256
#endif
constexpr uint32_t kT = GC_T_INTS;               // output ints per tile
constexpr uint32_t kDT = GC_DT;                  // decode threads per CTA (kT / 32)
constexpr uint32_t kDW = kDT / 32;               // decode warps per CTA
static_assert(kT == 32 * kDT, "the d-gap pass scans 32 ints per thread");
constexpr uint32_t kQPT = 9;                     // quads per thread per unpack round
constexpr uint32_t kR = kQPT * kThreads;         // quad ordinals per unpack round (2304)
#ifndef GC_LC
#define GC_LC 128
#endif
#ifndef GC_CCAP
#define GC_CCAP 1536
#endif
#ifndef GC_DCAP
#define GC_DCAP 1600
#endif
constexpr uint32_t kLC = GC_LC;                  // lists per list round (list table)
#ifndef GC_UPT
#define GC_UPT 4
#endif
constexpr uint32_t kUPT = GC_UPT;                // parse units per thread per parse chunk
constexpr uint32_t kOutW = kT + 8;               // staging ints: index = tile position + 4
constexpr uint32_t kCCap = GC_CCAP;              // staged control words
constexpr uint32_t kDCap = GC_DCAP;              // staged data vectors (25 KiB)
constexpr uint32_t kECap = 4096;                 // staged exception bytes

// Look-back flags.
constexpr uint32_t kFlagAgg = 1, kFlagIncl = 2;

// Tile-start descriptor written by the index kernel (one per decode tile, 64 B): the
// quadruple holding output int t*kT and the control word whose groups include it.
struct Entry {
  uint32_t l;           // list of the quad containing output position t*kT
  uint32_t k;           // its quad index within the list
  uint32_t wq;          // raw quads of the list before control word w
  uint32_t valid;       // 1 once written
  uint64_t w;           // global control word whose groups include quad k
  uint64_t wd;          // absolute data lane-bit at the start of w
  uint64_t we;          // absolute exception byte at the start of w
  uint64_t wd_end;      // ... at the end of w (bounds the previous tile's data)
  uint64_t we_end;
  uint64_t pad;
};
static_assert(sizeof(Entry) == 64, "Entry is 16 words");

// Index-kernel look-back slot of a control tile: the aggregate and the inclusive prefix,
// each written once as two self-flagged 64-bit words (a reader needs no fence: it accepts
// a slot when both words carry their flag).  Packing: w0 = 1<<63 | q<<31 | d[30:0],
// w1 = 1<<63 | d[46:31]<<47 | e[46:0]  (q quads mod 2^32; d lane-bits < 2^47 and e bytes
// < 2^47: the launch checks data_vectors < 2^42 and exc_bytes < 2^47).
struct TileA {
  uint64_t a0, a1;  // aggregate
  uint64_t i0, i1;  // inclusive prefix
};
__device__ __forceinline__ void tilea_pack(uint32_t q, uint64_t d, uint64_t e, uint64_t& w0,
                                           uint64_t& w1) {
  w0 = (1ull << 63) | ((uint64_t)q << 31) | (d & 0x7FFFFFFFull);
  w1 = (1ull << 63) | (((d >> 31) & 0xFFFFull) << 47) | (e & ((1ull << 47) - 1));
}
__device__ __forceinline__ void tilea_unpack(uint64_t w0, uint64_t w1, uint32_t& q, uint64_t& d,
                                             uint64_t& e) {
  q = (uint32_t)(w0 >> 31);
  d = (w0 & 0x7FFFFFFFull) | (((w1 >> 47) & 0xFFFFull) << 31);
  e = w1 & ((1ull << 47) - 1);
}

struct WsHeader {
  uint32_t status;
  uint32_t counter_a;
  uint32_t counter_b;
  uint32_t vb_long;  // Variable Byte: k_varbyte_short saw a list of >= kVbShort ints
  uint32_t pad[12];
  unsigned long long prof[24];  // GC_TIMING builds: cycles per decode phase (debugging aid)
};

__host__ __device__ __forceinline__ uint64_t mn64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t mx64(uint64_t a, uint64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t smin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t smax64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ uint32_t mn32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- checked builds
// -DGC_CHECKED (the stand-in for compute-sanitizer, which this pool does not run): every
// shared- and global-memory index of the decode kernels is asserted against the extent of
// the buffer it addresses; a failed check prints the kernel line and traps, so the test
// that ran it fails.  Product builds compile the checks out.
#ifdef GC_CHECKED
#define GC_CHECK(cond)                                                                    \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("GC_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                          \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define GC_CHECK(cond) \
  do {                 \
  } while (0)
#endif

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

// Tensor bulk async store shared -> global (TMA engine, SASS UTMASTG): one box of the 2-D
// tensor map tm at coordinates (c0 inner, c1 outer), tracked by the issuing thread's bulk
// groups.  The source's writers fence (fence.proxy.async.shared::cta) before the barrier
// that precedes the issue; the issuer waits for the reads (wait_group.read) before the
// buffer is written again.
__device__ __forceinline__ void tma_store_2d(const void* tm, const void* src_smem, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tm),
               "r"(smem_addr(src_smem)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ uint4 ldg_nc_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------- scans
// Segmented value: f = "a segment (list) starts inside"; (q, d, e) = sums since the
// last segment start (raw quads, data lane-bits, exception bytes; tile-relative u32).
// a (+) b = b.f ? b : (a.f, a + b).
struct Seg4 {
  uint32_t f, q, d, e;
};
__device__ __forceinline__ Seg4 seg4_op(const Seg4& a, const Seg4& b) {
  return b.f ? b : Seg4{a.f, a.q + b.q, a.d + b.d, a.e + b.e};
}

// Block-wide scans.  Each warp scans with shuffles; the NW warp totals are then
// scanned by every warp at once (lane w holds warp w's total), so no thread loops over
// the warps.  scratch: NW entries; two barriers (the second frees scratch).
__device__ __forceinline__ Seg4 shfl_seg4(const Seg4& v, int src) {
  return Seg4{__shfl_sync(0xffffffffu, v.f, src), __shfl_sync(0xffffffffu, v.q, src),
              __shfl_sync(0xffffffffu, v.d, src), __shfl_sync(0xffffffffu, v.e, src)};
}
template <bool kExc>
__device__ __forceinline__ Seg4 warp_incl_seg4(Seg4 inc, uint32_t lane, uint32_t width) {
  for (uint32_t o = 1; o < width; o <<= 1) {
    Seg4 n;
    n.f = __shfl_up_sync(0xffffffffu, inc.f, o);
    n.q = __shfl_up_sync(0xffffffffu, inc.q, o);
    n.d = __shfl_up_sync(0xffffffffu, inc.d, o);
    n.e = kExc ? __shfl_up_sync(0xffffffffu, inc.e, o) : 0u;
    if (lane >= o) inc = seg4_op(n, inc);
  }
  return inc;
}
// Without exceptions the flag rides in bit 31 of q (a segment's raw quads stay < 2^31):
// (f<<31 | q, d), two shuffles per step instead of three, and b (+) ... keeps b's word
// when its flag is set, else adds (b has no flag bit, so a's flag survives the add).
#ifndef GC_SEG_PACK
#define GC_SEG_PACK 1
#endif
__device__ __forceinline__ uint2 warp_incl_seg2(uint2 inc, uint32_t lane, uint32_t width) {
#pragma unroll
  for (uint32_t o = 1; o < 32; o <<= 1) {
    if (o >= width) break;
    const uint32_t nx = __shfl_up_sync(0xffffffffu, inc.x, o);
    const uint32_t ny = __shfl_up_sync(0xffffffffu, inc.y, o);
    if (lane >= o && !(inc.x >> 31)) {
      inc.x += nx;
      inc.y += ny;
    }
  }
  return inc;
}

// Exclusive segmented scan; returns this thread's prefix, *total = the block aggregate.
template <bool kExc, uint32_t NW = kWarps>
__device__ __forceinline__ Seg4 block_excl_seg4(Seg4 v, Seg4* scratch, Seg4* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (!kExc && GC_SEG_PACK) {
    uint2* scr = reinterpret_cast<uint2*>(scratch);
    const uint2 inc = warp_incl_seg2(make_uint2(v.q | (v.f ? 0x80000000u : 0u), v.d), lane, 32);
    if (lane == 31) scr[warp] = inc;
    uint2 ex = make_uint2(__shfl_up_sync(0xffffffffu, inc.x, 1), __shfl_up_sync(0xffffffffu, inc.y, 1));
    if (lane == 0) ex = make_uint2(0u, 0u);
    __syncthreads();
    uint2 w = lane < NW ? scr[lane] : make_uint2(0u, 0u);
    w = warp_incl_seg2(w, lane, NW);
    const uint32_t src = warp ? warp - 1 : 0;
    uint2 wpre = make_uint2(__shfl_sync(0xffffffffu, w.x, src), __shfl_sync(0xffffffffu, w.y, src));
    if (warp == 0) wpre = make_uint2(0u, 0u);
    const uint32_t tx = __shfl_sync(0xffffffffu, w.x, NW - 1), ty = __shfl_sync(0xffffffffu, w.y, NW - 1);
    *total = Seg4{tx >> 31, tx & 0x7FFFFFFFu, ty, 0u};
    __syncthreads();
    const uint2 r = (ex.x >> 31) ? ex : make_uint2(wpre.x + ex.x, wpre.y + ex.y);
    return Seg4{r.x >> 31, r.x & 0x7FFFFFFFu, r.y, 0u};
  }
  const Seg4 inc = warp_incl_seg4<kExc>(v, lane, 32);
  if (lane == 31) scratch[warp] = inc;
  Seg4 ex;
  ex.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
  ex.q = __shfl_up_sync(0xffffffffu, inc.q, 1);
  ex.d = __shfl_up_sync(0xffffffffu, inc.d, 1);
  ex.e = kExc ? __shfl_up_sync(0xffffffffu, inc.e, 1) : 0u;
  if (lane == 0) ex = Seg4{0, 0, 0, 0};
  __syncthreads();
  Seg4 w = lane < NW ? scratch[lane] : Seg4{0, 0, 0, 0};
  w = warp_incl_seg4<kExc>(w, lane, NW);
  Seg4 wpre = shfl_seg4(w, warp ? warp - 1 : 0);
  if (warp == 0) wpre = Seg4{0, 0, 0, 0};
  *total = shfl_seg4(w, NW - 1);
  __syncthreads();
  return seg4_op(wpre, ex);
}

// Block-wide exclusive sum of u32.
template <uint32_t NW = kWarps>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* scratch,
                                                   uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  uint32_t w = lane < NW ? scratch[lane] : 0u;
#pragma unroll
  for (uint32_t o = 1; o < NW; o <<= 1) {
    uint32_t n = __shfl_up_sync(0xffffffffu, w, o);
    if (lane >= o) w += n;
  }
  const uint32_t wpre = warp ? __shfl_sync(0xffffffffu, w, warp - 1) : 0u;
  *total = __shfl_sync(0xffffffffu, w, NW - 1);
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
template <uint32_t NW = kWarps>
__device__ __forceinline__ Seg1 block_excl_seg1(Seg1 x, Seg1* scratch, Seg1* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Seg1 inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg1 n;
    n.f = __shfl_up_sync(0xffffffffu, inc.f, o);
    n.v = __shfl_up_sync(0xffffffffu, inc.v, o);
    if (lane >= o) inc = seg1_op(n, inc);
  }
  if (lane == 31) scratch[warp] = inc;
  Seg1 ex;
  ex.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
  ex.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
  if (lane == 0) ex = Seg1{0, 0};
  __syncthreads();
  Seg1 w = lane < NW ? scratch[lane] : Seg1{0, 0};
#pragma unroll
  for (uint32_t o = 1; o < NW; o <<= 1) {
    Seg1 n;
    n.f = __shfl_up_sync(0xffffffffu, w.f, o);
    n.v = __shfl_up_sync(0xffffffffu, w.v, o);
    if (lane >= o) w = seg1_op(n, w);
  }
  Seg1 wpre{__shfl_sync(0xffffffffu, w.f, warp ? warp - 1 : 0),
            __shfl_sync(0xffffffffu, w.v, warp ? warp - 1 : 0)};
  if (warp == 0) wpre = Seg1{0, 0};
  *total = Seg1{__shfl_sync(0xffffffffu, w.f, NW - 1), __shfl_sync(0xffffffffu, w.v, NW - 1)};
  __syncthreads();
  return seg1_op(wpre, ex);
}

// ---------------------------------------------------------------- decoupled look-back
// d-gap carry: one 64-bit word per tile, (flag << 32) | value.  Called by one full
// warp; returns the sum of the aggregates of the tiles before `tile` back to (and
// including) the nearest tile that published an inclusive prefix.  Lane i watches tile
// base-i; a window is usable as soon as every lane up to the nearest inclusive one has
// published (the older tiles of the window are not waited for).
__device__ __forceinline__ uint32_t lookback_u32(uint64_t* status, uint32_t tile,
                                                 unsigned long long* prof = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
#ifdef GC_TIMING
  if (prof && lane == 0) atomicAdd(prof + 0, 1ull);
  const long long t_enter = clock64();
#else
  (void)prof;
#endif
  uint32_t acc = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    uint64_t s = (uint64_t)kFlagIncl << 32;  // before tile 0: an empty inclusive prefix
    if (idx >= 0) s = ld_relaxed_u64(status + idx);
#ifdef GC_TIMING
    if (prof && lane == 0) atomicAdd(prof + 1, 1ull);
#endif
    while (true) {
      const uint32_t flag = (uint32_t)(s >> 32);
      const uint32_t valid = __ballot_sync(0xffffffffu, flag != 0);
      const uint32_t incl = __ballot_sync(0xffffffffu, flag == kFlagIncl);
      const uint32_t first = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;
      const uint32_t need = first == 31u ? 0xffffffffu : ((2u << first) - 1u);
      if ((valid & need) == need) break;
#ifdef GC_TIMING
      if (prof) {
        const uint32_t bad = need & ~valid;
        if (lane == 0) {
          atomicAdd(prof + 2, 1ull);
          const int64_t dist = (int64_t)tile - (base - (int64_t)(__ffs(bad) - 1));
          const int b = dist <= 1 ? 3 : dist <= 4 ? 4 : dist <= 16 ? 5 : dist <= 128 ? 6 : 7;
          atomicAdd(prof + b, 1ull);
        }
      }
#endif
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
    if (incl) {
#ifdef GC_TIMING
      if (prof && lane == 0) atomicAdd(prof + 8, (unsigned long long)(clock64() - t_enter));
#endif
      return acc;
    }
    base -= 32;
  }
}

// Decoupled look-back over TileA slots (the index kernel's control tiles, the Variable Byte
// byte tiles); one full warp.  Returns in (pq, pd, pe) the sums of the tiles before `tile`
// back to (and including) the nearest one that published an inclusive prefix.  A slot is
// published when both of its words carry bit 63 (tilea_pack).
__device__ __forceinline__ void lookback_tilea(const TileA* tiles, uint32_t tile, uint32_t& pq,
                                               uint64_t& pd, uint64_t& pe) {
  const uint32_t lane = threadIdx.x & 31;
  pq = 0;
  pd = pe = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    const TileA* t = tiles + (idx >= 0 ? idx : 0);
    uint64_t i0 = 1ull << 63, i1 = 1ull << 63, a0 = 0, a1 = 0;  // before tile 0: zero
    if (idx >= 0) {
      i0 = ld_relaxed_u64(&t->i0);
      i1 = ld_relaxed_u64(&t->i1);
      a0 = ld_relaxed_u64(&t->a0);
      a1 = ld_relaxed_u64(&t->a1);
    }
    uint32_t inclm, first;
    while (true) {
      const bool hi = (i0 >> 63) && (i1 >> 63), ha = (a0 >> 63) && (a1 >> 63);
      const uint32_t valid = __ballot_sync(0xffffffffu, hi || ha);
      inclm = __ballot_sync(0xffffffffu, hi);
      first = inclm ? (uint32_t)(__ffs(inclm) - 1) : 31u;
      const uint32_t need = first == 31u ? 0xffffffffu : ((2u << first) - 1u);
      if ((valid & need) == need) break;
      if (!(valid & (1u << lane)) && (need & (1u << lane))) {
        __nanosleep(32);
        i0 = ld_relaxed_u64(&t->i0);
        i1 = ld_relaxed_u64(&t->i1);
        a0 = ld_relaxed_u64(&t->a0);
        a1 = ld_relaxed_u64(&t->a1);
      }
    }
    const bool hi = (i0 >> 63) && (i1 >> 63);
    uint32_t q = 0;
    uint64_t d = 0, e = 0;
    if (lane <= first) tilea_unpack(hi ? i0 : a0, hi ? i1 : a1, q, d, e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      q += __shfl_xor_sync(0xffffffffu, q, o);
      d += __shfl_xor_sync(0xffffffffu, d, o);
      e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    pq += q;
    pd += d;
    pe += e;
    if (inclm) return;
    base -= 32;
  }
}

// Largest l in [lo, hi) with off[l] <= key (off non-decreasing, off[lo] <= key); one full
// warp, 32 probes per step.
__device__ __forceinline__ uint64_t warp_find(const uint64_t* off, uint64_t lo, uint64_t hi,
                                              uint64_t key) {
  const uint32_t lane = threadIdx.x & 31;
  while (hi - lo > 1) {
    const uint64_t span = hi - lo;
    const uint64_t p = lo + ((span * (lane + 1)) >> 5);  // non-decreasing in lane; lane 31: hi
    const bool le = p < hi && off[p] <= key;
    const uint32_t m = __ballot_sync(0xffffffffu, le);  // a prefix of the lanes
    const uint64_t nlo = m ? __shfl_sync(0xffffffffu, p, 31 - __clz(m)) : lo;
    const uint32_t nm = ~m;
    hi = __shfl_sync(0xffffffffu, p, __ffs(nm) - 1);
    lo = nlo;
  }
  return lo;
}

__device__ __forceinline__ uint32_t mask_bits(uint32_t b) {
  return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u);
}

}  // namespace gcd
