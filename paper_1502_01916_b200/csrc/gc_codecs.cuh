// gc_codecs.cuh -- per-codec parsers of one 32-bit control word (sm_100a device code).
//
// Every list's control area starts 4-byte aligned, so a 32-bit
// control word belongs to exactly one list.  For each codec a word is parsed on
// its own (plus, for complete unary, the previous word of the same list) into the
// "groups" whose control it owns, in stream order.  A group is the unit one
// control pattern describes (§3.1: a pattern that described N ints now
// describes N quadruples):
//   Group-Simple  one 4-bit selector  -> NUM quads in one 128-bit vector (Table III)
//   Group-Scheme  one length descriptor -> one quad at BW bits (Eq. (2))
//   Group-AFOR    one header byte      -> a frame of 8/16/32 quads at one bw
//   Group-PFD     one 4-byte header    -> a frame of F quads at b bits + exceptions
// Quad counts are "raw" (not clamped to the list end); the caller clamps with the
// list's quad count Q, which is how padding groups are ignored.
#pragma once
#include <cstdint>
#include <type_traits>
#include <utility>

#include "gc_device.cuh"

#ifndef GC_AFOR_SUB
#define GC_AFOR_SUB 1  // Group-AFOR parse units per frame header (4: 8-quad parts, measured 6% slower)
#endif
#ifndef GC_AFOR_SPLIT
#define GC_AFOR_SPLIT 1
#endif
#ifndef GC_FRAME_UPT
#define GC_FRAME_UPT 2  // parse units per thread per chunk for the frame codecs (AFOR, PFD)
#endif
#ifndef GC_CU8_PARTS
#define GC_CU8_PARTS 2
#endif
#ifndef GC_IU8_PARTS
#define GC_IU8_PARTS 4
#endif

namespace gcd {

// One group, relative to the word's running prefix (quads, lane bits, exception bytes).
struct Grp {
  uint32_t q0;    // raw quad offset of the group within the word
  uint32_t nq;    // raw quads the group covers
  int32_t d0;     // first data lane-bit of the group, relative to the word's data prefix
  uint32_t dlen;  // lane bits the group occupies
  uint32_t bw;    // bits per value
  uint32_t step;  // lane bits between consecutive quads of the group
  uint32_t e0;    // exception bytes before the group (PFD)
  uint32_t elen;  // exception bytes of the group (PFD)
  uint32_t cnt;   // PFD exception count
  uint32_t wb;    // PFD exception value bytes (1/2/4)
  uint32_t err;   // GC_DEV_* bits, reported only if the group starts before the list end
  uint32_t t0;    // PFD: first quad of the group within its frame
  uint32_t fq;    // PFD: quads of the frame (the list's tail frame may be short)
};

struct WCtx {
  uint32_t w;      // the control word (little-endian load of 4 control bytes)
  uint32_t prev;   // previous control word of the same list (valid iff widx > 0)
  uint64_t widx;   // word index within the list's control area
  uint64_t Q;      // quads of the list
  uint32_t part;   // which kParts-th of the word (codecs with kParts > 1)
};

struct WAgg {
  uint32_t q, d, e;  // raw quads, lane bits, exception bytes owned by the word
};

__device__ __forceinline__ Grp grp0() {
  Grp g;
  g.q0 = 0; g.nq = 0; g.d0 = 0; g.dlen = 0; g.bw = 1; g.step = 0;
  g.e0 = 0; g.elen = 0; g.cnt = 0; g.wb = 0; g.err = 0; g.t0 = 0; g.fq = 0;
  return g;
}

// ---------------------------------------------------------------- Group-Simple
// Table III, 6-bit fields packed into one constant each.
constexpr uint64_t kGsNum = (32ull << 0) | (16ull << 6) | (10ull << 12) | (8ull << 18) |
                            (6ull << 24) | (5ull << 30) | (4ull << 36) | (3ull << 42) |
                            (2ull << 48) | (1ull << 54);
constexpr uint64_t kGsBw = (1ull << 0) | (2ull << 6) | (3ull << 12) | (4ull << 18) |
                           (5ull << 24) | (6ull << 30) | (8ull << 36) | (10ull << 42) |
                           (16ull << 48) | (32ull << 54);

__device__ __forceinline__ uint32_t gs_num(uint32_t s) {
  return s <= 9 ? (uint32_t)(kGsNum >> (6 * s)) & 63u : 1u;
}
__device__ __forceinline__ uint32_t gs_bw(uint32_t s) {
  return s <= 9 ? (uint32_t)(kGsBw >> (6 * s)) & 63u : 32u;
}

struct CodecGS {
  static constexpr bool kExc = false;
  static constexpr uint64_t kBackBits = 0;
  static constexpr int kParts = 2;           // a parse unit = 4 selectors (half a word)
  static constexpr bool kNeedsPrev = false;
  static constexpr bool kMultiQuad = true;   // a group may hold several quads
  static constexpr bool kVectorGroups = true;
  __device__ static WAgg agg(const WCtx& c) {
    uint32_t q = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) q += gs_num((c.w >> (16 * c.part + 4 * k)) & 15u);  // low nibble first (A6)
    return WAgg{q, 4u * 32u, 0u};
  }
  // may the word hold a malformed group?  (a nibble > 9: bit 3 and bit 2 or 1)
  __device__ static bool suspect(const WCtx& c) {
    return ((c.w >> 3) & ((c.w >> 2) | (c.w >> 1)) & 0x11111111u) != 0;
  }
  template <class F>
  __device__ static void walk(const WCtx& c, F&& f) {
    uint32_t q = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t s = (c.w >> (16 * c.part + 4 * k)) & 15u;
      Grp g = grp0();
      g.q0 = q;
      g.nq = gs_num(s);
      g.d0 = 32 * k;       // one 128-bit vector per selector
      g.dlen = 32;
      g.bw = gs_bw(s);
      g.step = g.bw;       // int t of the component at [t*BW, (t+1)*BW) (A7)
      g.err = s > 9 ? GC_DEV_BAD_SELECTOR : 0u;
      f(g);
      q += g.nq;
    }
  }
};

// ---------------------------------------------------------------- Group-Scheme, binary LD
// Field packing (A18): CG=1 three 5-bit fields per 16-bit unit; CG=2 two 4-bit per
// byte; CG=4 two 3-bit per byte; CG=8 four 2-bit per byte; LSB-first.
template <int CG>
struct CodecGscB {
  static constexpr bool kExc = false;
  static constexpr uint64_t kBackBits = 0;
  static constexpr bool kNeedsPrev = false;
  static constexpr bool kMultiQuad = false;
  static constexpr bool kVectorGroups = false;
  static constexpr int kFields = CG == 1 ? 6 : (CG == 8 ? 16 : 8);
  // a word is parsed as kParts units of kFields/kParts fields (balances the work per lane)
  static constexpr int kParts = CG == 8 ? 4 : 2;
  static constexpr int kPF = kFields / kParts;
  __device__ static __forceinline__ uint32_t field(uint32_t w, int k) {
    if (CG == 1) return (w >> (16 * (k / 3) + 5 * (k % 3))) & 31u;
    if (CG == 2) return (w >> (4 * k)) & 15u;
    if (CG == 4) return (w >> (8 * (k / 2) + 3 * (k % 2))) & 7u;
    return (w >> (2 * k)) & 3u;
  }
  // Eq. (2) summed over fields by bit planes: sum of the field values = sum over bits b of
  // 2^b x popc(bit b of every field) (a handful of popcounts instead of a loop over fields)
  static constexpr int kFW = CG == 1 ? 5 : (CG == 2 ? 4 : (CG == 4 ? 3 : 2));  // field bits
  __host__ __device__ static constexpr uint32_t fpos(int k) {
    return CG == 1 ? 16 * (k / 3) + 5 * (k % 3) : (CG == 2 ? 4 * k : (CG == 4 ? 8 * (k / 2) + 3 * (k % 2) : 2 * k));
  }
  __host__ __device__ static constexpr uint32_t plane(int b, int nf) {  // bit b of fields 0 .. nf-1
    uint32_t m = 0;
    for (int k = 0; k < nf; k++) m |= 1u << (fpos(k) + b);
    return m;
  }
  __device__ static __forceinline__ uint32_t field_sum(uint32_t x, int nf) {
    uint32_t t = 0;
#pragma unroll
    for (int b = 0; b < kFW; b++) t += (uint32_t)__popc(x & plane(b, nf)) << b;
    return t;
  }
  __device__ static WAgg agg(const WCtx& c) {
    // part p's fields sit 32/kParts bits above part 0's (every CG)
    const uint32_t x = c.w >> ((32 / kParts) * c.part);
    return WAgg{(uint32_t)kPF, CG * (field_sum(x, kPF) + kPF), 0u};
  }
  __device__ static WAgg word_agg_fast(const WCtx& c) {
    return WAgg{(uint32_t)kFields, CG * (field_sum(c.w, kFields) + kFields), 0u};
  }
  __device__ static bool suspect(const WCtx&) { return false; }  // every field value is valid
  // emit(j, pos, bw) for the quads j in [qa, qb) of this unit (q, d: the unit's prefix)
  template <class F>
  __device__ static __forceinline__ void emit(const WCtx& c, uint32_t q, uint32_t d, uint32_t qa,
                                              uint32_t qb, F&& f) {
#pragma unroll
    for (int k = 0; k < kPF; k++) {
      const uint32_t bw = CG * (field(c.w, c.part * kPF + k) + 1);
      const uint32_t j = q + k;
      if (j >= qa && j < qb) f(j, d, bw);
      d += bw;
    }
  }
  template <class F>
  __device__ static void walk(const WCtx& c, F&& f) {
    int32_t d = 0;
#pragma unroll
    for (int k = 0; k < kPF; k++) {
      Grp g = grp0();
      g.q0 = k;
      g.nq = 1;
      g.d0 = d;
      g.bw = CG * (field(c.w, c.part * kPF + k) + 1);  // BW = CG*(LD+1)
      g.dlen = g.bw;
      f(g);
      d += (int32_t)g.bw;
    }
  }
};

// ---------------------------------------------------------------- Group-Scheme, complete unary
// Codes are (LD-1) ones then a 0, read MSB-first (A15/A16) and may cross
// bytes and words.  Each control bit stands for CG data bits per lane, so the data
// offset of a code is CG x its start bit (closed form); a word owns the codes whose
// terminating 0 it holds.
template <int CG>
struct CodecGscCU {
  static constexpr bool kExc = false;
  static constexpr uint64_t kBackBits = 32 * CG;  // a code may start in the previous word
  // a parse unit = the codes whose terminating 0 lies in 32/kParts control bits of a word
  // (larger CG means shorter codes, more of them per word: split so the units stay even)
  static constexpr int kParts = CG == 8 ? GC_CU8_PARTS : 1;
  static constexpr uint32_t kB = 32u / kParts;  // control bits per part
  static constexpr bool kNeedsPrev = true;
  static constexpr bool kMultiQuad = false;
  static constexpr bool kVectorGroups = false;
  // stream-order positions [0, n) of a byte-swapped word (bit 31 = first bit)
  __device__ static __forceinline__ uint32_t top(uint32_t n) {
    return n >= 32u ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> n);
  }
  __device__ static __forceinline__ uint32_t part_mask(uint32_t p) {
    return top((p + 1u) * kB) & ~top(p * kB);
  }
  __device__ static WAgg agg(const WCtx& c) {
    if (kParts == 1) return WAgg{(uint32_t)__popc(~c.w), (uint32_t)(CG * 32), 0u};
    const uint32_t z = ~__byte_perm(c.w, 0, 0x0123) & part_mask(c.part);
    return WAgg{(uint32_t)__popc(z), (uint32_t)(CG * kB), 0u};
  }
  __device__ static WAgg word_agg_fast(const WCtx& c) {
    return WAgg{(uint32_t)__popc(~c.w), (uint32_t)(CG * 32), 0u};
  }
  // a run of >= 32/CG ones ending in this word (stream order, MSB first; the previous word
  // of the list included): one inside the word, or the previous word's trailing ones plus
  // this word's leading ones
  __device__ static bool suspect(const WCtx& c) {
    constexpr uint32_t L = 32u / CG;
    const uint32_t cur = __byte_perm(c.w, 0, 0x0123);
    uint32_t y = cur;
    uint32_t have = 1;
#pragma unroll
    for (int s = 0; s < 5; s++) {
      if (have * 2 > L) break;
      y &= y >> have;
      have *= 2;
    }
    if (have < L) y &= y >> (L - have);
    const uint32_t lead = __clz(~cur);  // leading ones of this word (32 if all ones)
    const uint32_t prv = c.widx ? __byte_perm(c.prev, 0, 0x0123) : 0u;
    const uint32_t trail = prv == 0xFFFFFFFFu ? 32u : (uint32_t)(__ffs(~prv) - 1);  // trailing ones
    return y != 0 || (lead > 0 && lead + trail >= L);
  }
  // the start (stream position relative to the word, negative: in the previous word) of
  // the first code ending in part p; *from_prev: it begins in the previous word
  __device__ static __forceinline__ int32_t first_start(const WCtx& c, uint32_t zs, bool& from_prev,
                                                        bool& prev_run) {
    const uint32_t before = zs & top(c.part * kB);
    from_prev = false;
    prev_run = false;
    if (before) return 33 - (int32_t)__ffs(before);  // one bit after the last 0 before p
    if (c.widx == 0) return 0;
    from_prev = true;
    const uint32_t mp = ~__byte_perm(c.prev, 0, 0x0123);
    prev_run = mp == 0;
    return mp ? -(int32_t)(__ffs(mp) - 1) : -32;
  }
  template <class F>
  __device__ static __forceinline__ void emit(const WCtx& c, uint32_t q, uint32_t d, uint32_t qa,
                                              uint32_t qb, F&& f) {
    const uint32_t zs = ~__byte_perm(c.w, 0, 0x0123);
    bool fp, pr;
    int32_t start = first_start(c, zs, fp, pr);
    const int32_t base = (int32_t)(c.part * kB);  // d is the part's data prefix
    uint32_t m = zs & part_mask(c.part);
    uint32_t j = q;
    while (m && j < qb) {
      const int32_t z = (int32_t)__clz(m);
      if (j >= qa) f(j, d + (uint32_t)(CG * (start - base)), min(32u, (uint32_t)(CG * (z - start + 1))));
      start = z + 1;
      m ^= 0x80000000u >> z;
      j++;
    }
  }
  template <class F>
  __device__ static void walk(const WCtx& c, F&& f) {
    const uint32_t zs = ~__byte_perm(c.w, 0, 0x0123);
    bool fp, pr;
    int32_t start = first_start(c, zs, fp, pr);
    const int32_t base = (int32_t)(c.part * kB);
    uint32_t carry_err = (fp && pr) ? (uint32_t)GC_DEV_BAD_LD : 0u;  // a run of >= 32 ones
    uint32_t m = zs & part_mask(c.part);
    uint32_t q = 0;
    while (m) {
      int32_t z = (int32_t)__clz(m);
      uint32_t u = (uint32_t)(z - start + 1);  // LD = code length in bits
      Grp g = grp0();
      g.q0 = q;
      g.nq = 1;
      g.d0 = CG * (start - base);
      g.err = (u > 32u / CG) ? GC_DEV_BAD_LD : carry_err;
      g.bw = g.err ? 32u : CG * u;  // BW = CG*LD
      g.dlen = g.bw;
      f(g);
      carry_err = 0;
      q++;
      start = z + 1;
      m &= ~(0x80000000u >> z);
    }
  }
};

template <int CG>
struct CodecGscIU {
  static constexpr bool kExc = false;
  static constexpr uint64_t kBackBits = 0;
  // a parse unit = 4/kParts control bytes (IU codes never cross a byte; CG 8 packs more,
  // shorter codes per byte, so its words are split)
  static constexpr int kParts = CG == 8 ? GC_IU8_PARTS : 1;
  static constexpr int kBy = 4 / kParts;  // bytes per part
  static constexpr bool kNeedsPrev = false;
  static constexpr bool kMultiQuad = false;
  static constexpr bool kVectorGroups = false;
  __device__ static __forceinline__ WAgg byte_agg(uint32_t w, int i) {
    const uint32_t m = ~(w >> (8 * i)) & 0xFFu;
    return WAgg{(uint32_t)__popc(m), m ? CG * (9u - (uint32_t)__ffs(m)) : 0u, 0u};  // used bits
  }
  __device__ static WAgg agg(const WCtx& c) {
    WAgg t{0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < kBy; i++) {
      const WAgg a = byte_agg(c.w, (int)c.part * kBy + i);
      t.q += a.q;
      t.d += a.d;
    }
    return t;
  }
  __device__ static WAgg word_agg_fast(const WCtx& c) {
    uint32_t d = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) d += byte_agg(c.w, i).d;
    return WAgg{(uint32_t)__popc(~c.w), d, 0u};
  }
  // a byte without a 0, or a code of more than 32/CG units (padding ones excluded)
  __device__ static bool suspect(const WCtx& c) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      uint32_t b = (c.w >> (8 * i)) & 0xFFu;
      if (b == 0xFFu) return true;
      if (32u / CG >= 8u) continue;  // (a code of > 8 units needs a byte of ones: above)
      uint32_t t = b & (b + 1);  // clear the trailing (padding) ones
      uint32_t y = t;
#pragma unroll
      for (uint32_t r = 1; r < 32u / CG; r++) y &= t << r;
      if (y & 0xFFu) return true;
    }
    return false;
  }
  template <class F>
  __device__ static __forceinline__ void emit(const WCtx& c, uint32_t q, uint32_t d, uint32_t qa,
                                              uint32_t qb, F&& f) {
    uint32_t j = q;
#pragma unroll
    for (int i = 0; i < kBy; i++) {
      uint32_t mm = (~(c.w >> (8 * ((int)c.part * kBy + i))) & 0xFFu) << 24;
      uint32_t start = 0;
      while (mm && j < qb) {
        const uint32_t z = __clz(mm);
        if (j >= qa) f(j, d + CG * start, min(32u, CG * (z - start + 1)));
        start = z + 1;
        mm ^= 0x80000000u >> z;
        j++;
      }
      d += CG * start;  // used bits of the byte (the trailing 1s are padding)
    }
  }
  template <class F>
  __device__ static void walk(const WCtx& c, F&& f) {
    int32_t dpos = 0;
    uint32_t q = 0;
#pragma unroll
    for (int i = 0; i < kBy; i++) {
      const uint32_t m = ~(c.w >> (8 * ((int)c.part * kBy + i))) & 0xFFu;
      if (m == 0) {  // 0xFF: a byte with no code
        Grp g = grp0();
        g.q0 = q;
        g.nq = 0;
        g.d0 = dpos;
        g.err = GC_DEV_BAD_LD;
        f(g);
        continue;
      }
      uint32_t mm = m << 24;
      int32_t start = 0;
      while (mm) {
        int32_t z = (int32_t)__clz(mm);
        uint32_t u = (uint32_t)(z - start + 1);
        Grp g = grp0();
        g.q0 = q;
        g.nq = 1;
        g.d0 = dpos + CG * start;
        g.err = (u > 32u / CG) ? GC_DEV_BAD_LD : 0u;
        g.bw = g.err ? 32u : CG * u;
        g.dlen = g.bw;
        f(g);
        q++;
        start = z + 1;
        mm &= ~(0x80000000u >> z);
      }
      dpos += CG * start;
    }
  }
};

// ---------------------------------------------------------------- Group-AFOR
// Header byte (A22): bits 0-1 length code (8/16/32 quads), bits 2-6 bw-1, bit 7 = 0.
// Each frame starts a fresh 128-bit vector: ceil(L*bw/32) vectors.
struct CodecAFOR {
  // a parse unit = one 8-quad part of a frame (frames hold 8, 16 or 32 quads): a
  // header byte per frame, kSub parts per header (those past the frame's length are empty),
  // so a tile of long frames still gives every thread work
  static constexpr uint32_t kSub = GC_AFOR_SUB;
  static constexpr bool kExc = false;
  static constexpr uint64_t kBackBits = 0;
  static constexpr int kParts = 4 * kSub;
  static constexpr uint32_t kUnitsPerThread = GC_FRAME_UPT;
  static constexpr bool kNeedsPrev = false;
  static constexpr bool kMultiQuad = true;
  static constexpr bool kVectorGroups = true;
  static constexpr bool kSplitPieces = GC_AFOR_SPLIT != 0;  // decode: frames queued in 8-quad pieces
  __device__ static __forceinline__ void frame(uint32_t h, uint32_t& L, uint32_t& bw) {
    L = (h & 3u) == 3u ? 8u : (8u << (h & 3u));
    bw = ((h >> 2) & 31u) + 1u;
  }
  // part p: header p / kSub, frame quads [8 s, 8 s + 8) with s = p % kSub (kSub = 1: the
  // whole frame); the frame's padding to whole vectors goes to its last part
  __device__ static __forceinline__ void part(const WCtx& c, uint32_t& h, uint32_t& nq, uint32_t& bw,
                                              uint32_t& d) {
    h = (c.w >> (8 * (c.part / kSub))) & 0xFFu;
    uint32_t L;
    frame(h, L, bw);
    const uint32_t dlen = 32u * ((L * bw + 31u) / 32u);
    if (kSub == 1) {
      nq = L;
      d = dlen;
      return;
    }
    const uint32_t s = c.part % kSub, ns = L / 8u;
    nq = s < ns ? 8u : 0u;
    d = s + 1 < ns ? 8u * bw : (s + 1 == ns ? dlen - 8u * bw * (ns - 1) : 0u);
  }
  __device__ static WAgg agg(const WCtx& c) {
    uint32_t h, nq, bw, d;
    part(c, h, nq, bw, d);
    return WAgg{nq, d, 0u};
  }
  __device__ static WAgg word_agg_fast(const WCtx& c) {
    WAgg t{0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t L, bw;
      frame((c.w >> (8 * k)) & 0xFFu, L, bw);
      t.q += L;
      t.d += 32u * ((L * bw + 31u) / 32u);
    }
    return t;
  }
  __device__ static bool suspect(const WCtx& c) {  // length code 3 or bit 7
    return ((c.w & (c.w >> 1) & 0x01010101u) | (c.w & 0x80808080u)) != 0;
  }
  template <class F>
  __device__ static void walk(const WCtx& c, F&& f) {
    uint32_t h, nq, bw, d;
    part(c, h, nq, bw, d);
    if (nq == 0) return;  // (a part past its frame's end)
    Grp g = grp0();
    g.nq = nq;
    g.bw = bw;
    g.step = bw;
    g.dlen = d;
    g.err = (c.part % kSub == 0 && ((h & 3u) == 3u || (h & 0x80u))) ? GC_DEV_BAD_FRAME : 0u;
    f(g);
  }
};

// ---------------------------------------------------------------- Group-PFD
// Batch-form frame header (A31): byte 0 = b, byte 1 = wcode (0 none, 1/2/3 -> 8/16/32-bit
// values), bytes 2-3 = exception count (LE).  Exceptions of the frame live in the
// exception stream: count positions (u8, or u16 LE when 4F > 256) then count values.
// kE = false: SIMD-BP128 as the special case of P:L424 (PFD variant 1) -- the same frame
// format, every frame packed at its maximum width, no exception stream.
template <int F, bool kE = true>
struct CodecPFD {
  static constexpr bool kExc = kE;
  static constexpr uint32_t kFrameQuads = F;
  static constexpr uint32_t kUnitsPerThread = GC_FRAME_UPT;
  static constexpr uint64_t kBackBits = 0;
  static constexpr int kParts = F / 8;        // a parse unit = 8 quads of one frame
  static constexpr bool kNeedsPrev = false;
  static constexpr bool kMultiQuad = true;
  static constexpr bool kVectorGroups = true;
  static constexpr uint32_t kPosBytes = 4 * F <= 256 ? 1u : 2u;
  __device__ static __forceinline__ uint32_t frame_q(const WCtx& c) {
    uint64_t first = c.widx * (uint64_t)F;
    return c.Q > first ? (uint32_t)mn64((uint64_t)F, c.Q - first) : 0u;
  }
  __device__ static __forceinline__ void decode_hdr(const WCtx& c, Grp& g) {
    uint32_t b = c.w & 0xFFu, wc = (c.w >> 8) & 0xFFu, cnt = c.w >> 16;
    uint32_t q = frame_q(c);
    g.err = 0;
    if (b < 1 || b > 32 || wc > 3) g.err |= GC_DEV_BAD_FRAME;
    if (cnt > 4 * q || (cnt > 0 && wc == 0)) g.err |= GC_DEV_BAD_EXCEPTION;
    if (!kE && (cnt | wc)) g.err |= GC_DEV_BAD_EXCEPTION;  // BP128 frames have none
    g.bw = (b >= 1 && b <= 32) ? b : 32u;
    g.step = g.bw;
    g.fq = q;
    g.dlen = 32u * ((q * g.bw + 31u) / 32u);   // the frame's data: fresh vectors
    g.wb = wc == 1 ? 1u : (wc == 2 ? 2u : (wc == 3 ? 4u : 0u));
    g.cnt = (g.err || !kE) ? 0u : cnt;
    g.elen = kE ? cnt * (kPosBytes + g.wb) : 0u;
  }
  // part p covers frame quads [8p, 8p+8): 8*b data lane-bits each, the frame's padding to
  // whole vectors and all its exception bytes charged to the last / first part
  __device__ static WAgg agg(const WCtx& c) {
    Grp g = grp0();
    decode_hdr(c, g);
    const uint32_t d = c.part + 1 < (uint32_t)kParts ? 8u * g.bw : g.dlen - 8u * g.bw * (kParts - 1);
    return WAgg{8u, d, c.part == 0 ? g.elen : 0u};
  }
  __device__ static bool suspect(const WCtx& c) {
    Grp g = grp0();
    decode_hdr(c, g);
    return g.err != 0;
  }
  template <class F2>
  __device__ static void walk(const WCtx& c, F2&& f) {
    Grp g = grp0();
    decode_hdr(c, g);
    const uint32_t elen = g.elen;
    g.t0 = 8u * c.part;
    g.nq = 8u;
    // data this part really needs (the bounds check), and the frame's exception area
    // relative to the part's exception prefix (parts after the first follow it)
    g.dlen = g.fq > g.t0 ? min(8u, g.fq - g.t0) * g.bw : 0u;
    g.elen = c.part == 0 ? elen : 0u;
    g.e0 = c.part == 0 ? 0u : 0u - elen;
    f(g);
  }
};

// A codec may sum a whole word faster than its parts one by one (word_agg_fast).
template <class C, class = void>
struct HasWordAggFast : std::false_type {};
template <class C>
struct HasWordAggFast<C, std::void_t<decltype(C::word_agg_fast(std::declval<const WCtx&>()))>>
    : std::true_type {};

// Whole-word helpers over a codec's kParts units (the index kernel parses whole words).
template <class C>
__device__ __forceinline__ WAgg word_agg(WCtx c) {
  if constexpr (HasWordAggFast<C>::value) return C::word_agg_fast(c);
  WAgg t{0, 0, 0};
#pragma unroll
  for (int p = 0; p < C::kParts; p++) {
    c.part = p;
    const WAgg a = C::agg(c);
    t.q += a.q;
    t.d += a.d;
    t.e += a.e;
  }
  return t;
}
template <class C, class F>
__device__ __forceinline__ void word_walk(WCtx c, F&& f) {
  uint32_t q = 0, d = 0, e = 0;
#pragma unroll
  for (int p = 0; p < C::kParts; p++) {
    c.part = p;
    C::walk(c, [&](Grp g) {
      g.q0 += q;
      g.d0 += (int32_t)d;
      g.e0 += e;
      f(g);
    });
    if (C::kParts > 1) {
      const WAgg a = C::agg(c);
      q += a.q;
      d += a.d;
      e += a.e;
    }
  }
}

}  // namespace gcd
