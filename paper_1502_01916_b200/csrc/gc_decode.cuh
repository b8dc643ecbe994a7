// gc_decode.cuh -- k_decode (subsystems (b)-(d)); included inside
// namespace gcd by gc_kernels.cu.
//
// Output-space tiles: tile t owns the output ints [t*kT, (t+1)*kT) exactly and decodes
// every quadruple holding one of them (a quad straddling a tile edge is decoded by both
// tiles; each keeps its own ints).  One CTA of kDT threads decodes one tile at a
// time.  Tiles are assigned round-robin (tile = blockIdx.x + i*gridDim.x) to a
// cooperative (co-resident) grid, so the next tile's entries and copies are known early
// and the decoupled look-back always makes progress.  Per tile:
//   1. Entry[t], Entry[t+1] (index kernel) give the tile's control words, data vectors and
//      exception bytes, staged into shared memory by 1-D bulk async copies (TMA engine)
//      issued while the previous tile was being stored.
//   2. List table: the lists the tile touches (rounds of kLC) with their kept quads; the
//      list starts inside the tile go to a reset bitmap.
//   3. Parse + unpack: thread-blocked parse units (a control word or a fixed part of one).
//      A block scan segmented at list starts gives each unit its quad / data / exception
//      prefix; the unit's thread then unpacks its kept quads straight into the staging
//      window: per lane the paper's high-first split is shl/shr/select;
//      Group-PFD exceptions of the unit overwrite their slots.
//   4. d-gap scan: 32 consecutive staged ints per thread, serial, then across the
//      block (segmented by the reset bitmap), then across tiles (decoupled look-back).
//   5. Stores: 128-bit streaming stores, carry-free chunks first, the chunks before the
//      tile's first list start after the look-back.

__host__ __device__ constexpr uint32_t al128(uint32_t x) { return (x + 127u) & ~127u; }
// Tile stores by TMA (cp.async.bulk.tensor, 128-byte swizzle; -DGC_TMA_STORE=1): the staging
// window's swizzle (below) is the TMA's SWIZZLE_128B pattern when the window is 1024-byte
// aligned, so boxes of 8 rows x 32 ints leave straight from it.  The halo is then one whole
// 1 KiB swizzle atom, so every box starts 1024-byte aligned.  Correct (the GPU suite passes
// with it) but 1-2% slower than the 128-bit stores, so off by default.
#ifndef GC_TMA_STORE
#define GC_TMA_STORE 0
#endif
constexpr bool kTma = GC_TMA_STORE != 0;
// Software-pipelined unpack of the one-quad-per-group codecs (-DGC_PIPE=1): see units().
#ifndef GC_PIPE
#define GC_PIPE 0
#endif
constexpr bool kPipe = GC_PIPE != 0;
constexpr uint32_t kHalo = kTma ? 256 : 32;        // staging index = tile position + kHalo
constexpr uint32_t kBoxC = 64;                     // 16-B chunks per TMA store box (8 rows of 32 ints)
constexpr uint32_t kStW = kHalo + kT + 8;          // staging ints
// Staging capacities of a codec.  Frame codecs (PFD, SIMD-BP128) need one control word
// per 4F ints (a tile spans <= 66), so their control staging is small and the space goes to
// data: wide frames (up to 32 bits per int for BP128) still fit; the CTA's shared memory
// is the same as for the other codecs.
template <class C, class = void>
struct Caps {
  static constexpr uint32_t ccap = kCCap, dcap = kDCap;
};
template <class C>
struct Caps<C, std::void_t<decltype(C::kFrameQuads)>> {
  static constexpr uint32_t ccap = 256;
  static constexpr uint32_t dcap = kDCap + (kCCap - ccap) * 4 / 16 + (C::kExc ? 0u : kECap / 16);
};
// Group-AFOR: one header byte per 8..32-quad frame, so a tile needs ~64 control words (plus
// one per list start): 512 staged words leave room for the piece queue.
template <>
struct Caps<CodecAFOR, void> {
  static constexpr uint32_t ccap = 512, dcap = kDCap;
};
template <class C>
struct DS {  // dynamic shared memory layout (byte offsets)
  static constexpr uint32_t kCC = Caps<C>::ccap, kDC = Caps<C>::dcap;
  static constexpr uint32_t kOut = 0;                                 // kStW u32, swizzled
  static constexpr uint32_t kData = al128(kOut + kStW * 4);           // (kDC + 1) uint4
  static constexpr uint32_t kCtrl = al128(kData + (kDC + 1) * 16);    // kCC u32
  static constexpr uint32_t kLtF = 8;                                 // list table fields
  static constexpr uint32_t kLt = al128(kCtrl + kCC * 4);             // kLtF x (kLC + 1) u32
  static constexpr uint32_t kRst = al128(kLt + kLtF * (kLC + 1) * 4);  // kT/32 u32 bitmap
  static constexpr uint32_t kExcB = al128(kRst + kT / 8);             // kECap bytes (PFD)
  __host__ __device__ static constexpr uint32_t bytes() {
    return C::kExc ? al128(kExcB + kECap) : kExcB;
  }
};

// Staging swizzle: 16-B chunk c lives at chunk c ^ ((c >> 3) & 7), which keeps the blocked
// (8 chunks per thread) and striped (one chunk per thread) 128-bit accesses conflict-free
// and spreads the scalar writes of thread-serial runs.
__device__ __forceinline__ uint32_t sw_chunk(uint32_t c) { return c ^ ((c >> 3) & 7u); }
__device__ __forceinline__ uint32_t sw_word(uint32_t x) {  // == sw_chunk(x >> 2) * 4 + (x & 3)
  return x ^ ((x >> 3) & 0x1Cu);
}

#ifdef GC_TIMING
#define GC_T(i)                                                         \
  do {                                                                  \
    if (tid == 0) {                                                     \
      const long long now = clock64();                                  \
      atomicAdd(&D.hdr->prof[i], (unsigned long long)(now - t_last));   \
      t_last = now;                                                     \
    }                                                                   \
  } while (0)
#else
#define GC_T(i) \
  do {          \
  } while (0)
#endif

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Stream ranges of one tile (set up by one thread from the tile's two entries).
struct Geo {
  uint32_t ok, k0, k1, ctrl_st;
  uint32_t data_st, exc_st, pad0, pad1;
  uint64_t wa, wb, cbase, cstop, va, vb, ea, eb, la, lb;
  Seg4 seed;  // (list start flag, raw quads, data lane-bits, exception bytes) at word wa
};

// Parse units per thread per parse chunk: kUPT, or a codec's own kUnitsPerThread (the
// frame codecs, whose units are whole 8..32-quad frame parts, balance better with 2).
template <class C, class = void>
struct UnitsPerThread {
  static constexpr uint32_t v = kUPT;
};
template <class C>
struct UnitsPerThread<C, std::void_t<decltype(C::kUnitsPerThread)>> {
  static constexpr uint32_t v = C::kUnitsPerThread;
};

// Work split for codecs with long multi-quad groups (Group-AFOR frames of 8..32 quads, one
// parse unit each): a unit's thread unpacks the first kPiece quads of its frame and queues
// the rest as kPiece-quad pieces, which every thread then takes round-robin -- the lanes of
// a warp no longer wait for the one holding a 32-quad frame (ncu: 12 of 32 lanes active in
// the unpack loop without it).
template <class C, class = void>
struct SplitPieces {
  static constexpr bool v = false;
};
template <class C>
struct SplitPieces<C, std::void_t<decltype(C::kSplitPieces)>> {
  static constexpr bool v = C::kSplitPieces;
};
#ifndef GC_PIECE
#define GC_PIECE 4
#endif
constexpr uint32_t kPiece = GC_PIECE;                // quads per queued piece
constexpr uint32_t kPQ = 2560 / kPiece;              // queue capacity (a tile holds <= ~2050 quads)

#ifndef GC_DECODE_MINB
#define GC_DECODE_MINB 3
#endif
// PAIR: one pass over two batches of one codec that share the output tiling -- a posting
// store's docIDs (batch 0, d-gap scan) and term frequencies (batch 1, raw) -- their tiles
// interleaved (virtual tile 2t = docIDs tile t, 2t+1 = TFs tile t): one launch, the same
// CTAs, the TF tiles' unpack filling the docID tiles' look-back latency.
// tm0 / tm1: 2-D tensor maps of out0 / out1 ({32 ints, total_out / 32 rows}, boxes of 8 rows,
// 128-byte swizzle); bit b of tma says tm<b> is valid (else plain 128-bit stores).
template <class C, bool DGAPS, bool PAIR = false>
__global__ void __launch_bounds__(kDT, GC_DECODE_MINB) k_decode(Dev D0, uint32_t* __restrict__ out0,
                                                                Dev D1, uint32_t* __restrict__ out1,
                                                                const __grid_constant__ CUtensorMap tm0,
                                                                const __grid_constant__ CUtensorMap tm1,
                                                                uint32_t tma) {
  const Dev& D = D0;       // (the docIDs batch: the look-back and the deferred carry stores)
  uint32_t* out = out0;
  // virtual tile vt -> its batch and its tile index in that batch
  auto bat = [&](uint32_t vt) -> const Dev& { return (PAIR && (vt & 1u)) ? D1 : D0; };
  auto tix = [&](uint32_t vt) { return PAIR ? vt >> 1 : vt; };
  const uint32_t nvt = PAIR ? 2 * D0.n_tiles_b : D0.n_tiles_b;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t* s_out = reinterpret_cast<uint32_t*>(sm + DS<C>::kOut);
  uint4* s_out4 = reinterpret_cast<uint4*>(sm + DS<C>::kOut);
  uint4* s_data = reinterpret_cast<uint4*>(sm + DS<C>::kData);
  uint32_t* s_ctrl = reinterpret_cast<uint32_t*>(sm + DS<C>::kCtrl);
  uint32_t* s_lt = reinterpret_cast<uint32_t*>(sm + DS<C>::kLt);
  uint32_t* s_rst = reinterpret_cast<uint32_t*>(sm + DS<C>::kRst);
  uint8_t* s_exc = sm + DS<C>::kExcB;
  uint32_t* lt_cw = s_lt + 0 * (kLC + 1);    // first control word, relative to cbase (wraps)
  uint32_t* lt_q = s_lt + 1 * (kLC + 1);     // quads
  uint32_t* lt_n = s_lt + 2 * (kLC + 1);     // ints
  uint32_t* lt_klo = s_lt + 3 * (kLC + 1);   // first quad kept by the tile
  uint32_t* lt_kend = s_lt + 4 * (kLC + 1);  // one past the last
  uint32_t* lt_oref = s_lt + 5 * (kLC + 1);  // staging index of quad j = oref + 4j (wraps)
  uint32_t* lt_db = s_lt + 6 * (kLC + 1);    // data lane-bit of the list start, rel. to va*32
  uint32_t* lt_eb = s_lt + 7 * (kLC + 1);    // exception byte of the list start, rel. to ea
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ __align__(16) Entry s_e[2];   // entries of the next tile
  __shared__ Geo s_g[2];                   // geometry of the current / next tile
  __shared__ Seg4 s_scr4[kDW];
  __shared__ Seg1 s_scr1[kDW];
  __shared__ uint32_t s_reset0[2], s_cin;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!kTma || (smem_addr(sm) & 1023u) != 0) tma = 0;  // (the swizzle atoms must be aligned)
  constexpr uint32_t kU = UnitsPerThread<C>::v;  // parse units per thread per parse chunk
  uint32_t phase = 0, err = 0;

  // Entries of virtual tile vt -> s_e (one warp)
  auto load_entries = [&](uint32_t vt) {
    const Dev& B = bat(vt);
    const uint32_t tile = tix(vt);
    if (vt < nvt) {
      if (lane < 16) {
        reinterpret_cast<uint32_t*>(s_e)[lane] =
            reinterpret_cast<const uint32_t*>(B.entries + tile)[lane];
      } else if (tile + 1 < B.n_tiles_b) {
        reinterpret_cast<uint32_t*>(s_e)[lane] =
            reinterpret_cast<const uint32_t*>(B.entries + tile + 1)[lane - 16];
      }
    }
  };
  // One thread: the tile's stream ranges from s_e -> s_g[buf], and the bulk async copies
  // of its control / exception bytes (barrier 0) and data (barrier 1).  A tile past the
  // end or with bad entries arms both barriers with 0 bytes.
  auto setup = [&](uint32_t vt, uint32_t buf) {
    const Dev& D = bat(vt);
    const uint32_t tile = tix(vt);
    Geo& g = s_g[buf];
    const Entry& E0 = s_e[0];
    const Entry& E1 = s_e[1];
    const bool last = tile + 1 == D.n_tiles_b;
    // the batch's stream ends bound only the last tile: read them there alone (thread 0's
    // global round trip would otherwise sit in every tile's path to the next barrier)
    uint64_t cend = 0, dend = 0, eend = 0;
    if (last && vt < nvt) {
      cend = D.ctrl_off[D.n_lists] >> 2;  // end of the last list's control
      dend = D.data_off[D.n_lists];
      eend = C::kExc ? D.exc_off[D.n_lists] : 0ull;
    }
    g.ok = 0;
    uint32_t cbytes = 0, xbytes = 0, dbytes = 0;
    if (vt < nvt) {
      const uint64_t wa = E0.w, wb = last ? cend - 1 : E1.w;
      g.ok = (E0.valid && (last || E1.valid) && wb >= wa && wb < D.n_ctrl_words &&
              E0.l < D.n_lists && (last || (E1.l >= E0.l && E1.l < D.n_lists))) ? 1u : 0u;
      if (!g.ok) atomicOr(&D.hdr->status, (uint32_t)GC_DEV_TRUNCATED);
    }
    if (g.ok) {
      const uint64_t wa = E0.w, wb = last ? cend - 1 : E1.w;
      g.wa = wa;
      g.wb = wb;
      g.cbase = (wa ? wa - 1 : 0) & ~3ull;
      g.cstop = mn64((wb + 4) & ~3ull, D.n_ctrl_words);
      g.ctrl_st = g.cstop - g.cbase <= DS<C>::kCC;
      // a group may start before its word's data prefix (complete unary: up to CG*32 lane
      // bits, the code's start in the previous word)
      g.va = (E0.wd - mn64(E0.wd, C::kBackBits)) >> 5;
      g.vb = mx64(g.va, mn64(last ? dend : (E1.wd_end + 31) >> 5, D.data_vectors));
      g.data_st = g.vb - g.va <= DS<C>::kDC;
      g.ea = g.eb = 0;
      g.exc_st = 0;
      if (C::kExc) {
        g.ea = E0.we & ~15ull;
        g.eb = mx64(g.ea, mn64(((last ? eend : E1.we_end) + 15) & ~15ull, D.exc_bytes));
        g.exc_st = g.eb - g.ea <= kECap;
      }
      g.la = E0.l;
      g.lb = last ? D.n_lists - 1 : E1.l;
      g.k0 = E0.k;
      g.k1 = last ? 0x7FFFFFFFu : E1.k;  // (the last tile keeps every quad of its last list)
      g.seed = Seg4{1u, E0.wq, (uint32_t)(E0.wd - g.va * 32ull), (uint32_t)(E0.we - g.ea)};
      cbytes = g.ctrl_st ? (uint32_t)(g.cstop - g.cbase) * 4 : 0u;
      xbytes = g.exc_st ? (uint32_t)(g.eb - g.ea) : 0u;
      dbytes = g.data_st ? (uint32_t)(g.vb - g.va) * 16 : 0u;
    }
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[0], cbytes + xbytes);
    if (cbytes) bulk_g2s(s_ctrl, D.ctrl_words + g.cbase, cbytes, &s_bar[0]);
    if (xbytes) bulk_g2s(s_exc, D.exc + g.ea, xbytes, &s_bar[0]);
    mbar_expect_tx(&s_bar[1], dbytes);
    if (dbytes) bulk_g2s(s_data, D.data + g.va, dbytes, &s_bar[1]);
  };

  // A tile whose first list continues from earlier tiles publishes its aggregate and
  // stores its carry-free chunks at once; its look-back and carry chunks wait until the
  // next tile has parsed (just before that tile's first staging write), so the predecessors
  // have had time to publish and the wait overlaps the next tile's list table and parse.
  struct Pend {
    uint32_t on, tile, nvalid, cfree, reset0, f, v, pad;
    uint64_t tT;
  };
  __shared__ Pend s_pend;
  constexpr bool kSplit = SplitPieces<C>::v;
  // piece = (data lane-bit of its first quad, idx[13:0] | rem[19:14] | cnt[23:20] | bw[29:24])
  __shared__ uint2 s_pq[kSplit ? kPQ : 1];
  __shared__ uint32_t s_qn;
  auto flush_pending = [&]() {  // all threads; s_pend.on was read after a barrier
    if (warp == 0) {
#ifdef GC_ABL_NOLB
      const uint32_t cin = 0;
#else
      const uint32_t cin = lookback_u32(D.tiles_b, s_pend.tile, D.hdr->prof + 12);
#endif
      if (tid == 0) {
        if (!s_pend.f) st_relaxed_u64(D.tiles_b + s_pend.tile, ((uint64_t)kFlagIncl << 32) | (cin + s_pend.v));
        s_cin = cin;
      }
    }
    __syncthreads();
    const uint32_t cin = s_cin, reset0 = s_pend.reset0, nvalid = s_pend.nvalid, cfree = s_pend.cfree;
    const uint64_t tT = s_pend.tT;
    // every thread has tested s_pend.on (before entering) and read it (above): clear it
    // before the closing barrier, so no thread can see the stale flag afterwards
    if (tid == 0) s_pend.on = 0;
    // chunks wholly before the first list start and wholly valid: the plain path
    const uint32_t cfast = min(cfree, min(reset0, nvalid) >> 2);
    uint4* o4 = reinterpret_cast<uint4*>(out + tT);
#pragma unroll 2
    for (uint32_t c = tid; c < cfast; c += kDT) {
      GC_CHECK(tT + 4 * c + 4 <= D.total_out);
      uint4 v = s_out4[sw_chunk(kHalo / 4 + c)];
      v.x += cin;
      v.y += cin;
      v.z += cin;
      v.w += cin;
      __stcs(o4 + c, v);
    }
    for (uint32_t c = cfast + tid; c < cfree; c += kDT) {
      uint4 v = s_out4[sw_chunk(kHalo / 4 + c)];
      const uint32_t p = 4 * c;
      if (p + 4 <= reset0) {
        v.x += cin;
        v.y += cin;
        v.z += cin;
        v.w += cin;
      } else {
        if (p < reset0) v.x += cin;
        if (p + 1 < reset0) v.y += cin;
        if (p + 2 < reset0) v.z += cin;
      }
      GC_CHECK(tT + p + 4 <= D.total_out || p + 4 > nvalid);
      if (p + 4 <= nvalid) {
        __stcs(reinterpret_cast<uint4*>(out + tT) + c, v);
      } else {
        const uint32_t a4[4] = {v.x, v.y, v.z, v.w};
        for (uint32_t k = 0; k < 4; k++)
          if (p + k < nvalid) out[tT + p + k] = a4[k];
      }
    }
    __syncthreads();
  };

  // prologue: the first tile's entries and copies
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  const uint32_t first_tile = blockIdx.x;
  if (warp == 0) load_entries(first_tile);
  if (DGAPS) s_rst[tid] = 0u;  // kT / 32 == kDT words
  if (tid == 0) {
    s_reset0[0] = kT;
    s_pend.on = 0;
    s_qn = 0;
  }
  __syncthreads();
  if (tid == 0) setup(first_tile, 0);
  __syncthreads();

  uint32_t buf = 0;
  long long t_last = clock64();
  for (uint32_t vt = first_tile; vt < nvt; vt += gridDim.x, buf ^= 1u) {
    GC_T(0);
    const Dev& D = bat(vt);                             // this tile's batch
    uint32_t* const out = (PAIR && (vt & 1u)) ? out1 : out0;
    const uint32_t tile = tix(vt);
    const bool dg = DGAPS && !(PAIR && (vt & 1u));    // (TFs: no d-gap)
    const bool use_tma = (tma >> ((PAIR && (vt & 1u)) ? 1 : 0)) & 1u;
    const CUtensorMap* tm = (PAIR && (vt & 1u)) ? &tm1 : &tm0;
    // warp 1 prefetches the next tile's entries (read after this tile's unpack)
    if (warp == 1) load_entries(vt + gridDim.x);
    if (tid == 0) s_reset0[buf ^ 1u] = kT;  // the next tile's
    const Geo& G = s_g[buf];
    const bool ok = G.ok;
    const bool last = tile + 1 == D.n_tiles_b;
    const uint64_t tT = (uint64_t)tile * kT;
    uint64_t cbase = 0, va = 0, ea = 0, la = 0, nl = 0;
    uint32_t ncw = 0, dlim = 1, elim = 0, E0k = 0, E1k = 0, rwa = 0, rwb = 0;
    bool data_st = false;
    const uint32_t* cwp = D.ctrl_words;
    const uint8_t* eptr = D.exc;
    Seg4 seed{0u, 0u, 0u, 0u};
    if (ok) {
      cbase = G.cbase;
      va = G.va;
      ea = G.ea;
      la = G.la;
      nl = G.lb - G.la + 1;
      ncw = (uint32_t)(G.cstop - cbase);
      dlim = (uint32_t)mn64(mx64(G.vb - va, 1), 0x7FFFFFFFull);
      elim = (uint32_t)mn64(G.eb - ea, 0x7FFFFFFFull);
      data_st = G.data_st;
      cwp = G.ctrl_st ? s_ctrl : D.ctrl_words + cbase;  // word w at cwp[w - cbase]
      eptr = G.exc_st ? s_exc : D.exc + ea;
      E0k = G.k0;
      E1k = G.k1;
      seed = G.seed;
      rwa = (uint32_t)(G.wa - cbase);
      rwb = (uint32_t)(G.wb + 1 - cbase);
    }
    const uint64_t lb = la + nl - 1;
    bool w0done = false, w1done = false;

    // the two data vectors of a quad at data lane-bit pos
    auto load_quad = [&](uint32_t pos, uint4& v0, uint4& v1, auto staged) {
      constexpr bool kStaged = decltype(staged)::value;
      const uint32_t m = min(pos >> 5, dlim - 1u);
      if constexpr (kStaged) {
        GC_CHECK(m + 1 <= DS<C>::kDC);
        v0 = s_data[m];
        v1 = s_data[m + 1];  // slack vector past the staged range
      } else {
        GC_CHECK(va + m < D.data_vectors);
        v0 = __ldg(D.data + va + m);
        v1 = __ldg(D.data + va + min(m + 1, dlim - 1u));
      }
    };
    // 4 values of BW bits at bit `off` of v0 (continued in v1) to staging indices idx ..
    // idx + min(4, rem) - 1
    auto stage_quad = [&](const uint4& v0, const uint4& v1, uint32_t off, uint32_t bw, uint32_t idx,
                          uint32_t rem) {
      // the value's high part is the top of the current component, its low part the
      // bottom of the next vector's component
      const bool strad = off + bw > 32u;
      const uint32_t shl = strad ? 0u : 32u - off - bw, shr = 32u - bw;
      const uint32_t ml = strad ? (1u << (off + bw - 32u)) - 1u : 0u;
      const uint32_t x0 = (((v0.x << shl) >> shr) & ~ml) | (v1.x & ml);
      const uint32_t x1 = (((v0.y << shl) >> shr) & ~ml) | (v1.y & ml);
      const uint32_t x2 = (((v0.z << shl) >> shr) & ~ml) | (v1.z & ml);
      const uint32_t x3 = (((v0.w << shl) >> shr) & ~ml) | (v1.w & ml);
      idx = min(idx, kStW - 4u);
      GC_CHECK(sw_word(idx) < kStW && sw_word(idx + 3) < kStW);
      if (rem >= 4u && (idx & 3u) == 0) {
        s_out4[sw_chunk(idx >> 2)] = make_uint4(x0, x1, x2, x3);
      } else {
        // a list's quads sit at any word offset: four scalar stores, branch-free (the ints
        // past the list's end go to halo words 0..2, which no tile position maps to)
        s_out[sw_word(idx)] = x0;
        s_out[rem > 1u ? sw_word(idx + 1) : 0u] = x1;
        s_out[rem > 2u ? sw_word(idx + 2) : 1u] = x2;
        s_out[rem > 3u ? sw_word(idx + 3) : 2u] = x3;
      }
    };
    // one quad: 4 values of BW bits at data lane-bit pos; their ints go to staging
    // indices idx .. idx + min(4, rem) - 1
    auto unpack_quad = [&](uint32_t pos, uint32_t bw, uint32_t idx, uint32_t rem, auto staged) {
      uint4 v0, v1;
      load_quad(pos, v0, v1, staged);
      stage_quad(v0, v1, pos & 31u, bw, idx, rem);
    };

    for (uint64_t lr = 0; lr < nl; lr += kLC) {
      // ---------------------------------------------------------------- list table
      const uint32_t cnt = (uint32_t)mn64(kLC, nl - lr);
      if (lr) __syncthreads();  // the previous list round is done with the table
      if (tid < cnt) {
        const uint64_t l = la + lr + tid;
        GC_CHECK(l < D.n_lists && tid < kLC);
        const uint32_t n = D.list_n[l];
        const uint32_t Q = (n + 3) >> 2;
        const uint32_t klo = l == la ? E0k : 0u;
        const uint32_t kend = l == lb ? min(Q, E1k + 1) : Q;
        const uint32_t oref = (uint32_t)(D.out_off[l] - tT + kHalo);
        lt_cw[tid] = (uint32_t)((D.ctrl_off[l] >> 2) - cbase);
        lt_q[tid] = Q;
        lt_n[tid] = n;
        lt_klo[tid] = klo;
        lt_kend[tid] = kend;
        lt_oref[tid] = oref;
        lt_db[tid] = (uint32_t)(D.data_off[l] * 32ull - va * 32ull);
        lt_eb[tid] = C::kExc ? (uint32_t)(D.exc_off[l] - ea) : 0u;
        // a list that starts inside the tile resets the d-gap scan
        if (dg && n > 0 && klo == 0 && oref >= kHalo && oref < kHalo + kT) {
          atomicOr(&s_rst[(oref - kHalo) >> 5], 1u << ((oref - kHalo) & 31u));
          atomicMin(&s_reset0[buf], oref - kHalo);
        }
      }
      if (tid == 0) lt_cw[cnt] = lr + cnt < nl ? (uint32_t)((D.ctrl_off[la + lr + cnt] >> 2) - cbase) : rwb;
      if (!w0done) {
        mbar_wait(&s_bar[0], phase);
        w0done = true;
      }
      if (kTma && warp == 0) bulk_wait_read0();  // the previous tile's TMA stores have read staging
      __syncthreads();
      GC_T(1);
      const uint32_t rw0 = lr == 0 ? rwa : lt_cw[0];
      const uint32_t rw1 = lt_cw[cnt];

      // -------------------------------------------------------------- parse + unpack
      constexpr uint32_t P = C::kParts;
      const uint32_t ru0 = rw0 * P, ru1 = rw1 * P;
      const uint32_t nu = ru1 > ru0 ? ru1 - ru0 : 0u;
      const uint32_t ku = max(1u, min(kU, (nu + kDT - 1) / kDT));
      Seg4 carry = lr == 0 ? seed : Seg4{0u, 0u, 0u, 0u};
      for (uint32_t cb0 = ru0; cb0 < ru1; cb0 += kDT * ku) {
        const uint32_t my0 = cb0 + tid * ku;
        const uint32_t myn = my0 < ru1 ? min(ku, ru1 - my0) : 0u;
        uint32_t li = 0;
        if (myn) {  // the last table entry whose first word is <= my first word
          const uint32_t key = my0 / P;
          uint32_t a = 0, b = cnt;
          while (b - a > 1) {
            const uint32_t m = (a + b) >> 1;
            if (lt_cw[m] <= key) a = m;
            else b = m;
          }
          li = a;
        }
        uint32_t wv[kU], pv[kU], wl[kU];
        WAgg wg[kU];
        Seg4 agg{0u, 0u, 0u, 0u};
#pragma unroll
        for (uint32_t k = 0; k < kU; k++) {
          wv[k] = pv[k] = 0u;
          wl[k] = li;
          wg[k] = WAgg{0u, 0u, 0u};
          if (k < myn) {
            const uint32_t un = my0 + k, w = un / P, part = un % P;
            while (li + 1 < cnt && lt_cw[li + 1] <= w) li++;
            wl[k] = li;
            GC_CHECK(w >= ncw || !G.ctrl_st || w < DS<C>::kCC);
            GC_CHECK(w >= ncw || cbase + w < D.n_ctrl_words);
            wv[k] = w < ncw ? cwp[w] : 0u;
            pv[k] = (C::kNeedsPrev && w >= 1 && w - 1 < ncw) ? cwp[w - 1] : 0u;
            const uint32_t widx = w - lt_cw[li];
            const WAgg a = C::agg(WCtx{wv[k], pv[k], widx, lt_q[li], part});
            wg[k] = a;
            agg = (widx == 0 && part == 0) ? Seg4{1u, a.q, lt_db[li] + a.d, lt_eb[li] + a.e}
                                           : Seg4{agg.f, agg.q + a.q, agg.d + a.d, agg.e + a.e};
          }
        }
        Seg4 tot;
        Seg4 S = seg4_op(carry, block_excl_seg4<C::kExc, kDW>(agg, s_scr4, &tot));
        carry = seg4_op(carry, tot);
        GC_T(2);
        if (!w1done) {
          mbar_wait(&s_bar[1], phase);
          w1done = true;
        }
        auto units = [&](auto staged) {
          uint4 p_v0 = make_uint4(0u, 0u, 0u, 0u), p_v1 = p_v0;  // (kPipe) the quad in flight
          uint32_t p_off = 0, p_bw = 0, p_idx = 0, p_rem = 0;
          bool p_have = false;
#pragma unroll
          for (uint32_t k = 0; k < kU; k++) {
            if (k >= myn) break;
            const uint32_t un = my0 + k, w = un / P, part = un % P;
            const uint32_t i = wl[k];
            const uint32_t widx = w - lt_cw[i];
            if (widx == 0 && part == 0) S = Seg4{1u, 0u, lt_db[i], lt_eb[i]};
            const WAgg a = wg[k];
            const uint32_t qa = max(S.q, lt_klo[i]), qb = min(S.q + a.q, lt_kend[i]);
            if (qb > qa) {
              const WCtx c{wv[k], pv[k], widx, lt_q[i], part};
              const uint32_t n = lt_n[i], oref = lt_oref[i];
              if constexpr (!C::kMultiQuad && kPipe) {
                // one quad per group, software-pipelined: a quad's vectors are loaded before
                // the previous quad is shifted, masked and staged, so the shared-memory load
                // latency overlaps that work (the compiler cannot move the loads above the
                // staging stores itself: both are shared memory)
                C::emit(c, S.q, S.d, qa, qb, [&](uint32_t j, uint32_t pos, uint32_t bw) {
                  uint4 v0, v1;
                  load_quad(pos, v0, v1, staged);
                  if (p_have) stage_quad(p_v0, p_v1, p_off, p_bw, p_idx, p_rem);
                  p_v0 = v0;
                  p_v1 = v1;
                  p_off = pos & 31u;
                  p_bw = bw;
                  p_idx = oref + 4u * j;
                  p_rem = n - 4u * j;
                  p_have = true;
                });
              } else if constexpr (!C::kMultiQuad) {
                // one quad per group: the codec's tight loop straight into the unpack
                C::emit(c, S.q, S.d, qa, qb, [&](uint32_t j, uint32_t pos, uint32_t bw) {
                  unpack_quad(pos, bw, oref + 4u * j, n - 4u * j, staged);
                });
              } else {
                const Seg4 SW = S;
                C::walk(c, [&](const Grp& g) {
                  const uint32_t gq = SW.q + g.q0;
                  const uint32_t ja = max(gq, qa), jb = min(gq + g.nq, qb);
                  if (ja >= jb) return;
                  const uint32_t gd = SW.d + (uint32_t)g.d0;
                  uint32_t jend = jb;
                  if constexpr (kSplit) {
                    if (jb - ja > kPiece) {
                      jend = ja + kPiece;
                      // one slot reservation for all of the group's pieces
                      const uint32_t np = (jb - jend + kPiece - 1) / kPiece;
                      uint32_t slot = oref + 4u * jb < (1u << 14) ? atomicAdd(&s_qn, np) : kPQ;
                      for (uint32_t p = jend; p < jb; p += kPiece, slot++) {
                        const uint32_t cnt = min(kPiece, jb - p);
                        const uint32_t pos = gd + (p - gq) * g.step, idx = oref + 4u * p;
                        if (slot < kPQ) {
                          s_pq[slot] = make_uint2(pos, idx | (min(n - 4u * p, 32u) << 14) | (cnt << 20) |
                                                           (g.bw << 24));
                        } else {
                          for (uint32_t j = p; j < p + cnt; j++)
                            unpack_quad(gd + (j - gq) * g.step, g.bw, oref + 4u * j, n - 4u * j, staged);
                        }
                      }
                    }
                  }
                  for (uint32_t j = ja; j < jend; j++)
                    unpack_quad(gd + (j - gq) * g.step, g.bw, oref + 4u * j, n - 4u * j, staged);
                  if constexpr (C::kExc) {
                    // Group-PFD: the frame's exceptions in this unit's quads overwrite their
                    // slots; positions are frame-relative ints, values follow them
                    const uint32_t pb = C::kPosBytes;
                    const uint32_t e0 = SW.e + g.e0;
                    const uint32_t fq0 = gq - g.t0;  // the frame's first quad in the list
                    const uint32_t ta = 4u * (ja - fq0), tb = 4u * (jb - fq0);
                    if (e0 + g.cnt * (pb + g.wb) > elim) {
                      err |= GC_DEV_TRUNCATED;
                    } else {
                      uint32_t pprev = 0;
                      for (uint32_t x = 0; x < g.cnt; x++) {
                        GC_CHECK(e0 + x * pb + pb <= elim && (!G.exc_st || elim <= kECap));
                        uint32_t p = eptr[e0 + x * pb];
                        if (pb == 2) p |= (uint32_t)eptr[e0 + x * pb + 1] << 8;
                        if (p >= 4u * g.fq || (x > 0 && p <= pprev)) {
                          err |= GC_DEV_BAD_EXCEPTION;
                          break;
                        }
                        pprev = p;
                        if (p < ta) continue;
                        if (p >= tb) break;
                        const uint32_t b0 = e0 + g.cnt * pb + x * g.wb;
                        GC_CHECK(b0 + g.wb <= elim);
                        uint32_t v = eptr[b0];
                        if (g.wb > 1) v |= (uint32_t)eptr[b0 + 1] << 8;
                        if (g.wb > 2) v |= ((uint32_t)eptr[b0 + 2] << 16) | ((uint32_t)eptr[b0 + 3] << 24);
                        s_out[sw_word(min(oref + 4u * fq0 + p, kStW - 1u))] = v;
                      }
                    }
                  }
                });
              }
            }
            S.q += a.q;
            S.d += a.d;
            S.e += a.e;
          }
          if (kPipe && p_have) stage_quad(p_v0, p_v1, p_off, p_bw, p_idx, p_rem);
        };
        if (DGAPS && s_pend.on) {  // (uniform: s_pend.on only changes behind barriers)
          GC_T(3);
          flush_pending();
          GC_T(8);
        }
        if (data_st) units(std::true_type{});
        else units(std::false_type{});
        GC_T(3);
      }
    }
    if (!w0done) mbar_wait(&s_bar[0], phase);
    if (!w1done) mbar_wait(&s_bar[1], phase);
    phase ^= 1u;
    if constexpr (kSplit) {
      __syncthreads();  // every unit has queued its pieces
      const uint32_t nq = min(s_qn, kPQ);
      auto pieces = [&](auto staged) {
        for (uint32_t x = tid; x < nq; x += kDT) {
          const uint2 pc = s_pq[x];
          const uint32_t idx = pc.y & 0x3FFFu, rem = (pc.y >> 14) & 63u;
          const uint32_t cnt = (pc.y >> 20) & 15u, bw = pc.y >> 24;
          for (uint32_t k = 0; k < cnt; k++) unpack_quad(pc.x + k * bw, bw, idx + 4u * k, rem - 4u * k, staged);
        }
      };
      if (data_st) pieces(std::true_type{});
      else pieces(std::false_type{});
    }
    if (DGAPS && s_pend.on) flush_pending();  // (a tile that staged nothing)
    if (kTma && warp == 0) bulk_wait_read0();  // (a tile without list rounds)
    if (kTma && !dg) fence_proxy_async_smem();  // the staged ints are read by the TMA stores
    __syncthreads();  // the tile is staged; the staging buffers and the next entries are free
    // the next tile's copies overlap this tile's scan, look-back and stores
    if (tid == 0) {
      setup(vt + gridDim.x, buf ^ 1u);
      if (kSplit) s_qn = 0;  // (every thread read it before the barrier above)
    }
    GC_T(4);

    // ------------------------------------------------------------------ d-gap scan
    const uint32_t nvalid = ok ? (last ? (uint32_t)(D.total_out - tT) : kT) : 0u;
    const uint32_t nch = (nvalid + 3) / 4;
    Seg1 rcarry{0u, 0u};
    if (dg && ok) {
      // thread t scans tile positions [32t, 32t+32) (staging chunks kHalo/4 + 8t ..)
      uint32_t v[32];
      const uint32_t cb = kHalo / 4 + 8 * tid;
#pragma unroll
      for (uint32_t a = 0; a < 8; a++) {
        const uint4 q = s_out4[sw_chunk(cb + a)];
        v[4 * a] = q.x;
        v[4 * a + 1] = q.y;
        v[4 * a + 2] = q.z;
        v[4 * a + 3] = q.w;
      }
      const uint32_t rb = s_rst[tid];
      s_rst[tid] = 0u;  // clean for the next tile
      if (rb == 0) {
#pragma unroll
        for (uint32_t i = 1; i < 32; i++) v[i] += v[i - 1];
      } else {
#pragma unroll
        for (uint32_t i = 1; i < 32; i++) v[i] = ((rb >> i) & 1u) ? v[i] : v[i] + v[i - 1];
      }
      Seg1 rt;
      const Seg1 ex = block_excl_seg1<kDW>(Seg1{rb ? 1u : 0u, v[31]}, s_scr1, &rt);
      rcarry = rt;
      if (ex.v) {
        if (rb == 0) {  // no list starts in my 32 positions (the common case)
#pragma unroll
          for (uint32_t i = 0; i < 32; i++) v[i] += ex.v;
        } else {
          const uint32_t first = (uint32_t)(__ffs(rb) - 1);
#pragma unroll
          for (uint32_t i = 0; i < 32; i++)
            if (i < first) v[i] += ex.v;
        }
      }
#pragma unroll
      for (uint32_t a = 0; a < 8; a++)
        s_out4[sw_chunk(cb + a)] = make_uint4(v[4 * a], v[4 * a + 1], v[4 * a + 2], v[4 * a + 3]);
      if (kTma) fence_proxy_async_smem();  // the scanned ints are read by the TMA stores
      if (tid == 0)
        st_relaxed_u64(D.tiles_b + tile, ((uint64_t)(rcarry.f ? kFlagIncl : kFlagAgg) << 32) | rcarry.v);
      __syncthreads();
    } else if (dg && tid == 0) {
      st_relaxed_u64(D.tiles_b + tile, ((uint64_t)kFlagIncl << 32));
    }

    GC_T(5);
    // ------------------------------------------------------------------ stores
    // tile chunk c = positions 4c..4c+3; positions before the first list start (reset0)
    // get the carry of the earlier tiles
    auto store_chunk = [&](uint32_t c, uint32_t cin, uint32_t reset0) {
      uint4 v = s_out4[sw_chunk(kHalo / 4 + c)];
      if (cin) {
        const uint32_t p = 4 * c;
        if (p < reset0) v.x += cin;
        if (p + 1 < reset0) v.y += cin;
        if (p + 2 < reset0) v.z += cin;
        if (p + 3 < reset0) v.w += cin;
      }
      if (4 * c + 4 <= nvalid) {
        __stcs(reinterpret_cast<uint4*>(out + tT) + c, v);
      } else {
        const uint32_t a4[4] = {v.x, v.y, v.z, v.w};
        for (uint32_t k = 0; k < 4; k++)
          if (4 * c + k < nvalid) out[tT + 4 * c + k] = a4[k];
      }
    };
    auto store_plain = [&](uint32_t c0, uint32_t c1) {  // whole chunks, no carry
      uint4* o4 = reinterpret_cast<uint4*>(out + tT);
#pragma unroll 2
      for (uint32_t c = c0 + tid; c < c1; c += kDT) {
        GC_CHECK(tT + 4 * c + 4 <= D.total_out);
        __stcs(o4 + c, s_out4[sw_chunk(kHalo / 4 + c)]);
      }
    };
    // chunks [c0, nch), no carry: whole 8-row boxes by TMA (lane b of warp 0 issues box b),
    // the rest by 128-bit stores
    auto store_from = [&](uint32_t c0) {
      const uint32_t full = nvalid >> 2;
      const uint32_t b0 = (c0 + kBoxC - 1) / kBoxC, b1 = full / kBoxC;
      if (kTma && use_tma && b1 > b0) {
        if (warp == 0 && lane >= b0 && lane < b1) {
          tma_store_2d(tm, s_out + kHalo + lane * (kBoxC * 4), 0, (int32_t)((tT >> 5) + lane * 8));
          bulk_commit();
        }
        store_plain(c0, b0 * kBoxC);
        store_plain(b1 * kBoxC, full);
      } else {
        store_plain(c0, full);
      }
      for (uint32_t c = max(c0, full) + tid; c < nch; c += kDT) store_chunk(c, 0u, 0u);
    };
    if (dg) {
      const uint32_t reset0 = s_reset0[buf];
#ifdef GC_ABL_NOFLUSH
      const bool need_carry = false;
#else
      const bool need_carry = ok && reset0 != 0u;  // the tile's first int continues a list
#endif
      const uint32_t cfree = need_carry ? min(nch, (reset0 + 3u) / 4u) : 0u;
      store_from(cfree);
      if (need_carry && tid == 0) {
        s_pend.on = 1;
        s_pend.tile = tile;
        s_pend.tT = tT;
        s_pend.nvalid = nvalid;
        s_pend.cfree = cfree;
        s_pend.reset0 = reset0;
        s_pend.f = rcarry.f;
        s_pend.v = rcarry.v;
      }
      GC_T(6);
    } else {
      store_from(0u);
    }
    __syncthreads();  // staging window, bitmap and the next tile's geometry settled
    GC_T(7);
  }
  if (DGAPS && s_pend.on) flush_pending();
  if (kTma && warp == 0) bulk_wait0();  // the TMA stores are done with shared memory
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(&D.hdr->status, err);
}
