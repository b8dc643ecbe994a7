// gc_decode.cuh -- k_decode (subsystems (b)-(d)); included inside namespace gcd by
// gc_kernels.cu.  One CTA decodes one output tile of kT ints: the quadruples containing
// the output positions [t*kT, (t+1)*kT).  All in-tile arithmetic is 32-bit and relative to
// the tile's staged bases.

struct DecodeSmem {
  static constexpr uint32_t kOut = 0;                             // swizzled staging window
  static constexpr uint32_t kDesc = kOut + kOutChunks * 16;       // uint2 per quad of a round
  static constexpr uint32_t kData = kDesc + kRQ * 8;              // data vectors (+1 slack)
  static constexpr uint32_t kCtrl = kData + (kDCap + 1) * 16;     // control words
  static constexpr uint32_t kXinfo = kCtrl + kCCap * 4;           // PFD: exception info per quad
  __host__ __device__ static constexpr uint32_t exc_off() { return kXinfo + kRQ * 4; }
  __host__ __device__ static constexpr uint32_t bytes(bool exc) {
    return exc ? exc_off() + kECap : kXinfo;
  }
};

// In-tile scan state: f = a list starts in the range, q = raw quads of the list, d = data
// lane-bits and e = exception bytes, both relative to the tile's staged bases.
struct St {
  uint32_t f, q, d, e;
};
__device__ __forceinline__ St st_op(const St& a, const St& b) {
  return b.f ? b : St{a.f, a.q + b.q, a.d + b.d, a.e + b.e};
}
template <bool kExc>
__device__ __forceinline__ St block_excl_st(St v, uint32_t* scr, St* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  St inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    St n;
    n.f = __shfl_up_sync(0xffffffffu, inc.f, o);
    n.q = __shfl_up_sync(0xffffffffu, inc.q, o);
    n.d = __shfl_up_sync(0xffffffffu, inc.d, o);
    n.e = kExc ? __shfl_up_sync(0xffffffffu, inc.e, o) : 0u;
    if (lane >= o) inc = st_op(n, inc);
  }
  if (lane == 31) {
    scr[4 * warp + 0] = inc.f;
    scr[4 * warp + 1] = inc.q;
    scr[4 * warp + 2] = inc.d;
    scr[4 * warp + 3] = inc.e;
  }
  __syncthreads();
  St wpre{0, 0, 0, 0}, tot{0, 0, 0, 0};
#pragma unroll
  for (int w = 0; w < kWarps; w++) {
    St s{scr[4 * w], scr[4 * w + 1], scr[4 * w + 2], scr[4 * w + 3]};
    if (w < warp) wpre = st_op(wpre, s);
    tot = st_op(tot, s);
  }
  St ex;
  ex.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
  ex.q = __shfl_up_sync(0xffffffffu, inc.q, 1);
  ex.d = __shfl_up_sync(0xffffffffu, inc.d, 1);
  ex.e = kExc ? __shfl_up_sync(0xffffffffu, inc.e, 1) : 0u;
  if (lane == 0) ex = St{0, 0, 0, 0};
  *total = tot;
  __syncthreads();
  return st_op(wpre, ex);
}

// List cursor with tile-relative fields.
struct TileList {
  uint64_t l, cw_lo, cw_hi;
  uint32_t n, Q;
  uint32_t klo, kend;  // quads of this list owned by the tile: [klo, kend)
  uint32_t oref;       // staging index of quad j's first int = oref + 4j (mod 2^32)
  uint32_t dbase;      // staged data lane-bit of the list's first vector (lists after the first)
  uint32_t ebase;      // staged exception byte of the list's first exception
};

#ifndef GC_DECODE_MINB
#define GC_DECODE_MINB 4
#endif
template <class C, bool DGAPS>
__global__ void __launch_bounds__(kThreads, GC_DECODE_MINB) k_decode(Dev D, uint32_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint4* s_out4 = reinterpret_cast<uint4*>(smem + DecodeSmem::kOut);
  uint32_t* s_out = reinterpret_cast<uint32_t*>(smem + DecodeSmem::kOut);
  uint2* s_desc = reinterpret_cast<uint2*>(smem + DecodeSmem::kDesc);
  uint4* s_data = reinterpret_cast<uint4*>(smem + DecodeSmem::kData);
  uint32_t* s_ctrl = reinterpret_cast<uint32_t*>(smem + DecodeSmem::kCtrl);
  uint32_t* s_xinfo = reinterpret_cast<uint32_t*>(smem + DecodeSmem::kXinfo);
  uint8_t* s_exc = smem + DecodeSmem::exc_off();

  __shared__ Entry s_e0, s_e1;
  __shared__ uint32_t s_scr[kWarps * 4];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t s_tile, s_err, s_carry, s_reset0;

  const int tid = threadIdx.x;
  if (tid == 0) {
    s_tile = atomicAdd(&D.hdr->counter_b, 1u);
    s_err = 0;
    s_carry = 0;
    const uint32_t t = s_tile;
    s_e0 = D.entries[t];
    if (t + 1 < D.n_tiles_b) {
      s_e1 = D.entries[t + 1];
    } else {
      Entry e;
      memset(&e, 0, sizeof(e));
      e.l = (uint32_t)D.n_lists;
      e.valid = 1;
      e.cend = D.ctrl_off[D.n_lists] >> 2;
      e.dend = D.data_off[D.n_lists] * 32ull;
      e.eend = D.exc_off ? D.exc_off[D.n_lists] : 0ull;
      s_e1 = e;
    }
    mbar_init(&s_bar, 1);
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const Entry E0 = s_e0, E1 = s_e1;
  const int64_t base_int = (int64_t)tile * kT - 4;  // global int at staging index 0

  if (!E0.valid || !E1.valid || E1.cend <= E0.gword || E0.l >= D.n_lists) {
    if (tid == 0) {
      atomicOr(&D.hdr->status, (uint32_t)GC_DEV_TRUNCATED);
      if (DGAPS) st_relaxed_u64(D.tiles_b + tile, ((uint64_t)kFlagIncl << 32));
    }
    return;
  }

  // ---- the three stream ranges of this tile -> shared memory (bulk async copies)
  const uint64_t wa = E0.gword, wb = E1.cend;
  const uint64_t cbase = (wa ? wa - 1 : 0) & ~3ull;
  const uint64_t cstop = mn64((wb + 3) & ~3ull, D.n_ctrl_words);
  const bool ctrl_staged = cstop - cbase <= kCCap;
  const uint64_t va = E0.dbeg >> 5;
  const uint64_t vb = mx64(va, mn64((E1.dend + 31) >> 5, D.data_vectors));
  const bool data_staged = vb - va <= kDCap;
  uint64_t ea = 0, eb = 0;
  bool exc_staged = false;
  if (C::kExc) {
    ea = E0.ebeg & ~15ull;
    eb = mx64(ea, mn64((E1.eend + 15) & ~15ull, D.exc_bytes));
    exc_staged = eb - ea <= kECap;
  }
  if (tid == 0) {
    uint32_t bytes = 0;
    if (ctrl_staged && cstop > cbase) bytes += (uint32_t)(cstop - cbase) * 4;
    if (data_staged && vb > va) bytes += (uint32_t)(vb - va) * 16;
    if (C::kExc && exc_staged && eb > ea) bytes += (uint32_t)(eb - ea);
    mbar_expect_tx(&s_bar, bytes);
    if (ctrl_staged && cstop > cbase)
      bulk_g2s(s_ctrl, D.ctrl_words + cbase, (uint32_t)(cstop - cbase) * 4, &s_bar);
    if (data_staged && vb > va) bulk_g2s(s_data, D.data + va, (uint32_t)(vb - va) * 16, &s_bar);
    if (C::kExc && exc_staged && eb > ea) bulk_g2s(s_exc, D.exc + ea, (uint32_t)(eb - ea), &s_bar);
  }
  const uint32_t* cwp = ctrl_staged ? s_ctrl : D.ctrl_words + cbase;  // word w at cwp[w-cbase]
  const uint4* dptr = data_staged ? s_data : D.data + va;
  const uint8_t* eptr = exc_staged ? s_exc : D.exc + ea;
  const uint32_t dlim = (uint32_t)mn64(vb - va, 0x7FFFFFFFull);
  const uint32_t elim = (uint32_t)mn64(eb - ea, 0x7FFFFFFFull);

  // ---- output window
  int64_t out_lo = (int64_t)(D.out_off[E0.l] + 4ull * E0.j);
  int64_t out_hi = E1.l < D.n_lists ? (int64_t)(D.out_off[E1.l] + 4ull * E1.j) : (int64_t)D.total_out;
  {
    int64_t clo = smax64(base_int, 0), chi = smin64(base_int + kOutWords, (int64_t)D.total_out);
    if (out_lo < clo || out_hi > chi || out_hi < out_lo) {
      if (tid == 0) atomicOr(&s_err, (uint32_t)GC_DEV_TRUNCATED);
      out_lo = smax64(out_lo, clo);
      out_hi = smax64(out_lo, smin64(out_hi, chi));
    }
  }
  const uint32_t lo_loc = (uint32_t)(out_lo - base_int), hi_loc = (uint32_t)(out_hi - base_int);
  if (tid == 0) s_reset0 = hi_loc;

  const uint64_t lf = E0.l, ll = E1.l;
  const uint32_t oref_first = lo_loc - 4u * E0.j;
  auto load_list = [&](TileList& L, uint64_t li) {
    L.l = li;
    if (li >= D.n_lists) {
      L.cw_lo = L.cw_hi = ~0ull;
      L.n = L.Q = L.klo = L.kend = 0;
      return;
    }
    L.cw_lo = D.ctrl_off[li] >> 2;
    L.cw_hi = D.ctrl_off[li + 1] >> 2;
    L.n = D.list_n[li];
    L.Q = (L.n + 3) >> 2;
    L.klo = li == lf ? E0.j : 0u;
    L.kend = li == ll ? mn32(L.Q, E1.j) : L.Q;
    L.oref = li == lf ? oref_first : (uint32_t)((int64_t)D.out_off[li] - base_int);
    L.dbase = (uint32_t)(D.data_off[li] * 32ull - va * 32ull);
    L.ebase = C::kExc ? (uint32_t)(D.exc_off[li] - ea) : 0u;
  };
  auto seek = [&](TileList& L, uint64_t w) {
    if (L.l < D.n_lists && w < L.cw_hi) return;
    uint64_t li = L.l;
    while (li < D.n_lists && (D.ctrl_off[li + 1] >> 2) <= w) li++;
    load_list(L, li);
  };

  mbar_wait(&s_bar, 0);
  __syncthreads();

  uint32_t err = 0;
  St carry{1u, E0.wq, (uint32_t)(E0.wd - va * 32ull), (uint32_t)(E0.we - ea)};
  Seg1 rcarry{0u, 0u};  // d-gap running state across rounds
  const uint64_t lsearch_hi = mn64(ll + 1, D.n_lists);

  for (uint64_t r0 = wa; r0 < wb; r0 += kRoundWords) {
    const uint64_t my0 = r0 + (uint64_t)tid * kCB;
    const uint32_t myn = my0 < wb ? (uint32_t)mn64(kCB, wb - my0) : 0u;
    TileList L0;
    load_list(L0, myn ? find_list(D.ctrl_off, lf, lsearch_hi, 4 * my0) : D.n_lists);
    uint32_t wv[kCB], pv[kCB];
#pragma unroll
    for (uint32_t k = 0; k < kCB; k++) {
      uint64_t w = my0 + k;
      wv[k] = (k < myn && w - cbase < cstop - cbase) ? cwp[w - cbase] : 0u;
      pv[k] = (C::kNeedsPrev && k < myn && w > cbase) ? cwp[w - 1 - cbase] : 0u;
    }

    // pass 1: per-word aggregates, segmented scan with the tile carry
    St agg{0, 0, 0, 0};
    {
      TileList L = L0;
#pragma unroll
      for (uint32_t k = 0; k < kCB; k++) {
        if (k >= myn) break;
        uint64_t w = my0 + k;
        seek(L, w);
        if (L.l >= D.n_lists) break;
        WCtx c{wv[k], pv[k], w - L.cw_lo, L.Q};
        WAgg a = C::agg(c);
        if (c.widx == 0 && w != wa)
          agg = St{1u, a.q, L.dbase + a.d, L.ebase + a.e};
        else
          agg = St{agg.f, agg.q + a.q, agg.d + a.d, agg.e + a.e};
      }
    }
    St rtot;
    const St S0 = st_op(carry, block_excl_st<C::kExc>(agg, s_scr, &rtot));
    carry = st_op(carry, rtot);

    // pass 2: quads each word contributes to the tile -> local quad indices
    uint32_t kept = 0;
    {
      TileList L = L0;
      St S = S0;
#pragma unroll
      for (uint32_t k = 0; k < kCB; k++) {
        if (k >= myn) break;
        uint64_t w = my0 + k;
        seek(L, w);
        if (L.l >= D.n_lists) break;
        WCtx c{wv[k], pv[k], w - L.cw_lo, L.Q};
        if (c.widx == 0 && w != wa) S = St{1u, 0u, L.dbase, L.ebase};
        WAgg a = C::agg(c);
        uint32_t qa = max(S.q, L.klo), qb = min(S.q + a.q, L.kend);
        kept += qb > qa ? qb - qa : 0u;
        S.q += a.q;
        S.d += a.d;
        S.e += a.e;
      }
    }
    uint32_t K;
    const uint32_t lq0 = block_excl_sum(kept, s_scr, &K);

    for (uint32_t u = 0; u < K; u += kRQ) {
      // pass 3: per-quad descriptors (position, width, output slot) for quads [u, u+kRQ)
      if (kept) {
        TileList L = L0;
        St S = S0;
        uint32_t x = lq0;
#pragma unroll
        for (uint32_t k = 0; k < kCB; k++) {
          if (k >= myn) break;
          uint64_t w = my0 + k;
          seek(L, w);
          if (L.l >= D.n_lists) break;
          WCtx c{wv[k], pv[k], w - L.cw_lo, L.Q};
          if (c.widx == 0 && w != wa) S = St{1u, 0u, L.dbase, L.ebase};
          WAgg a = C::agg(c);
          const uint32_t qa = max(S.q, L.klo), qb = min(S.q + a.q, L.kend);
          const uint32_t nk = qb > qa ? qb - qa : 0u;
          if (nk && x < u + kRQ && x + nk > u) {
            const St SW = S;
            const uint32_t xw = x;
            C::walk(c, [&](const Grp& g) {
              const uint32_t gq = SW.q + g.q0;
              const uint32_t ja = max(max(gq, qa), qa + (u > xw ? u - xw : 0u));
              const uint32_t jb = min(min(gq + g.nq, qb), qa + (u + kRQ - xw));
              if (ja >= jb) return;
              const uint32_t gd = SW.d + (uint32_t)g.d0;
              uint32_t ei = 0, erank = 0;
              uint32_t pprev = 0;
              const uint32_t qf = C::kExc ? min(g.nq, L.Q - gq) : 0u;
              for (uint32_t j = ja; j < jb; j++) {
                const uint32_t loc = xw + (j - qa) - u;
                const uint32_t pos = gd + (j - gq) * g.step;
                const uint32_t op = L.oref + 4u * j;
                const uint32_t cnt = min(4u, L.n - 4u * j);
                const uint32_t rst = j == 0 ? 1u : 0u;
                if (op + cnt > hi_loc || op < lo_loc) err |= GC_DEV_TRUNCATED;
                s_desc[loc] = make_uint2(pos, g.bw | (min(op, kOutWords - 4) << 6) |
                                                  ((cnt - 1) << 19) | (rst << 21));
                if (DGAPS && rst) atomicMin(&s_reset0, op);
                if (C::kExc) {
                  // exceptions of this quad: positions [4t, 4t+4) of the frame
                  const uint32_t t = j - gq;
                  const uint32_t pb = 4 * g.nq <= 256 ? 1u : 2u;
                  const uint32_t e0 = SW.e + g.e0;
                  uint32_t mask = 0;
                  while (ei < g.cnt) {
                    if (e0 + (ei + 1) * pb > elim) {
                      err |= GC_DEV_TRUNCATED;
                      ei = g.cnt;
                      break;
                    }
                    uint32_t p = eptr[e0 + ei * pb];
                    if (pb == 2) p |= (uint32_t)eptr[e0 + ei * pb + 1] << 8;
                    if (p >= 4 * qf || (ei > 0 && p <= pprev)) {
                      err |= GC_DEV_BAD_EXCEPTION;
                      ei = g.cnt;
                      break;
                    }
                    if (p >= 4 * t + 4) break;
                    pprev = p;
                    if (p >= 4 * t) mask |= 1u << (p - 4 * t);
                    else erank++;
                    ei++;
                  }
                  const uint32_t wbc = g.wb == 1 ? 1u : (g.wb == 2 ? 2u : 3u);
                  s_xinfo[loc] = mask ? (((e0 + g.cnt * pb + erank * g.wb) << 6) | (wbc << 4) | mask)
                                      : 0u;
                  erank += __popc(mask);
                }
              }
            });
          }
          x += nk;
          S.q += a.q;
          S.d += a.d;
          S.e += a.e;
        }
      }
      __syncthreads();

      // unpack 4 consecutive quads per thread: shift/mask over the 4 vertical lanes, the
      // high part of a straddling value from the current vector
      const uint32_t nr = min(kRQ, K - u);
      uint32_t y[16], opq[4], cq[4];
      uint32_t rsts = 0, run = 0, fl = 0;
#pragma unroll
      for (int s = 0; s < 4; s++) {
        const uint32_t qi = 4 * tid + s;
        uint32_t xq[4] = {0, 0, 0, 0};
        uint32_t op = 0, c = 0, rst = 0;
        if (qi < nr) {
          const uint2 dsc = s_desc[qi];
          const uint32_t bw = dsc.y & 63u;
          op = (dsc.y >> 6) & 0x1FFFu;
          c = ((dsc.y >> 19) & 3u) + 1u;
          rst = (dsc.y >> 21) & 1u;
          const uint32_t m = dsc.x >> 5, off = dsc.x & 31u;
          const bool straddle = off + bw > 32;
          if (m < dlim && (!straddle || m + 1 < dlim)) {
            const uint4 v0 = dptr[m];
            const uint4 v1 = straddle ? dptr[m + 1] : make_uint4(0, 0, 0, 0);
            const uint32_t lo = straddle ? off + bw - 32 : 0u;
            const uint32_t mk = mask_bits(bw), ml = (1u << lo) - 1u;
            xq[0] = (((v0.x >> off) << lo) | (v1.x & ml)) & mk;
            xq[1] = (((v0.y >> off) << lo) | (v1.y & ml)) & mk;
            xq[2] = (((v0.z >> off) << lo) | (v1.z & ml)) & mk;
            xq[3] = (((v0.w >> off) << lo) | (v1.w & ml)) & mk;
          } else {
            err |= GC_DEV_TRUNCATED;
          }
          if (C::kExc) {
            const uint32_t xi = s_xinfo[qi];
            if (xi & 15u) {  // Group-PFD: overwrite exception slots before the scan
              const uint32_t wb = 1u << (((xi >> 4) & 3u) - 1u);
              const uint32_t eb0 = xi >> 6;
              if (eb0 + __popc(xi & 15u) * wb > elim) {
                err |= GC_DEV_TRUNCATED;
              } else {
                uint32_t r = 0;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                  if (xi & (1u << k)) {
                    const uint32_t b0 = eb0 + r * wb;
                    uint32_t v = eptr[b0];
                    if (wb > 1) v |= (uint32_t)eptr[b0 + 1] << 8;
                    if (wb > 2) v |= ((uint32_t)eptr[b0 + 2] << 16) | ((uint32_t)eptr[b0 + 3] << 24);
                    xq[k] = v;
                    r++;
                  }
                }
              }
            }
          }
        }
        opq[s] = op;
        cq[s] = c;
        rsts |= rst << s;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t v = (uint32_t)k < c ? xq[k] : 0u;
          if (DGAPS) {
            if (k == 0 && rst) {
              run = v;
              fl = 1;
            } else {
              run += v;
            }
            y[4 * s + k] = run;
          } else {
            y[4 * s + k] = v;
          }
        }
      }
      if (DGAPS) {
        Seg1 rt;
        const Seg1 ex = seg1_op(rcarry, block_excl_seg1(Seg1{fl, run}, reinterpret_cast<Seg1*>(s_scr), &rt));
        rcarry = seg1_op(rcarry, rt);
        // values before this thread's first list start continue the running prefix
        bool seen = false;
#pragma unroll
        for (int s = 0; s < 4; s++) {
          if ((rsts >> s) & 1u) seen = true;
#pragma unroll
          for (int k = 0; k < 4; k++)
            if (!seen) y[4 * s + k] += ex.v;
        }
      }
#pragma unroll
      for (int s = 0; s < 4; s++) {
#pragma unroll
        for (int k = 0; k < 4; k++)
          if ((uint32_t)k < cq[s]) s_out[sw_word(opq[s] + k)] = y[4 * s + k];
      }
      __syncthreads();
    }
  }

  // ---- d-gap look-back across tiles (segmented by list)
  if (DGAPS) {
    if (tid < 32) {
      const bool need_carry = E0.j > 0;  // the tile's first quad continues a list
      if (tid == 0)
        st_relaxed_u64(D.tiles_b + tile, ((uint64_t)((rcarry.f || !need_carry) ? kFlagIncl : kFlagAgg)
                                          << 32) | rcarry.v);
      uint32_t cin = 0;
      if (need_carry) {
        cin = lookback_u32(D.tiles_b, tile);
        if (tid == 0 && !rcarry.f)
          st_relaxed_u64(D.tiles_b + tile, ((uint64_t)kFlagIncl << 32) | (cin + rcarry.v));
      }
      if (tid == 0) s_carry = cin;
    }
    __syncthreads();
  }

  // ---- coalesced 128-bit store of [out_lo, out_hi); the tile's first list segment
  // (before the first list start) gets the carry from the look-back
  {
    const uint32_t cin = DGAPS ? s_carry : 0u;
    const uint32_t r0loc = DGAPS ? s_reset0 : 0u;
    const int64_t c_lo = out_lo >> 2, c_hi = (out_hi + 3) >> 2;
    const int64_t cb = base_int / 4;
    for (int64_t c = c_lo + tid; c < c_hi; c += kThreads) {
      const uint32_t lc = (uint32_t)(c - cb);
      uint4 v = s_out4[sw_chunk(lc)];
      if (DGAPS && cin) {
        const uint32_t p = 4 * lc;
        if (p + 0 < r0loc) v.x += cin;
        if (p + 1 < r0loc) v.y += cin;
        if (p + 2 < r0loc) v.z += cin;
        if (p + 3 < r0loc) v.w += cin;
      }
      const int64_t g = 4 * c;
      if (g >= out_lo && g + 4 <= out_hi) {
        __stcs(reinterpret_cast<uint4*>(out + g), v);
      } else {
        const uint32_t a[4] = {v.x, v.y, v.z, v.w};
        for (int k = 0; k < 4; k++)
          if (g + k >= out_lo && g + k < out_hi) out[g + k] = a[k];
      }
    }
  }
  if (err) atomicOr(&s_err, err);
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(&D.hdr->status, s_err);
}
