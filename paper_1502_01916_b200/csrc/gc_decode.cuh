// gc_decode.cuh -- k_decode (subsystems (b)-(d)); included inside namespace gcd by
// gc_kernels.cu.
//
// Persistent warps.  A warp repeatedly claims an output warp-tile t (atomic counter, so
// tiles start in order and the decoupled look-back always makes progress) and decodes the
// quadruples containing the output positions [t*kT, (t+1)*kT) with warp-shuffle scans
// only: no block barriers.  In-tile arithmetic is 32-bit and relative to the tile's staged
// bases; the tile's lists live in a per-warp shared-memory table.

struct WarpSmem {  // per-warp shared memory, byte offsets
  static constexpr uint32_t kOut = 0;                            // swizzled staging window
  static constexpr uint32_t kDesc = kOut + kOutChunks * 16;      // uint2 per quad of a window
  static constexpr uint32_t kData = kDesc + kRQ * 8;             // data vectors (+1 slack)
  static constexpr uint32_t kCtrl = kData + (kDCap + 1) * 16;    // control words
  static constexpr uint32_t kLt = kCtrl + kCCap * 4;             // list table (SoA)
  static constexpr uint32_t kLtFields = 9;
  static constexpr uint32_t kEnt = (kLt + kLtFields * (kLT + 1) * 4 + 15) & ~15u;  // 2 Entries
  static constexpr uint32_t kXinfo = kEnt + 2 * sizeof(Entry);   // PFD per-quad info
  __host__ __device__ static constexpr uint32_t exc_off() { return (kXinfo + kRQ * 4 + 15) & ~15u; }
  __host__ __device__ static constexpr uint32_t bytes(bool exc) {
    return exc ? ((exc_off() + kECap + 127) & ~127u) : ((kXinfo + 127) & ~127u);
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
// Warp-wide exclusive segmented scan; *total = the warp aggregate.
template <bool kExc>
__device__ __forceinline__ St warp_excl_st(St v, St* total) {
  const int lane = threadIdx.x & 31;
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
  total->f = __shfl_sync(0xffffffffu, inc.f, 31);
  total->q = __shfl_sync(0xffffffffu, inc.q, 31);
  total->d = __shfl_sync(0xffffffffu, inc.d, 31);
  total->e = kExc ? __shfl_sync(0xffffffffu, inc.e, 31) : 0u;
  St ex;
  ex.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
  ex.q = __shfl_up_sync(0xffffffffu, inc.q, 1);
  ex.d = __shfl_up_sync(0xffffffffu, inc.d, 1);
  ex.e = kExc ? __shfl_up_sync(0xffffffffu, inc.e, 1) : 0u;
  if (lane == 0) ex = St{0, 0, 0, 0};
  return ex;
}
__device__ __forceinline__ uint32_t warp_excl_sum(uint32_t v, uint32_t* total) {
  const int lane = threadIdx.x & 31;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  *total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}
__device__ __forceinline__ Seg1 warp_excl_seg1(Seg1 x, Seg1* total) {
  const int lane = threadIdx.x & 31;
  Seg1 inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg1 n;
    n.f = __shfl_up_sync(0xffffffffu, inc.f, o);
    n.v = __shfl_up_sync(0xffffffffu, inc.v, o);
    if (lane >= o) inc = seg1_op(n, inc);
  }
  total->f = __shfl_sync(0xffffffffu, inc.f, 31);
  total->v = __shfl_sync(0xffffffffu, inc.v, 31);
  Seg1 ex;
  ex.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
  ex.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
  if (lane == 0) ex = Seg1{0, 0};
  return ex;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

#ifndef GC_DECODE_MINB
#define GC_DECODE_MINB 2
#endif
template <class C, bool DGAPS, int kWPC>
__global__ void __launch_bounds__(32 * kWPC, GC_DECODE_MINB) k_decode(Dev D, uint32_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem_all[];
  __shared__ __align__(8) uint64_t s_bar[kWPC];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* smem = smem_all + wid * WarpSmem::bytes(C::kExc);
  uint4* s_out4 = reinterpret_cast<uint4*>(smem + WarpSmem::kOut);
  uint32_t* s_out = reinterpret_cast<uint32_t*>(smem + WarpSmem::kOut);
  uint2* s_desc = reinterpret_cast<uint2*>(smem + WarpSmem::kDesc);
  uint4* s_data = reinterpret_cast<uint4*>(smem + WarpSmem::kData);
  uint32_t* s_ctrl = reinterpret_cast<uint32_t*>(smem + WarpSmem::kCtrl);
  uint32_t* s_lt = reinterpret_cast<uint32_t*>(smem + WarpSmem::kLt);
  uint32_t* lt_cw = s_lt + 0 * (kLT + 1);     // first control word (relative to cbase)
  uint32_t* lt_q = s_lt + 1 * (kLT + 1);      // quads
  uint32_t* lt_n = s_lt + 2 * (kLT + 1);      // ints
  uint32_t* lt_klo = s_lt + 3 * (kLT + 1);    // first quad owned by the tile
  uint32_t* lt_kend = s_lt + 4 * (kLT + 1);   // one past the last
  uint32_t* lt_oref = s_lt + 5 * (kLT + 1);   // staging index of quad j = oref + 4j
  uint32_t* lt_db = s_lt + 6 * (kLT + 1);     // staged data lane-bit of the list start
  uint32_t* lt_eb = s_lt + 7 * (kLT + 1);     // staged exception byte of the list start
  uint32_t* lt_lb = s_lt + 8 * (kLT + 1);     // local index of quad klo within the round
  uint32_t* s_ent = reinterpret_cast<uint32_t*>(smem + WarpSmem::kEnt);
  uint32_t* s_xinfo = reinterpret_cast<uint32_t*>(smem + WarpSmem::kXinfo);
  uint8_t* s_exc = smem + WarpSmem::exc_off();
  uint64_t* bar = &s_bar[wid];
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  uint32_t phase = 0;
  uint32_t err = 0;

  // 128-bit store of staging chunk c (the 16-B output block 4c..4c+3 clipped to [lo, hi));
  // ints before staging index r0 get the look-back carry cin
  auto store_chunk = [&](int64_t c, int64_t cb, int64_t lo, int64_t hi, uint32_t cin, uint32_t r0) {
    const uint32_t lc = (uint32_t)(c - cb);
    uint4 v = s_out4[sw_chunk(lc)];
    if (cin) {
      const uint32_t p = 4 * lc;
      if (p < r0) v.x += cin;
      if (p + 1 < r0) v.y += cin;
      if (p + 2 < r0) v.z += cin;
      if (p + 3 < r0) v.w += cin;
    }
    const int64_t g = 4 * c;
    if (g >= lo && g + 4 <= hi) {
      __stcs(reinterpret_cast<uint4*>(out + g), v);
    } else {
      const uint32_t a4[4] = {v.x, v.y, v.z, v.w};
      for (int k = 0; k < 4; k++)
        if (g + k >= lo && g + k < hi) out[g + k] = a4[k];
    }
  };
  // A tile whose first list segment needs the carry of earlier tiles is finished only after
  // this warp has claimed and set up its next tile, so the look-back wait overlaps that
  // tile's bulk copies (its staging window is not touched before then).
  bool pd_on = false;
  uint32_t pd_tile = 0, pd_reset0 = 0, pd_f = 0, pd_v = 0;
  int64_t pd_lo = 0, pd_hi = 0, pd_clo = 0, pd_cmid = 0, pd_cb = 0;
  auto finish_pending = [&]() {
    if (!pd_on) return;
    const uint32_t cin = lookback_u32(D.tiles_b, pd_tile);
    if (lane == 0 && !pd_f)
      st_relaxed_u64(D.tiles_b + pd_tile, ((uint64_t)kFlagIncl << 32) | (cin + pd_v));
    for (int64_t c = pd_clo + lane; c < pd_cmid; c += 32) store_chunk(c, pd_cb, pd_lo, pd_hi, cin, pd_reset0);
    pd_on = false;
    __syncwarp();
  };

  while (true) {
    // ---------------------------------------------------------------- claim a tile
    uint32_t tile = 0;
    if (lane == 0) tile = atomicAdd(&D.hdr->counter_b, 1u);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= D.n_tiles_b) {
      finish_pending();
      break;
    }
    // the two boundary Entries (80 B each) -> shared, 20 lanes x 2 words
    {
      const uint32_t* e0p = reinterpret_cast<const uint32_t*>(D.entries + tile);
      if (lane < 20) {
        s_ent[lane] = e0p[lane];
        if (tile + 1 < D.n_tiles_b) s_ent[20 + lane] = e0p[20 + lane];
      }
      __syncwarp();
    }
    const Entry& E0 = *reinterpret_cast<const Entry*>(s_ent);
    Entry E1;
    if (tile + 1 < D.n_tiles_b) {
      E1 = *reinterpret_cast<const Entry*>(s_ent + 20);
    } else {
      E1.l = (uint32_t)D.n_lists;
      E1.j = 0;
      E1.valid = 1;
      E1.cend = D.ctrl_off[D.n_lists] >> 2;
      E1.dend = D.data_off[D.n_lists] * 32ull;
      E1.eend = D.exc_off ? D.exc_off[D.n_lists] : 0ull;
    }
    const int64_t base_int = (int64_t)tile * kT - 4;  // global int at staging index 0
    if (!(E0.valid && E1.valid && E1.cend > E0.gword && E0.l < D.n_lists)) {
      if (lane == 0) {
        atomicOr(&D.hdr->status, (uint32_t)GC_DEV_TRUNCATED);
        if (DGAPS) st_relaxed_u64(D.tiles_b + tile, ((uint64_t)kFlagIncl << 32));
      }
      __syncwarp();
      continue;
    }
    // ---------------------------------------------------------------- stream ranges
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
    if (lane == 0) {
      uint32_t bytes = 0;
      if (ctrl_staged && cstop > cbase) bytes += (uint32_t)(cstop - cbase) * 4;
      if (data_staged && vb > va) bytes += (uint32_t)(vb - va) * 16;
      if (C::kExc && exc_staged && eb > ea) bytes += (uint32_t)(eb - ea);
      fence_proxy_async_smem();
      mbar_expect_tx(bar, bytes);
      if (ctrl_staged && cstop > cbase)
        bulk_g2s(s_ctrl, D.ctrl_words + cbase, (uint32_t)(cstop - cbase) * 4, bar);
      if (data_staged && vb > va) bulk_g2s(s_data, D.data + va, (uint32_t)(vb - va) * 16, bar);
      if (C::kExc && exc_staged && eb > ea) bulk_g2s(s_exc, D.exc + ea, (uint32_t)(eb - ea), bar);
    }
    finish_pending();  // the previous tile's look-back, now that this tile's copies are in flight
    const uint32_t ncw = (uint32_t)(cstop - cbase);
    const uint32_t* cwp = ctrl_staged ? s_ctrl : D.ctrl_words + cbase;  // word w at cwp[w-cbase]
    const uint4* dptr = data_staged ? s_data : D.data + va;
    const uint8_t* eptr = exc_staged ? s_exc : D.exc + ea;
    const uint32_t dlim = (uint32_t)mn64(vb - va, 0x7FFFFFFFull);
    const uint32_t elim = (uint32_t)mn64(eb - ea, 0x7FFFFFFFull);

    // ---------------------------------------------------------------- output window
    int64_t out_lo = (int64_t)(D.out_off[E0.l] + 4ull * E0.j);
    int64_t out_hi = E1.l < D.n_lists ? (int64_t)(D.out_off[E1.l] + 4ull * E1.j) : (int64_t)D.total_out;
    {
      const int64_t clo = smax64(base_int, 0);
      const int64_t chi = smin64(base_int + kOutWords, (int64_t)D.total_out);
      if (out_lo < clo || out_hi > chi || out_hi < out_lo) {
        err |= GC_DEV_TRUNCATED;
        out_lo = smax64(out_lo, clo);
        out_hi = smax64(out_lo, smin64(out_hi, chi));
      }
    }
    const uint32_t lo_loc = (uint32_t)(out_lo - base_int), hi_loc = (uint32_t)(out_hi - base_int);
    const uint64_t lf = E0.l, ll = E1.l;
    const uint32_t j0 = E0.j, j1 = E1.j;
    const uint64_t lend = j1 > 0 && ll < D.n_lists ? ll + 1 : ll;
    const uint32_t nlists = (uint32_t)(lend - lf);
    const St carry0{1u, E0.wq, (uint32_t)(E0.wd - va * 32ull), (uint32_t)(E0.we - ea)};
    __syncwarp();  // everyone has read s_ent

    Seg1 rcarry{0u, 0u};  // d-gap running state across windows
    uint32_t reset0 = hi_loc;  // staging index of the tile's first list start
    bool waited = false;

    for (uint32_t lr = 0; lr < nlists; lr += kLT) {
      // ---------------------------------------------------------------- list table
      const uint32_t cnt = min(kLT, nlists - lr);
      uint32_t kept = 0;
      {
        const uint64_t l = lf + lr + lane;
        if (lane <= cnt) lt_cw[lane] = (uint32_t)((D.ctrl_off[mn64(l, D.n_lists)] >> 2) - cbase);
        if (lane == 0 && cnt == 32) lt_cw[32] = (uint32_t)((D.ctrl_off[mn64(l + 32, D.n_lists)] >> 2) - cbase);
        if (lane < cnt) {
          const uint32_t n = D.list_n[l];
          const uint32_t Q = (n + 3) >> 2;
          const uint32_t klo = l == lf ? j0 : 0u;
          const uint32_t kend = l == ll ? min(Q, j1) : Q;
          lt_q[lane] = Q;
          lt_n[lane] = n;
          lt_klo[lane] = klo;
          lt_kend[lane] = kend;
          lt_oref[lane] = l == lf ? lo_loc - 4u * j0 : (uint32_t)((int64_t)D.out_off[l] - base_int);
          lt_db[lane] = (uint32_t)(D.data_off[l] * 32ull - va * 32ull);
          lt_eb[lane] = C::kExc ? (uint32_t)(D.exc_off[l] - ea) : 0u;
          kept = kend > klo ? kend - klo : 0u;
        }
      }
      uint32_t K;
      const uint32_t lbk = warp_excl_sum(kept, &K);
      if (lane < cnt) lt_lb[lane] = lbk;
      if (!waited) {
        mbar_wait(bar, phase);
        waited = true;
      }
      __syncwarp();

      const uint64_t rw0 = lr == 0 ? wa : cbase + lt_cw[0];
      const uint64_t rw1 = mn64(wb, cbase + lt_cw[cnt]);

      for (uint32_t u = 0; u < K; u += kRQ) {
        St carry = carry0;
        // control units (a word, or a kParts-th of one) in rounds of 32 x kCBW
        constexpr uint32_t P = C::kParts;
        const uint64_t ru0 = rw0 * P, ru1 = rw1 * P;
        for (uint64_t r0 = ru0; r0 < ru1; r0 += kRoundWords) {
          const uint64_t my0 = r0 + (uint64_t)lane * kCBW;
          const uint32_t myn = my0 < ru1 ? (uint32_t)mn64(kCBW, ru1 - my0) : 0u;
          uint32_t li = 0;
          if (myn) {  // the last table entry whose first word is <= my first word
            const uint32_t key = (uint32_t)(my0 / P - cbase);
            uint32_t a = 0, b = cnt;
            while (b - a > 1) {
              const uint32_t m = (a + b) >> 1;
              if (lt_cw[m] <= key) a = m;
              else b = m;
            }
            li = a;
          }
          uint32_t wv[kCBW], pv[kCBW], wl[kCBW];
          St agg{0, 0, 0, 0};
#pragma unroll
          for (uint32_t k = 0; k < kCBW; k++) {
            const uint64_t un = my0 + k;
            const uint64_t w = un / P;
            const uint32_t part = (uint32_t)(un % P);
            const uint32_t wr = (uint32_t)(w - cbase);
            wv[k] = pv[k] = wl[k] = 0;
            if (k < myn) {
              while (li + 1 < cnt && lt_cw[li + 1] <= wr) li++;
              wl[k] = li;
              wv[k] = wr < ncw ? cwp[wr] : 0u;
              pv[k] = (C::kNeedsPrev && wr >= 1 && wr - 1 < ncw) ? cwp[wr - 1] : 0u;
              const uint32_t widx = wr - lt_cw[li];
              const WCtx c{wv[k], pv[k], widx, lt_q[li], part};
              const WAgg a = C::agg(c);
              agg = (widx == 0 && part == 0 && w != wa)
                        ? St{1u, a.q, lt_db[li] + a.d, lt_eb[li] + a.e}
                        : St{agg.f, agg.q + a.q, agg.d + a.d, agg.e + a.e};
            }
          }
          St rtot;
          St S = st_op(carry, warp_excl_st<C::kExc>(agg, &rtot));
          carry = st_op(carry, rtot);

          // per-quad descriptors (position, width, staging slot) of the window's quads
#pragma unroll
          for (uint32_t k = 0; k < kCBW; k++) {
            if (k >= myn) break;
            const uint64_t un = my0 + k;
            const uint64_t w = un / P;
            const uint32_t part = (uint32_t)(un % P);
            const uint32_t wr = (uint32_t)(w - cbase);
            const uint32_t i = wl[k];
            const uint32_t widx = wr - lt_cw[i];
            const WCtx c{wv[k], pv[k], widx, lt_q[i], part};
            if (widx == 0 && part == 0 && w != wa) S = St{1u, 0u, lt_db[i], lt_eb[i]};
            const WAgg a = C::agg(c);
            const uint32_t klo = lt_klo[i], kend = lt_kend[i];
            const uint32_t qa = max(S.q, klo), qb = min(S.q + a.q, kend);
            const uint32_t x0 = lt_lb[i] + (qa - klo);  // local index of quad qa
            if (!(qb > qa && x0 < u + kRQ && x0 + (qb - qa) > u)) {
            } else if constexpr (!C::kMultiQuad) {
              // one quad per group: tight codec loop straight into the descriptors
              const uint32_t ja = qa + (u > x0 ? u - x0 : 0u);
              const uint32_t jb = min(qb, qa + (u + kRQ - x0));
              const uint32_t n = lt_n[i], oref = lt_oref[i];
              const uint32_t lbase = x0 - qa - u;  // descriptor slot of quad j = lbase + j
              C::emit(c, S.q, S.d, ja, jb, [&](uint32_t j, uint32_t pos, uint32_t bw) {
                const uint32_t op = oref + 4u * j;
                const uint32_t cq = min(4u, n - 4u * j);
                const uint32_t rst = j == 0 ? 1u : 0u;
                s_desc[lbase + j] = make_uint2(pos, bw | (op << 6) | ((cq - 1) << 19) | (rst << 21));
                if (DGAPS && rst) reset0 = min(reset0, op);
              });
            } else {
              const St SW = S;
              const uint32_t n = lt_n[i], oref = lt_oref[i], Qi = lt_q[i];
              C::walk(c, [&](const Grp& g) {
                const uint32_t gq = SW.q + g.q0;
                const uint32_t ja = max(max(gq, qa), qa + (u > x0 ? u - x0 : 0u));
                const uint32_t jb = min(min(gq + g.nq, qb), qa + (u + kRQ - x0));
                if (ja >= jb) return;
                const uint32_t gd = SW.d + (uint32_t)g.d0;
                uint32_t ei = 0, erank = 0, pprev = 0;
                const uint32_t qf = C::kExc ? min(g.nq, Qi - gq) : 0u;
                for (uint32_t j = ja; j < jb; j++) {
                  const uint32_t loc = x0 + (j - qa) - u;
                  const uint32_t op = oref + 4u * j;
                  const uint32_t cq = min(4u, n - 4u * j);
                  const uint32_t rst = j == 0 ? 1u : 0u;
                  if (op + cq > hi_loc || op < lo_loc) err |= GC_DEV_TRUNCATED;
                  s_desc[loc] = make_uint2(gd + (j - gq) * g.step,
                                           g.bw | (min(op, kOutWords - 4) << 6) |
                                               ((cq - 1) << 19) | (rst << 21));
                  if (DGAPS && rst) reset0 = min(reset0, op);
                  if (C::kExc) {
                    // exceptions of this quad: frame positions [4t, 4t+4)
                    const uint32_t t4 = 4 * (j - gq);
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
                      if (p >= t4 + 4) break;
                      pprev = p;
                      if (p >= t4) mask |= 1u << (p - t4);
                      else erank++;
                      ei++;
                    }
                    const uint32_t wbc = g.wb == 1 ? 1u : (g.wb == 2 ? 2u : 3u);
                    s_xinfo[loc] =
                        mask ? (((e0 + g.cnt * pb + erank * g.wb) << 6) | (wbc << 4) | mask) : 0u;
                    erank += __popc(mask);
                  }
                }
              });
            }
            S.q += a.q;
            S.d += a.d;
            S.e += a.e;
          }
        }
        __syncwarp();

        // ---------------------------------------------------------------- unpack + d-gap scan
        // kQPL consecutive quads per lane: shift/mask over the 4 vertical lanes, the high
        // part of a straddling value from the current vector
        const uint32_t nr = min(kRQ, K - u);
        uint32_t y[4 * kQPL], opq[kQPL], cqs = 0, rsts = 0;
        uint32_t run = 0, fl = 0;
#pragma unroll
        for (uint32_t s = 0; s < kQPL; s++) {
          const uint32_t qi = kQPL * lane + s;
          uint32_t xq[4] = {0, 0, 0, 0};
          uint32_t op = 0, c = 0, rst = 0;
          if (qi < nr) {
            const uint2 dsc = s_desc[qi];
            const uint32_t bw = dsc.y & 63u;
            op = min((dsc.y >> 6) & 0x1FFFu, kOutWords - 4);
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
          cqs |= c << (3 * s);
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
          const Seg1 ex = seg1_op(rcarry, warp_excl_seg1(Seg1{fl, run}, &rt));
          rcarry = seg1_op(rcarry, rt);
          bool seen = false;  // values before this lane's first list start continue the prefix
#pragma unroll
          for (uint32_t s = 0; s < kQPL; s++) {
            if ((rsts >> s) & 1u) seen = true;
#pragma unroll
            for (int k = 0; k < 4; k++)
              if (!seen) y[4 * s + k] += ex.v;
          }
        }
#pragma unroll
        for (uint32_t s = 0; s < kQPL; s++) {
          const uint32_t c = (cqs >> (3 * s)) & 7u;
          const uint32_t op = opq[s];
          if (c == 4 && (op & 3u) == 0) {
            s_out4[sw_chunk(op >> 2)] = make_uint4(y[4 * s], y[4 * s + 1], y[4 * s + 2], y[4 * s + 3]);
          } else {
#pragma unroll
            for (int k = 0; k < 4; k++)
              if ((uint32_t)k < c) s_out[sw_word(op + k)] = y[4 * s + k];
          }
        }
        __syncwarp();
      }
    }
    if (!waited) mbar_wait(bar, phase);
    phase ^= 1u;

    // ---------------------------------------------------------------- publish + store
    // publish the tile aggregate and store every chunk that needs no carry; the first list
    // segment (before the tile's first list start) waits for the look-back
    const int64_t c_lo = out_lo >> 2, c_hi = (out_hi + 3) >> 2;
    const int64_t cb = base_int / 4;
    const bool need_carry = DGAPS && j0 > 0;  // the tile's first quad continues a list
    if (DGAPS) {
      reset0 = __reduce_min_sync(0xffffffffu, reset0);
      if (lane == 0)
        st_relaxed_u64(D.tiles_b + tile,
                       ((uint64_t)((rcarry.f || !need_carry) ? kFlagIncl : kFlagAgg) << 32) |
                           rcarry.v);
    }
    const int64_t c_mid =
        need_carry ? smin64(c_hi, smax64(c_lo, (base_int + (int64_t)reset0 + 3) >> 2)) : c_lo;
    for (int64_t c = c_mid + lane; c < c_hi; c += 32) store_chunk(c, cb, out_lo, out_hi, 0u, 0u);
    if (need_carry) {
      pd_on = true;
      pd_tile = tile;
      pd_reset0 = reset0;
      pd_f = rcarry.f;
      pd_v = rcarry.v;
      pd_lo = out_lo;
      pd_hi = out_hi;
      pd_clo = c_lo;
      pd_cmid = c_mid;
      pd_cb = cb;
    }
    __syncwarp();
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) atomicOr(&D.hdr->status, err);
}
