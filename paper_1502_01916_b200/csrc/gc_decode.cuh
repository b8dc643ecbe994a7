// gc_decode.cuh -- k_decode (subsystems (b)-(d)); included inside namespace gcd by
// gc_kernels.cu.  One CTA decodes one output tile of kT ints: the quadruples containing
// the output positions [t*kT, (t+1)*kT).  In-tile arithmetic is 32-bit and relative to the
// tile's staged bases; the tile's lists live in a shared-memory table.

struct DecodeSmem {
  static constexpr uint32_t kOut = 0;                             // swizzled staging window
  static constexpr uint32_t kDesc = kOut + kOutChunks * 16;       // uint2 per quad of a window
  static constexpr uint32_t kData = kDesc + kRQ * 8;              // data vectors (+1 slack)
  static constexpr uint32_t kCtrl = kData + (kDCap + 1) * 16;     // control words
  static constexpr uint32_t kLt = kCtrl + kCCap * 4;              // list table (SoA)
  static constexpr uint32_t kLtFields = 9;
  static constexpr uint32_t kXinfo = (kLt + kLtFields * (kLT + 1) * 4 + 15) & ~15u;  // PFD info
  __host__ __device__ static constexpr uint32_t exc_off() { return (kXinfo + kRQ * 4 + 15) & ~15u; }
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

struct TileInfo {
  uint64_t wa, wb, cbase, cstop, va, vb, ea, eb, lf, ll;
  int64_t out_lo, out_hi;
  uint64_t wd0, we0;
  uint32_t lo_loc, hi_loc, dlim, elim, j0, j1, wq0, nlists;
  uint32_t ctrl_staged, data_staged, exc_staged, ok;
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
  uint32_t* s_lt = reinterpret_cast<uint32_t*>(smem + DecodeSmem::kLt);
  uint32_t* lt_cw = s_lt + 0 * (kLT + 1);     // first control word (relative to cbase)
  uint32_t* lt_q = s_lt + 1 * (kLT + 1);      // quads
  uint32_t* lt_n = s_lt + 2 * (kLT + 1);      // ints
  uint32_t* lt_klo = s_lt + 3 * (kLT + 1);    // first quad owned by the tile
  uint32_t* lt_kend = s_lt + 4 * (kLT + 1);   // one past the last
  uint32_t* lt_oref = s_lt + 5 * (kLT + 1);   // staging index of quad j = oref + 4j
  uint32_t* lt_db = s_lt + 6 * (kLT + 1);     // staged data lane-bit of the list start
  uint32_t* lt_eb = s_lt + 7 * (kLT + 1);     // staged exception byte of the list start
  uint32_t* lt_lb = s_lt + 8 * (kLT + 1);     // local index of quad klo within the round
  uint32_t* s_xinfo = reinterpret_cast<uint32_t*>(smem + DecodeSmem::kXinfo);
  uint8_t* s_exc = smem + DecodeSmem::exc_off();

  __shared__ TileInfo s_ti;
  __shared__ uint32_t s_scr[kWarps * 4];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t s_tile, s_err, s_carry, s_reset0;

  const int tid = threadIdx.x;
  // ---------------------------------------------------------------- tile setup (thread 0)
  if (tid == 0) {
    const uint32_t t = atomicAdd(&D.hdr->counter_b, 1u);
    s_tile = t;
    s_err = 0;
    s_carry = 0;
    TileInfo ti;
    const Entry E0 = D.entries[t];
    Entry E1;
    if (t + 1 < D.n_tiles_b) {
      E1 = D.entries[t + 1];
    } else {
      E1.l = (uint32_t)D.n_lists;
      E1.j = 0;
      E1.valid = 1;
      E1.cend = D.ctrl_off[D.n_lists] >> 2;
      E1.dend = D.data_off[D.n_lists] * 32ull;
      E1.eend = D.exc_off ? D.exc_off[D.n_lists] : 0ull;
    }
    ti.ok = E0.valid && E1.valid && E1.cend > E0.gword && E0.l < D.n_lists;
    if (ti.ok) {
      const int64_t base_int = (int64_t)t * kT - 4;
      ti.wa = E0.gword;
      ti.wb = E1.cend;
      ti.cbase = (ti.wa ? ti.wa - 1 : 0) & ~3ull;
      ti.cstop = mn64((ti.wb + 3) & ~3ull, D.n_ctrl_words);
      ti.ctrl_staged = ti.cstop - ti.cbase <= kCCap;
      ti.va = E0.dbeg >> 5;
      ti.vb = mx64(ti.va, mn64((E1.dend + 31) >> 5, D.data_vectors));
      ti.data_staged = ti.vb - ti.va <= kDCap;
      ti.ea = ti.eb = 0;
      ti.exc_staged = 0;
      if (C::kExc) {
        ti.ea = E0.ebeg & ~15ull;
        ti.eb = mx64(ti.ea, mn64((E1.eend + 15) & ~15ull, D.exc_bytes));
        ti.exc_staged = ti.eb - ti.ea <= kECap;
      }
      ti.dlim = (uint32_t)mn64(ti.vb - ti.va, 0x7FFFFFFFull);
      ti.elim = (uint32_t)mn64(ti.eb - ti.ea, 0x7FFFFFFFull);
      uint32_t bytes = 0;
      if (ti.ctrl_staged && ti.cstop > ti.cbase) bytes += (uint32_t)(ti.cstop - ti.cbase) * 4;
      if (ti.data_staged && ti.vb > ti.va) bytes += (uint32_t)(ti.vb - ti.va) * 16;
      if (C::kExc && ti.exc_staged && ti.eb > ti.ea) bytes += (uint32_t)(ti.eb - ti.ea);
      mbar_init(&s_bar, 1);
      mbar_expect_tx(&s_bar, bytes);
      if (ti.ctrl_staged && ti.cstop > ti.cbase)
        bulk_g2s(s_ctrl, D.ctrl_words + ti.cbase, (uint32_t)(ti.cstop - ti.cbase) * 4, &s_bar);
      if (ti.data_staged && ti.vb > ti.va)
        bulk_g2s(s_data, D.data + ti.va, (uint32_t)(ti.vb - ti.va) * 16, &s_bar);
      if (C::kExc && ti.exc_staged && ti.eb > ti.ea)
        bulk_g2s(s_exc, D.exc + ti.ea, (uint32_t)(ti.eb - ti.ea), &s_bar);
      int64_t out_lo = (int64_t)(D.out_off[E0.l] + 4ull * E0.j);
      int64_t out_hi =
          E1.l < D.n_lists ? (int64_t)(D.out_off[E1.l] + 4ull * E1.j) : (int64_t)D.total_out;
      const int64_t clo = smax64(base_int, 0);
      const int64_t chi = smin64(base_int + kOutWords, (int64_t)D.total_out);
      if (out_lo < clo || out_hi > chi || out_hi < out_lo) {
        s_err = GC_DEV_TRUNCATED;
        out_lo = smax64(out_lo, clo);
        out_hi = smax64(out_lo, smin64(out_hi, chi));
      }
      ti.out_lo = out_lo;
      ti.out_hi = out_hi;
      ti.lo_loc = (uint32_t)(out_lo - base_int);
      ti.hi_loc = (uint32_t)(out_hi - base_int);
      ti.lf = E0.l;
      ti.ll = E1.l;
      ti.j0 = E0.j;
      ti.j1 = E1.j;
      ti.wq0 = E0.wq;
      ti.wd0 = E0.wd;
      ti.we0 = E0.we;
      const uint64_t lend = E1.j > 0 && E1.l < D.n_lists ? (uint64_t)E1.l + 1 : (uint64_t)E1.l;
      ti.nlists = (uint32_t)(lend - E0.l);
      s_reset0 = ti.hi_loc;
    } else {
      atomicOr(&D.hdr->status, (uint32_t)GC_DEV_TRUNCATED);
      if (DGAPS) st_relaxed_u64(D.tiles_b + t, ((uint64_t)kFlagIncl << 32));
    }
    s_ti = ti;
  }
  __syncthreads();
  if (!s_ti.ok) return;
  const uint32_t tile = s_tile;
  const int64_t base_int = (int64_t)tile * kT - 4;
  const uint64_t wa = s_ti.wa, wb = s_ti.wb, cbase = s_ti.cbase;
  const uint64_t va = s_ti.va, ea = s_ti.ea;
  const uint32_t dlim = s_ti.dlim, elim = s_ti.elim;
  const uint32_t lo_loc = s_ti.lo_loc, hi_loc = s_ti.hi_loc;
  const uint32_t ncw = (uint32_t)(s_ti.cstop - cbase);
  const uint32_t* cwp = s_ti.ctrl_staged ? s_ctrl : D.ctrl_words + cbase;  // word w: cwp[w-cbase]
  const uint4* dptr = s_ti.data_staged ? s_data : D.data + va;
  const uint8_t* eptr = s_ti.exc_staged ? s_exc : D.exc + ea;
  const uint64_t lf = s_ti.lf;
  const uint32_t nlists = s_ti.nlists;

  uint32_t err = 0;
  Seg1 rcarry{0u, 0u};  // d-gap running state across windows
  bool staged_waited = false;

  for (uint32_t lr = 0; lr < nlists; lr += kLT) {
    // ---------------------------------------------------------------- list table
    const uint32_t cnt = min(kLT, nlists - lr);
    uint32_t kept = 0;
    if ((uint32_t)tid <= cnt) {
      const uint64_t l = lf + lr + tid;
      const uint64_t cw = D.ctrl_off[mn64(l, D.n_lists)] >> 2;
      lt_cw[tid] = (uint32_t)(cw - cbase);
      if ((uint32_t)tid < cnt) {
        const uint32_t n = D.list_n[l];
        const uint32_t Q = (n + 3) >> 2;
        const uint32_t klo = l == lf ? s_ti.j0 : 0u;
        const uint32_t kend = l == s_ti.ll ? min(Q, s_ti.j1) : Q;
        lt_q[tid] = Q;
        lt_n[tid] = n;
        lt_klo[tid] = klo;
        lt_kend[tid] = kend;
        lt_oref[tid] = l == lf ? lo_loc - 4u * s_ti.j0 : (uint32_t)((int64_t)D.out_off[l] - base_int);
        lt_db[tid] = (uint32_t)(D.data_off[l] * 32ull - va * 32ull);
        lt_eb[tid] = C::kExc ? (uint32_t)(D.exc_off[l] - ea) : 0u;
        kept = kend > klo ? kend - klo : 0u;
      }
    }
    uint32_t K;
    const uint32_t lbk = block_excl_sum(kept, s_scr, &K);
    if ((uint32_t)tid < cnt) lt_lb[tid] = lbk;
    if (!staged_waited) {
      mbar_wait(&s_bar, 0);
      staged_waited = true;
    }
    __syncthreads();

    // words of this list round
    const uint64_t rw0 = lr == 0 ? wa : cbase + lt_cw[0];
    const uint64_t rw1 = mn64(wb, cbase + lt_cw[cnt]);

    for (uint32_t u = 0; u < K; u += kRQ) {
      St carry{1u, s_ti.wq0, (uint32_t)(s_ti.wd0 - va * 32ull), (uint32_t)(s_ti.we0 - ea)};
      for (uint64_t r0 = rw0; r0 < rw1; r0 += kRoundWords) {
        const uint64_t my0 = r0 + (uint64_t)tid * kCB;
        const uint32_t myn = my0 < rw1 ? (uint32_t)mn64(kCB, rw1 - my0) : 0u;
        // list of my first word: the last table entry whose first word is <= it
        uint32_t li = 0;
        if (myn) {
          const uint32_t key = (uint32_t)(my0 - cbase);
          uint32_t a = 0, b = cnt;
          while (b - a > 1) {
            const uint32_t m = (a + b) >> 1;
            if (lt_cw[m] <= key) a = m;
            else b = m;
          }
          li = a;
        }
        uint32_t wv[kCB], pv[kCB], wl[kCB];
        St agg{0, 0, 0, 0};
#pragma unroll
        for (uint32_t k = 0; k < kCB; k++) {
          const uint64_t w = my0 + k;
          const uint32_t wr = (uint32_t)(w - cbase);
          while (li + 1 < cnt && lt_cw[li + 1] <= wr) li++;
          wl[k] = li;
          wv[k] = (k < myn && wr < ncw) ? cwp[wr] : 0u;
          pv[k] = (C::kNeedsPrev && k < myn && wr >= 1 && wr - 1 < ncw) ? cwp[wr - 1] : 0u;
          if (k < myn) {
            const uint32_t widx = wr - lt_cw[li];
            WCtx c{wv[k], pv[k], widx, lt_q[li]};
            const WAgg a = C::agg(c);
            agg = (widx == 0 && w != wa) ? St{1u, a.q, lt_db[li] + a.d, lt_eb[li] + a.e}
                                         : St{agg.f, agg.q + a.q, agg.d + a.d, agg.e + a.e};
          }
        }
        St rtot;
        St S = st_op(carry, block_excl_st<C::kExc>(agg, s_scr, &rtot));
        carry = st_op(carry, rtot);

        // per-quad descriptors (position, width, staging slot) of the window's quads
#pragma unroll
        for (uint32_t k = 0; k < kCB; k++) {
          if (k >= myn) break;
          const uint64_t w = my0 + k;
          const uint32_t wr = (uint32_t)(w - cbase);
          const uint32_t i = wl[k];
          const uint32_t widx = wr - lt_cw[i];
          WCtx c{wv[k], pv[k], widx, lt_q[i]};
          if (widx == 0 && w != wa) S = St{1u, 0u, lt_db[i], lt_eb[i]};
          const WAgg a = C::agg(c);
          const uint32_t klo = lt_klo[i], kend = lt_kend[i];
          const uint32_t qa = max(S.q, klo), qb = min(S.q + a.q, kend);
          const uint32_t x0 = lt_lb[i] + (qa - klo);  // local index of quad qa
          if (qb > qa && x0 < u + kRQ && x0 + (qb - qa) > u) {
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
                                         g.bw | (min(op, kOutWords - 4) << 6) | ((cq - 1) << 19) |
                                             (rst << 21));
                if (DGAPS && rst) atomicMin(&s_reset0, op);
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
      __syncthreads();

      // ---------------------------------------------------------------- unpack + d-gap scan
      // kQPT consecutive quads per thread: shift/mask over the 4 vertical lanes, the high
      // part of a straddling value from the current vector
      const uint32_t nr = min(kRQ, K - u);
      uint32_t y[4 * kQPT], opq[kQPT], cqs = 0, rsts = 0;
      uint32_t run = 0, fl = 0;
#pragma unroll
      for (uint32_t s = 0; s < kQPT; s++) {
        const uint32_t qi = kQPT * tid + s;
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
        const Seg1 ex =
            seg1_op(rcarry, block_excl_seg1(Seg1{fl, run}, reinterpret_cast<Seg1*>(s_scr), &rt));
        rcarry = seg1_op(rcarry, rt);
        bool seen = false;  // values before this thread's first list start continue the prefix
#pragma unroll
        for (uint32_t s = 0; s < kQPT; s++) {
          if ((rsts >> s) & 1u) seen = true;
#pragma unroll
          for (int k = 0; k < 4; k++)
            if (!seen) y[4 * s + k] += ex.v;
        }
      }
#pragma unroll
      for (uint32_t s = 0; s < kQPT; s++) {
        const uint32_t c = (cqs >> (3 * s)) & 7u;
#pragma unroll
        for (int k = 0; k < 4; k++)
          if ((uint32_t)k < c) s_out[sw_word(opq[s] + k)] = y[4 * s + k];
      }
      __syncthreads();
    }
  }
  if (!staged_waited) mbar_wait(&s_bar, 0);

  // ---------------------------------------------------------------- look-back
  if (DGAPS) {
    if (tid < 32) {
      const bool need_carry = s_ti.j0 > 0;  // the tile's first quad continues a list
      if (tid == 0)
        st_relaxed_u64(D.tiles_b + tile,
                       ((uint64_t)((rcarry.f || !need_carry) ? kFlagIncl : kFlagAgg) << 32) |
                           rcarry.v);
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

  // ---------------------------------------------------------------- coalesced store
  // 128-bit stores of [out_lo, out_hi); the tile's first list segment (before its first
  // list start) gets the carry from the look-back
  {
    const uint32_t cin = DGAPS ? s_carry : 0u;
    const uint32_t r0loc = DGAPS ? s_reset0 : 0u;
    const int64_t out_lo = s_ti.out_lo, out_hi = s_ti.out_hi;
    const int64_t c_lo = out_lo >> 2, c_hi = (out_hi + 3) >> 2;
    const int64_t cb = base_int / 4;
    for (int64_t c = c_lo + tid; c < c_hi; c += kThreads) {
      const uint32_t lc = (uint32_t)(c - cb);
      uint4 v = s_out4[sw_chunk(lc)];
      if (DGAPS && cin) {
        const uint32_t p = 4 * lc;
        if (p < r0loc) v.x += cin;
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
