// gc_skip.cuh -- skip pointers (§7.5) and random access from them; included inside
// namespace gcd by gc_kernels.cu, after k_index (which writes the entries, gc_build_skip).
//
// gc_decode_range decodes the 512-int blocks overlapping an output range, each on its own
// from its skip entry: one warp per block parses the block's control words from the
// entry's word (the codec parsers of gc_codecs.cuh), a warp scan seeded with the entry's
// quad / data / exception prefixes places every group, the kept quads are unpacked with
// the paper's high-first split straight from the data stream, Group-PFD
// exceptions overwrite their slots, and the d-gap scan starts from the
// entry's docid.  Nothing depends on other blocks: no index stage, no look-back.

// skip_off[l] = sum over lists l' < l of ceil(n_l' / 512): one CTA, chunks of its width.
constexpr uint32_t kSkipT = 1024;
__global__ void __launch_bounds__(kSkipT) k_skip_off(Dev D) {
  __shared__ unsigned long long s_w[kSkipT / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long carry = 0;
  for (uint64_t base = 0; base < D.n_lists; base += kSkipT) {
    const uint64_t l = base + tid;
    const unsigned long long v = l < D.n_lists ? (D.list_n[l] + GC_SKIP_DIST - 1) / GC_SKIP_DIST : 0;
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (uint32_t)o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    unsigned long long wpre = 0, tot = 0;
    for (uint32_t x = 0; x < kSkipT / 32; x++) {
      if (x < warp) wpre += s_w[x];
      tot += s_w[x];
    }
    if (l < D.n_lists) D.skip_off[l] = carry + wpre + inc - v;
    carry += tot;
    __syncthreads();
  }
  if (tid == 0) D.skip_off[D.n_lists] = carry;
}

// The entry range [e0, e1) covering output ints [first, last): one warp (32-ary searches,
// a few dependent loads instead of log2(lists)).
__global__ void k_range_bounds(Dev D, uint64_t first, uint64_t last, unsigned long long* eb) {
  // the list holding output int p: the last l with out_off[l] <= p
  const uint64_t la = warp_find(D.out_off, 0, D.n_lists, first);
  const uint64_t lb = warp_find(D.out_off, la, D.n_lists, last - 1);
  if (threadIdx.x == 0) {
    D.hdr->status = 0u;  // (the call's status reset: k_range runs after this kernel)
    eb[0] = D.skip_off[la] + (first - D.out_off[la]) / GC_SKIP_DIST;
    eb[1] = D.skip_off[lb] + (last - 1 - D.out_off[lb]) / GC_SKIP_DIST + 1;
  }
}

constexpr uint32_t kRangeW = 4;  // warps per CTA of k_range
template <class C, bool DGAPS>
__global__ void __launch_bounds__(32 * kRangeW) k_range(Dev D, uint32_t* __restrict__ out,
                                                        uint64_t first, uint64_t last,
                                                        const unsigned long long* eb) {
  __shared__ uint32_t s_gap[kRangeW][GC_SKIP_DIST];
  const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* gap = s_gap[wl];
  constexpr uint32_t P = C::kParts;
  constexpr uint32_t FULL = 0xffffffffu;
  const uint64_t e0 = eb[0], e1 = eb[1];
  uint32_t err = 0;
  uint64_t lc = ~0ull;  // the list of the warp's previous block
  for (uint64_t e = e0 + (uint64_t)blockIdx.x * kRangeW + wl; e < e1; e += (uint64_t)gridDim.x * kRangeW) {
    // the block's list: skip_off[l] <= e < skip_off[l + 1] (a warp-wide 32-ary search,
    // starting from the previous block's list when it still holds this one)
    if (!(lc < D.n_lists && D.skip_off[lc] <= e && e < D.skip_off[lc + 1]))
      lc = warp_find(D.skip_off, lc < D.n_lists && D.skip_off[lc] <= e ? lc : 0, D.n_lists, e);
    const uint64_t l = lc;
    const uint64_t blk = e - D.skip_off[l];
    const uint32_t n = D.list_n[l];
    const uint64_t Q = (n + 3ull) >> 2, nblk = (n + GC_SKIP_DIST - 1) / GC_SKIP_DIST;
    const uint64_t cw0 = D.ctrl_off[l] >> 2, ncw = (D.ctrl_off[l + 1] >> 2) - cw0;
    const uint64_t dbase = D.data_off[l], dlim = D.data_off[l + 1] - dbase;
    const uint64_t ebase = C::kExc ? D.exc_off[l] : 0ull;
    const uint64_t elim = C::kExc ? D.exc_off[l + 1] - ebase : 0ull;
    const gc_skip_entry ent = D.skip[e];
    const uint32_t wa = ent.word;
    const uint32_t wb = blk + 1 < nblk ? D.skip[e + 1].word : (uint32_t)(ncw ? ncw - 1 : 0);
    if (blk >= nblk || wa > wb || wb >= ncw || dlim == 0) {  // (a bad table or directory)
      err |= GC_DEV_TRUNCATED;
      continue;
    }
    const uint32_t qa = (uint32_t)(128 * blk), qb = (uint32_t)mn64(128 * blk + 128, Q);
    for (uint32_t i = lane; i < GC_SKIP_DIST; i += 32) gap[i] = 0u;
    __syncwarp();
    auto unpack_quad = [&](uint32_t j, uint32_t pos, uint32_t bw) {
      const uint32_t m = pos >> 5, off = pos & 31u;
      if (m >= dlim) {
        err |= GC_DEV_TRUNCATED;
        return;
      }
      const uint4 v0 = __ldg(D.data + dbase + m);
      const uint4 v1 = __ldg(D.data + dbase + mn64(m + 1, dlim - 1));
      // the value's high part is the top of the current component, its low part the
      // bottom of the next vector's component
      const bool strad = off + bw > 32u;
      const uint32_t shl = strad ? 0u : 32u - off - bw, shr = 32u - bw;
      const uint32_t ml = strad ? (1u << (off + bw - 32u)) - 1u : 0u;
      const uint32_t s0 = 4u * (j - qa);
      GC_CHECK(s0 + 3 < GC_SKIP_DIST);
      gap[s0] = (((v0.x << shl) >> shr) & ~ml) | (v1.x & ml);
      gap[s0 + 1] = (((v0.y << shl) >> shr) & ~ml) | (v1.y & ml);
      gap[s0 + 2] = (((v0.z << shl) >> shr) & ~ml) | (v1.z & ml);
      gap[s0 + 3] = (((v0.w << shl) >> shr) & ~ml) | (v1.w & ml);
    };
    // the running (quads, lane-bits, exception bytes) prefix, seeded with the entry's
    uint32_t cq = ent.quads, cd = (uint32_t)ent.data_bits, ce = ent.exc_bytes;
    const uint32_t u0 = wa * P, u1 = (wb + 1) * P;
    for (uint32_t ub = u0; ub < u1; ub += 32) {
      const uint32_t un = ub + lane, w = un / P, part = un % P;
      const bool have = un < u1;
      const uint32_t wv = have ? D.ctrl_words[cw0 + w] : 0u;
      const uint32_t pv = (have && C::kNeedsPrev && w > 0) ? D.ctrl_words[cw0 + w - 1] : 0u;
      const WCtx c{wv, pv, w, Q, part};
      WAgg ag = have ? C::agg(c) : WAgg{0u, 0u, 0u};
      // exclusive warp scan of the unit aggregates (one list: no segments)
      uint32_t iq = ag.q, id = ag.d, ie = ag.e;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t tq = __shfl_up_sync(FULL, iq, o), td = __shfl_up_sync(FULL, id, o),
                       te = __shfl_up_sync(FULL, ie, o);
        if (lane >= (uint32_t)o) {
          iq += tq;
          id += td;
          ie += te;
        }
      }
      const uint32_t q0 = cq + iq - ag.q, d0 = cd + id - ag.d, x0 = ce + ie - ag.e;
      cq += __shfl_sync(FULL, iq, 31);
      cd += __shfl_sync(FULL, id, 31);
      ce += __shfl_sync(FULL, ie, 31);
      const uint32_t ja = max(q0, qa), jb = min(q0 + ag.q, qb);
      if (have && jb > ja) {
        if constexpr (!C::kMultiQuad) {
          C::emit(c, q0, d0, ja, jb, [&](uint32_t j, uint32_t pos, uint32_t bw) { unpack_quad(j, pos, bw); });
        } else {
          C::walk(c, [&](const Grp& g) {
            const uint32_t gq = q0 + g.q0;
            const uint32_t ga = max(gq, ja), gb = min(gq + g.nq, jb);
            if (g.err && gq < Q) err |= g.err;
            if (ga >= gb) return;
            const uint32_t gd = d0 + (uint32_t)g.d0;
            for (uint32_t j = ga; j < gb; j++) unpack_quad(j, gd + (j - gq) * g.step, g.bw);
            if constexpr (C::kExc) {
              // Group-PFD: the frame's exceptions in these quads overwrite their slots
              // (P:L416); positions are frame-relative ints, values follow them
              const uint32_t pb = C::kPosBytes;
              const uint64_t x = x0 + g.e0;
              const uint32_t fq0 = gq - g.t0;
              if (x + g.cnt * (pb + g.wb) > elim) {
                err |= GC_DEV_TRUNCATED;
                return;
              }
              const uint8_t* ex = D.exc + ebase + x;
              uint32_t pprev = 0;
              for (uint32_t t = 0; t < g.cnt; t++) {
                uint32_t p = ex[t * pb];
                if (pb == 2) p |= (uint32_t)ex[t * pb + 1] << 8;
                if (p >= 4u * g.fq || (t > 0 && p <= pprev)) {
                  err |= GC_DEV_BAD_EXCEPTION;
                  break;
                }
                pprev = p;
                const uint32_t j = fq0 + p / 4;
                if (j < ga || j >= gb) continue;
                const uint8_t* vb = ex + g.cnt * pb + t * g.wb;
                uint32_t v = vb[0];
                if (g.wb > 1) v |= (uint32_t)vb[1] << 8;
                if (g.wb > 2) v |= ((uint32_t)vb[2] << 16) | ((uint32_t)vb[3] << 24);
                gap[4u * (j - qa) + (p & 3u)] = v;
              }
            }
          });
        }
      }
    }
    __syncwarp();
    // d-gap scan: lane r owns the block's ints [16r, 16r+16); the carry is the
    // entry's docid, the list's ints before the block summed
    uint32_t v[16];
#pragma unroll
    for (uint32_t i = 0; i < 16; i++) v[i] = gap[16 * lane + i];
    if (DGAPS) {
#pragma unroll
      for (uint32_t i = 1; i < 16; i++) v[i] += v[i - 1];
      uint32_t inc = v[15];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc, o);
        if (lane >= (uint32_t)o) inc += t;
      }
      const uint32_t ex = ent.docid + inc - v[15];
#pragma unroll
      for (uint32_t i = 0; i < 16; i++) v[i] += ex;
    }
    // exactly the range's ints of this block
    const uint64_t ob = D.out_off[l] + GC_SKIP_DIST * blk;
#pragma unroll
    for (uint32_t i = 0; i < 16; i++) {
      const uint64_t p = 16 * lane + i;
      if (GC_SKIP_DIST * blk + p < n && ob + p >= first && ob + p < last) {
        GC_CHECK(ob + p < D.total_out);
        out[ob + p] = v[i];
      }
    }
    __syncwarp();
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err) atomicOr(&D.hdr->status, err);
}
