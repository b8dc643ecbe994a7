// gc_encoder.cpp -- multi-threaded host encoder of the product library.
//
// Produces the batch stream format of DESIGN.md §3 (byte-identical to oracle/'s
// encoder, which tests/test_encoder_parity.py checks) so that bench.py and users
// can build inputs without the test oracle.  Written independently of
// oracle/gc_oracle.c: streaming per-lane bit writers, OR-based pseudo quad maxima
// (equivalent by the theorem in DESIGN.md A9), a declarative form of
// Algorithm 1, block maxima for the AFOR DP and a width histogram for PFD.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "gc.h"

namespace {

inline uint32_t eff_width(uint32_t x) { return x ? 32u - (uint32_t)__builtin_clz(x) : 1u; }
inline uint32_t lowmask(uint32_t b) { return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u); }
inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

constexpr uint8_t kNum[10] = {32, 16, 10, 8, 6, 5, 4, 3, 2, 1};  // Table III
constexpr uint8_t kBw[10] = {1, 2, 3, 4, 5, 6, 8, 10, 16, 32};

struct Buf {
  std::vector<uint8_t> ctrl;
  std::vector<uint32_t> data;  // 4 words per 128-bit vector
  std::vector<uint8_t> exc;
};

// Four per-lane bit writers sharing one offset: values fill a component upward; a
// value that does not fit puts its high part in the current component and its low
// part at the bottom of the next vector's component (§5.2.2).
struct LaneWriter {
  std::vector<uint32_t>* out;
  uint32_t cur[4] = {0, 0, 0, 0};
  uint32_t off = 0;
  explicit LaneWriter(std::vector<uint32_t>* o) : out(o) {}
  void flush_vec() {
    out->insert(out->end(), cur, cur + 4);
    cur[0] = cur[1] = cur[2] = cur[3] = 0;
    off = 0;
  }
  void put(const uint32_t* v, uint32_t bw) {
    if (off + bw <= 32) {
      for (int k = 0; k < 4; k++) cur[k] |= (v[k] & lowmask(bw)) << off;
      off += bw;
      if (off == 32) flush_vec();
      return;
    }
    uint32_t r = 32 - off, rest = bw - r;
    for (int k = 0; k < 4; k++) cur[k] |= ((v[k] & lowmask(bw)) >> rest) << off;
    uint32_t low[4];
    for (int k = 0; k < 4; k++) low[k] = v[k] & lowmask(rest);
    flush_vec();
    for (int k = 0; k < 4; k++) cur[k] = low[k];
    off = rest;
  }
  void close() {  // pad to a whole vector
    if (off) flush_vec();
  }
};

// MSB-first control bit writer (unary LDs).
struct UnaryWriter {
  std::vector<uint8_t>* out;
  uint64_t base, bits = 0;
  explicit UnaryWriter(std::vector<uint8_t>* o) : out(o), base(o->size()) {}
  void bit(uint32_t b) {
    if ((bits & 7) == 0) out->push_back(0);
    if (b) (*out)[base + (bits >> 3)] |= (uint8_t)(0x80u >> (bits & 7));
    bits++;
  }
};

class ListEncoder {
 public:
  explicit ListEncoder(const gc_encode_params& p) : p_(p) {
    // SIMD-BP128 (PFD variant 1): b = the frame's maximum width, i.e. the PFD
    // rule with zeta = 0 (no exceptions)
    if (p_.codec == GC_GROUP_PFD && p_.variant == 1) {
      p_.zeta_num = 0;
      p_.zeta_den = 1;
    }
  }

  void encode(const uint32_t* x, uint32_t n, Buf& b) {
    if (p_.codec == GC_VARBYTE) {  // P §2.3: 7-bit groups, least significant first, MSB=1 last
      const size_t c0 = b.ctrl.size();
      for (uint32_t i = 0; i < n; i++) {
        uint32_t v = x[i];
        while (v >= 128) {
          b.ctrl.push_back((uint8_t)(v & 127));
          v >>= 7;
        }
        b.ctrl.push_back((uint8_t)(v | 128));
      }
      pad_ctrl(b, c0);
      return;
    }
    const uint64_t Q = cdiv(n, 4);
    quads_.assign(4 * Q, 0);
    std::memcpy(quads_.data(), x, 4ull * n);
    wq_.resize(Q);
    for (uint64_t j = 0; j < Q; j++) {
      const uint32_t* q = &quads_[4 * j];
      wq_[j] = eff_width(q[0] | q[1] | q[2] | q[3]);  // pseudo quad max
    }
    switch (p_.codec) {
      case GC_GROUP_SIMPLE: simple(Q, b); break;
      case GC_GROUP_SCHEME: scheme(Q, b); break;
      case GC_GROUP_AFOR: afor(Q, b); break;
      default: pfd(Q, b); break;
    }
  }

 private:
  // Group-Simple: each selector is the smallest SEL whose run over the remaining
  // quads reaches NUM or the end (Algorithm 1).
  void simple(uint64_t Q, Buf& b) {
    const size_t c0 = b.ctrl.size();
    uint64_t j = 0, s = 0;
    while (j < Q) {
      uint64_t rem = Q - j;
      uint32_t runmax[32];
      uint32_t m = 0;
      for (uint64_t t = 0; t < 32 && t < rem; t++) runmax[t] = m = std::max(m, wq_[j + t]);
      uint32_t sel = 9;
      for (uint32_t i = 0; i < 10; i++) {
        uint64_t c = std::min<uint64_t>(kNum[i], rem);
        if (runmax[c - 1] <= kBw[i]) {
          sel = i;
          break;
        }
      }
      uint64_t c = std::min<uint64_t>(kNum[sel], rem);
      uint32_t comp[4] = {0, 0, 0, 0};
      for (uint64_t t = 0; t < c; t++)
        for (int k = 0; k < 4; k++) comp[k] |= quads_[4 * (j + t) + k] << (t * kBw[sel]);
      b.data.insert(b.data.end(), comp, comp + 4);
      if ((s & 1) == 0) b.ctrl.push_back((uint8_t)sel);
      else b.ctrl.back() |= (uint8_t)(sel << 4);
      s++;
      j += c;
    }
    pad_ctrl(b, c0);
  }

  void scheme(uint64_t Q, Buf& b) {
    const uint32_t lg = p_.variant & 3u, CG = 1u << lg, kind = (p_.variant >> 2) & 3u;
    const size_t c0 = b.ctrl.size();
    units_.resize(Q);
    for (uint64_t j = 0; j < Q; j++) units_[j] = (wq_[j] + CG - 1) >> lg;  // Eq. (1)
    if (kind == 0) {
      const uint32_t fw = 5 - lg;
      for (uint64_t j = 0; j < Q; j++) {
        uint32_t ld = units_[j] - 1;
        if (CG == 1) {
          uint64_t unit = j / 3, f = j % 3;
          if (f == 0) b.ctrl.insert(b.ctrl.end(), 2, 0);
          uint16_t u16 = (uint16_t)(b.ctrl[c0 + 2 * unit] | (b.ctrl[c0 + 2 * unit + 1] << 8));
          u16 |= (uint16_t)(ld << (fw * f));
          b.ctrl[c0 + 2 * unit] = (uint8_t)u16;
          b.ctrl[c0 + 2 * unit + 1] = (uint8_t)(u16 >> 8);
        } else {
          const uint32_t per = 8 / (CG == 4 ? 4 : fw);  // fields per byte: 2, 2, 4
          uint64_t byte = j / per, f = j % per;
          if (f == 0) b.ctrl.push_back(0);
          b.ctrl[c0 + byte] |= (uint8_t)(ld << (fw * f));
        }
      }
    } else {
      UnaryWriter uw(&b.ctrl);
      for (uint64_t j = 0; j < Q; j++) {
        uint32_t u = units_[j];
        if (kind == 2 && (uw.bits & 7) && (uw.bits & 7) + u > 8)
          while (uw.bits & 7) uw.bit(1);  // IU: a code never crosses a byte
        for (uint32_t t = 1; t < u; t++) uw.bit(1);
        uw.bit(0);
      }
      if (kind == 2)
        while (uw.bits & 7) uw.bit(1);
    }
    LaneWriter lw(&b.data);
    for (uint64_t j = 0; j < Q; j++) lw.put(&quads_[4 * j], CG * units_[j]);
    lw.close();
    pad_ctrl(b, c0);
  }

  // Group-AFOR: DP over frames of {8,16,32} quads starting at multiples of 8; ties go
  // to the longer frame (A23-A25).
  void afor(uint64_t Q, Buf& b) {
    const size_t c0 = b.ctrl.size();
    const uint64_t nb = cdiv(Q, 8);  // 8-quad blocks; padded quads have width 1
    if (nb == 0) return;
    quads_.resize(32 * nb, 0);
    bmax_.assign(nb, 1);
    for (uint64_t j = 0; j < Q; j++) bmax_[j / 8] = std::max(bmax_[j / 8], wq_[j]);
    cost_.assign(nb + 1, 0);
    pick_.assign(nb + 1, 1);
    for (int64_t i = (int64_t)nb - 1; i >= 0; i--) {
      uint64_t best = ~0ull;
      uint32_t bl = 1;
      for (uint32_t blocks : {4u, 2u, 1u}) {
        if ((uint64_t)i + blocks > nb) continue;
        uint32_t bw = 1;
        for (uint32_t t = 0; t < blocks; t++) bw = std::max(bw, bmax_[i + t]);
        uint64_t c = 8 + 128 * cdiv(8ull * blocks * bw, 32) + cost_[i + blocks];
        if (c < best) {
          best = c;
          bl = blocks;
        }
      }
      cost_[i] = best;
      pick_[i] = bl;
    }
    for (uint64_t i = 0; i < nb; i += pick_[i]) {
      uint32_t blocks = pick_[i], bw = 1;
      for (uint32_t t = 0; t < blocks; t++) bw = std::max(bw, bmax_[i + t]);
      uint32_t code = blocks == 1 ? 0 : (blocks == 2 ? 1 : 2);
      b.ctrl.push_back((uint8_t)(code | ((bw - 1) << 2)));
      LaneWriter lw(&b.data);
      for (uint64_t j = 8 * i; j < 8 * (i + blocks); j++) lw.put(&quads_[4 * j], bw);
      lw.close();
    }
    pad_ctrl(b, c0);
  }

  void pfd(uint64_t Q, Buf& b) {
    const uint32_t F = p_.pfd_frame_quads;
    const uint32_t posb = 4 * F <= 256 ? 1 : 2;
    for (uint64_t f0 = 0; f0 < Q; f0 += F) {
      const uint32_t q = (uint32_t)std::min<uint64_t>(F, Q - f0);
      uint32_t hist[33] = {0};
      for (uint32_t j = 0; j < q; j++) hist[wq_[f0 + j]]++;
      // smallest b with #{quads wider than b} * den <= num * q
      uint32_t bsel = 32, above = 0;
      uint32_t gt[33];
      for (int w = 32; w >= 0; w--) {
        gt[w] = above;
        above += hist[w];
      }
      for (uint32_t bb = 1; bb <= 32; bb++)
        if ((uint64_t)gt[bb] * p_.zeta_den <= (uint64_t)p_.zeta_num * q) {
          bsel = bb;
          break;
        }
      const uint32_t* fq = &quads_[4 * f0];
      uint32_t cnt = 0, vmax = 0;
      for (uint32_t i = 0; i < 4 * q; i++)
        if (eff_width(fq[i]) > bsel) {
          cnt++;
          vmax = std::max(vmax, fq[i]);
        }
      const uint32_t wcode = cnt == 0 ? 0 : (vmax < 256u ? 1 : (vmax < 65536u ? 2 : 3));
      const uint32_t wbytes = wcode == 0 ? 0 : (wcode == 1 ? 1 : (wcode == 2 ? 2 : 4));
      b.ctrl.push_back((uint8_t)bsel);
      b.ctrl.push_back((uint8_t)wcode);
      b.ctrl.push_back((uint8_t)(cnt & 0xFF));
      b.ctrl.push_back((uint8_t)(cnt >> 8));
      size_t e0 = b.exc.size();
      b.exc.resize(e0 + (size_t)cnt * (posb + wbytes), 0);
      uint32_t e = 0;
      for (uint32_t i = 0; i < 4 * q; i++)
        if (eff_width(fq[i]) > bsel) {
          b.exc[e0 + (size_t)e * posb] = (uint8_t)i;
          if (posb == 2) b.exc[e0 + (size_t)e * posb + 1] = (uint8_t)(i >> 8);
          for (uint32_t t = 0; t < wbytes; t++)
            b.exc[e0 + (size_t)cnt * posb + (size_t)e * wbytes + t] = (uint8_t)(fq[i] >> (8 * t));
          e++;
        }
      LaneWriter lw(&b.data);
      for (uint32_t j = 0; j < q; j++) lw.put(&fq[4 * j], bsel);  // low b bits of every slot
      lw.close();
    }
  }

  static void pad_ctrl(Buf& b, size_t c0) {
    while ((b.ctrl.size() - c0) & 3) b.ctrl.push_back(0);
  }

  gc_encode_params p_;
  std::vector<uint32_t> quads_, wq_, units_, bmax_, pick_;
  std::vector<uint64_t> cost_;
};

struct Job {
  uint64_t l0 = 0, l1 = 0;
  Buf buf;
  std::vector<uint64_t> csz, dsz, esz;  // per list sizes
  gc_status rc = GC_OK;
};

struct Handle {
  std::vector<Job> jobs;
  uint64_t n_lists = 0;
  const uint64_t* ctrl_off = nullptr;  // caller arrays (kept for finish)
  const uint64_t* data_off = nullptr;
  const uint64_t* exc_off = nullptr;
  std::vector<uint64_t> coff, doff, eoff;
  uint64_t sizes[3] = {0, 0, 0};
};

void run_job(const gc_encode_params& p, const uint32_t* values, const uint32_t* list_n,
             const uint64_t* in_off, int delta, Job& J) {
  ListEncoder enc(p);
  std::vector<uint32_t> g;
  J.csz.resize(J.l1 - J.l0);
  J.dsz.resize(J.l1 - J.l0);
  J.esz.resize(J.l1 - J.l0);
  for (uint64_t l = J.l0; l < J.l1; l++) {
    const uint32_t n = list_n[l];
    const uint32_t* x = values + in_off[l];
    if (delta) {  // d-gap: g_1 = d_1, g_i = d_i - d_{i-1}
      g.resize(n);
      for (uint32_t i = 0; i < n; i++) {
        if (i > 0 && x[i] <= x[i - 1]) {
          J.rc = GC_ERR_NOT_INCREASING;
          return;
        }
        g[i] = i ? x[i] - x[i - 1] : x[0];
      }
      x = g.data();
    }
    size_t c = J.buf.ctrl.size(), d = J.buf.data.size(), e = J.buf.exc.size();
    enc.encode(x, n, J.buf);
    J.csz[l - J.l0] = J.buf.ctrl.size() - c;
    J.dsz[l - J.l0] = (J.buf.data.size() - d) / 4;
    J.esz[l - J.l0] = J.buf.exc.size() - e;
  }
}

bool valid_params(const gc_encode_params* p) {
  if (!p) return false;
  switch (p->codec) {
    case GC_VARBYTE:
    case GC_GROUP_SIMPLE:
    case GC_GROUP_AFOR:
      return true;
    case GC_GROUP_SCHEME: {
      uint32_t kind = (p->variant >> 2) & 3u, cg = 1u << (p->variant & 3u);
      return p->variant <= 15 && kind <= 2 && !(kind == 2 && cg < 4);
    }
    case GC_GROUP_PFD:
      return (p->pfd_frame_quads == 32 || p->pfd_frame_quads == 128) && p->variant <= 1 &&
             (p->zeta_den > 0 || p->variant == 1);
    default:
      return false;
  }
}

}  // namespace

extern "C" {

gc_status gc_encode_begin(const gc_encode_params* p, const uint32_t* values,
                          const uint32_t* list_n, uint64_t n_lists, int delta, int threads,
                          uint64_t* ctrl_off, uint64_t* data_off, uint64_t* exc_off,
                          uint64_t* out_off, uint64_t* sizes, void** handle) {
  if (!valid_params(p)) return p && p->codec >= 2 && p->codec <= 5 ? GC_ERR_BAD_VARIANT
                                                                    : GC_ERR_UNKNOWN_CODEC;
  if (!handle || !sizes || !ctrl_off || !data_off || !exc_off || !out_off ||
      (n_lists && (!list_n)))
    return GC_ERR_INVALID_ARGUMENT;
  *handle = nullptr;
  Handle* H = new (std::nothrow) Handle;
  if (!H) return GC_ERR_NOMEM;
  try {
    std::vector<uint64_t> in_off(n_lists + 1, 0);
    for (uint64_t l = 0; l < n_lists; l++) in_off[l + 1] = in_off[l] + list_n[l];
    if (in_off[n_lists] && !values) {
      delete H;
      return GC_ERR_INVALID_ARGUMENT;
    }
    int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)T, std::max<uint64_t>(n_lists, 1)));
    H->jobs.resize(T);
    uint64_t total = in_off[n_lists], l = 0;
    for (int t = 0; t < T; t++) {
      H->jobs[t].l0 = l;
      uint64_t target = total * (uint64_t)(t + 1) / (uint64_t)T;
      while (l < n_lists && (in_off[l] < target || t == T - 1)) l++;
      H->jobs[t].l1 = l;
    }
    H->jobs[T - 1].l1 = n_lists;
    std::vector<std::thread> pool;
    for (int t = 1; t < T; t++)
      pool.emplace_back(run_job, std::cref(*p), values, list_n, in_off.data(), delta,
                        std::ref(H->jobs[t]));
    run_job(*p, values, list_n, in_off.data(), delta, H->jobs[0]);
    for (auto& th : pool) th.join();
    for (auto& J : H->jobs)
      if (J.rc != GC_OK) {
        gc_status rc = J.rc;
        delete H;
        return rc;
      }
    ctrl_off[0] = data_off[0] = exc_off[0] = out_off[0] = 0;
    for (auto& J : H->jobs)
      for (uint64_t li = J.l0; li < J.l1; li++) {
        ctrl_off[li + 1] = ctrl_off[li] + J.csz[li - J.l0];
        data_off[li + 1] = data_off[li] + J.dsz[li - J.l0];
        exc_off[li + 1] = exc_off[li] + J.esz[li - J.l0];
        out_off[li + 1] = out_off[li] + list_n[li];
      }
    H->n_lists = n_lists;
    H->sizes[0] = (ctrl_off[n_lists] + 15) & ~15ull;
    H->sizes[1] = data_off[n_lists];
    H->sizes[2] = (exc_off[n_lists] + 15) & ~15ull;
    H->coff.assign(ctrl_off, ctrl_off + n_lists + 1);
    H->doff.assign(data_off, data_off + n_lists + 1);
    H->eoff.assign(exc_off, exc_off + n_lists + 1);
    sizes[0] = H->sizes[0];
    sizes[1] = H->sizes[1];
    sizes[2] = H->sizes[2];
  } catch (const std::bad_alloc&) {
    delete H;
    return GC_ERR_NOMEM;
  }
  *handle = H;
  return GC_OK;
}

gc_status gc_encode_finish(void* handle, uint8_t* ctrl, void* data, uint8_t* exc) {
  Handle* H = (Handle*)handle;
  if (!H) return GC_ERR_INVALID_ARGUMENT;
  if ((H->sizes[0] && !ctrl) || (H->sizes[1] && !data) || (H->sizes[2] && !exc)) {
    return GC_ERR_INVALID_ARGUMENT;
  }
  auto copy = [&](Job& J) {
    if (J.l0 == J.l1) return;
    uint64_t c = H->coff[J.l0], d = H->doff[J.l0], e = H->eoff[J.l0];
    if (!J.buf.ctrl.empty()) std::memcpy(ctrl + c, J.buf.ctrl.data(), J.buf.ctrl.size());
    if (!J.buf.data.empty())
      std::memcpy((uint8_t*)data + 16 * d, J.buf.data.data(), 4 * J.buf.data.size());
    if (!J.buf.exc.empty()) std::memcpy(exc + e, J.buf.exc.data(), J.buf.exc.size());
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < H->jobs.size(); t++) pool.emplace_back(copy, std::ref(H->jobs[t]));
  if (!H->jobs.empty()) copy(H->jobs[0]);
  for (auto& th : pool) th.join();
  uint64_t n = H->n_lists;
  if (ctrl && H->sizes[0] > H->coff[n]) std::memset(ctrl + H->coff[n], 0, H->sizes[0] - H->coff[n]);
  if (exc && H->sizes[2] > H->eoff[n]) std::memset(exc + H->eoff[n], 0, H->sizes[2] - H->eoff[n]);
  delete H;
  return GC_OK;
}

void gc_encode_abort(void* handle) { delete (Handle*)handle; }

}  // extern "C"
