/*
 * gc_oracle.c -- TEST INFRASTRUCTURE ONLY (see gc_oracle.h).
 *
 * A plain CPU implementation of the Group formats of arXiv 1502.01916,
 * written from PAPER.md in the paper's order and notation.  Loops, no
 * intrinsics, no lookup tables, no blocking or fusion.  Readings of silent or
 * garbled passages follow SURVEY.md §8(c) (ids A1..A45), restated in
 * DESIGN.md §3.
 *
 * Parity status of every function: pinned by tests/test_oracle_*.py
 * (paper worked examples, closed forms, an independent bit reader written from
 * the prose format, brute force over tiny inputs, round trip).  The exact byte
 * layout of the authors' unpublished implementation (Figs. 2-5 are missing
 * from PAPER.md) is "parity unpinned" -- see DESIGN.md §3.
 */
#include "gc_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* bitcore                                                              */
/* ------------------------------------------------------------------ */

/* Effective bit width, §2.1.2 "the minimum number of bits to encode an
 * integer in binary"; width(0) = 1 (A1). Counted by shifting, on purpose. */
uint32_t gco_width(uint32_t x) {
  uint32_t w = 0;
  while (x != 0) {
    w++;
    x >>= 1;
  }
  return w == 0 ? 1 : w;
}

static uint32_t mask_bits(uint32_t b) { return b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u); }

/* quadmax[i] = max(input[4i..4i+3]), §4.2. */
uint32_t gco_quad_max(const uint32_t* q4) {
  uint32_t m = q4[0];
  for (int k = 1; k < 4; k++)
    if (q4[k] > m) m = q4[k];
  return m;
}

/* pseudo quad max (bitwise OR), §4.4. Used only by tests (A9). */
uint32_t gco_quad_or(const uint32_t* q4) { return q4[0] | q4[1] | q4[2] | q4[3]; }

/* 4-way vertical layout, §2.1.2, §3.1: lane k of every
 * quadruple lives in 32-bit component k of consecutive 128-bit vectors.
 * Bits are consumed from the least-significant end (A2).  A value that does
 * not fit in the r bits left in the current component is split "from high to
 * low ... The first part is stored in the current data vector and the second
 * one would be stored in the next data vector" (§5.2.2, A3). */
static void put_quad(uint32_t* data, uint64_t base_vec, uint64_t pos, uint32_t bw,
                     const uint32_t* q) {
  uint64_t m = base_vec + (pos >> 5);
  uint32_t off = (uint32_t)(pos & 31);
  uint32_t r = 32 - off;
  for (int k = 0; k < 4; k++) {
    uint32_t v = q[k] & mask_bits(bw);
    if (bw <= r) {
      data[4 * m + k] |= v << off;
    } else {
      uint32_t low_len = bw - r;
      data[4 * m + k] |= (v >> low_len) << off;          /* high part: current vector */
      data[4 * (m + 1) + k] |= v & mask_bits(low_len);   /* low part: next vector */
    }
  }
}

/* Decode side of the split, §5.2.3: "we first left-shift the value
 * recovered in the current data vector, and then add it to the value
 * recovered in the next data vector". */
static void get_quad(const uint32_t* data, uint64_t base_vec, uint64_t pos, uint32_t bw,
                     uint32_t* q) {
  uint64_t m = base_vec + (pos >> 5);
  uint32_t off = (uint32_t)(pos & 31);
  uint32_t r = 32 - off;
  for (int k = 0; k < 4; k++) {
    if (bw <= r) {
      q[k] = (data[4 * m + k] >> off) & mask_bits(bw);
    } else {
      uint32_t low_len = bw - r;
      uint32_t high = data[4 * m + k] >> off; /* r bits */
      uint32_t low = data[4 * (m + 1) + k] & mask_bits(low_len);
      q[k] = (high << low_len) + low;
    }
  }
}

static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

int gco_pack_vertical(const uint32_t* quads, uint64_t Q, uint32_t bw, uint32_t* data,
                      uint64_t nvec) {
  if (bw < 1 || bw > 32) return GCO_ERR_ARG;
  if (nvec < ceil_div(Q * bw, 32)) return GCO_ERR_TRUNCATED;
  memset(data, 0, (size_t)(nvec * 16));
  for (uint64_t j = 0; j < Q; j++) {
    for (int k = 0; k < 4; k++)
      if (bw < 32 && (quads[4 * j + k] >> bw) != 0) return GCO_ERR_ARG;
    put_quad(data, 0, j * bw, bw, quads + 4 * j);
  }
  return GCO_OK;
}

int gco_unpack_vertical(const uint32_t* data, uint64_t nvec, uint32_t bw, uint64_t Q,
                        uint32_t* quads) {
  if (bw < 1 || bw > 32) return GCO_ERR_ARG;
  if (nvec < ceil_div(Q * bw, 32)) return GCO_ERR_TRUNCATED;
  for (uint64_t j = 0; j < Q; j++) get_quad(data, 0, j * bw, bw, quads + 4 * j);
  return GCO_OK;
}

/* Growable byte / vector buffers. */
typedef struct {
  uint8_t* p;
  uint64_t n, cap;
} bytebuf;

static int bb_reserve(bytebuf* b, uint64_t n) {
  if (n <= b->cap) return 0;
  uint64_t c = b->cap ? b->cap : 64;
  while (c < n) c *= 2;
  uint8_t* q = (uint8_t*)realloc(b->p, (size_t)c);
  if (!q) return -1;
  memset(q + b->cap, 0, (size_t)(c - b->cap));
  b->p = q;
  b->cap = c;
  return 0;
}

static int bb_push(bytebuf* b, uint8_t v) {
  if (bb_reserve(b, b->n + 1)) return -1;
  b->p[b->n++] = v;
  return 0;
}

/* Quadruples of a list, zero-padded to a whole quad (A5). */
static uint32_t* make_quads(const uint32_t* x, uint32_t n, uint64_t Q_alloc) {
  uint32_t* q = (uint32_t*)calloc((size_t)(4 * (Q_alloc ? Q_alloc : 1)), sizeof(uint32_t));
  if (!q) return NULL;
  for (uint32_t i = 0; i < n; i++) q[i] = x[i];
  return q;
}

/* ------------------------------------------------------------------ */
/* Group-Simple, §4, Table III                             */
/* ------------------------------------------------------------------ */

static const uint32_t GS_NUM[10] = {32, 16, 10, 8, 6, 5, 4, 3, 2, 1};
static const uint32_t GS_BW[10] = {1, 2, 3, 4, 5, 6, 8, 10, 16, 32};

/* Algorithm 1, transcribed line by line.  Returns TotalModeNum;
 * ModeArr[k] = selector i.  mask = Power(2,b)-1 is computed in 64 bits (A8). */
uint64_t gco_gs_select(const uint32_t* MaxArr, uint64_t L, uint8_t* ModeArr) {
  uint64_t TotalModeNum = 0;     /* line 2 */
  uint64_t l = L;                /* line 3 */
  uint64_t j = 0, k = 0;         /* line 4 */
  while (l > 0) {                /* line 5 */
    uint32_t i;
    uint64_t pos = 0;
    for (i = 0; i <= 9; i++) {   /* line 6 */
      uint64_t n = GS_NUM[i], b = GS_BW[i];            /* line 7 */
      uint64_t mask = (((uint64_t)1) << b) - 1;        /* line 8 */
      pos = 0;                                         /* line 9 */
      uint64_t lim = n < l ? n : l;
      while (pos < lim && (uint64_t)MaxArr[j + pos] <= mask) /* line 10 */
        pos = pos + 1;                                 /* line 11 */
      if (pos == n || pos == l) break;                 /* lines 13-14 */
    }
    l = l - pos;                 /* line 17 */
    j = j + pos;
    if (ModeArr) ModeArr[k] = (uint8_t)i; /* line 18 */
    k = k + 1;
    TotalModeNum = TotalModeNum + 1;      /* line 19 */
  }
  return TotalModeNum;
}

static int gs_encode(const uint32_t* x, uint32_t n, gco_stream* out) {
  uint64_t Q = ceil_div(n, 4);
  uint32_t* q = make_quads(x, n, Q);
  uint32_t* M = (uint32_t*)malloc((size_t)(Q ? Q : 1) * 4);
  uint8_t* modes = (uint8_t*)malloc((size_t)(Q ? Q : 1));
  if (!q || !M || !modes) return GCO_ERR_NOMEM;
  for (uint64_t j = 0; j < Q; j++) M[j] = gco_quad_max(q + 4 * j);
  uint64_t T = gco_gs_select(M, Q, modes);
  out->ctrl_bytes = ceil_div(T, 2);
  out->ctrl = (uint8_t*)calloc((size_t)(out->ctrl_bytes ? out->ctrl_bytes : 1), 1);
  out->nvec = T;
  out->data = (uint32_t*)calloc((size_t)(4 * (T ? T : 1)), 4);
  if (!out->ctrl || !out->data) return GCO_ERR_NOMEM;
  /* control: 4-bit selectors, low nibble first (A6) */
  for (uint64_t s = 0; s < T; s++) out->ctrl[s >> 1] |= (uint8_t)(modes[s] << (4 * (s & 1)));
  /* data: one 128-bit vector per selector, "Packing original integers
   * into vectors": loop NUM times, ints at [t*BW, (t+1)*BW) (A7). */
  uint64_t j0 = 0;
  for (uint64_t s = 0; s < T; s++) {
    uint32_t NUM = GS_NUM[modes[s]], BW = GS_BW[modes[s]];
    uint64_t c = Q - j0 < NUM ? Q - j0 : NUM;
    for (uint64_t t = 0; t < c; t++)
      for (int k = 0; k < 4; k++) out->data[4 * s + k] |= q[4 * (j0 + t) + k] << (t * BW);
    j0 += c;
  }
  free(q);
  free(M);
  free(modes);
  return GCO_OK;
}

/* Decoding procedure P:L262-267 §4.3: read a selector, decode one vector,
 * advance ModePos by 4 bits and DataPos by 128 bits. */
static int gs_decode(uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes, const uint32_t* data,
                     uint64_t nvec, uint32_t* q) {
  uint64_t Q = ceil_div(n, 4), done = 0, s = 0;
  while (done < Q) {
    if ((s >> 1) >= ctrl_bytes) return GCO_ERR_TRUNCATED;
    uint32_t SEL = (ctrl[s >> 1] >> (4 * (s & 1))) & 15;
    if (SEL > 9) return GCO_ERR_MALFORMED;
    if (s >= nvec) return GCO_ERR_TRUNCATED;
    uint32_t NUM = GS_NUM[SEL], BW = GS_BW[SEL];
    uint64_t c = Q - done < NUM ? Q - done : NUM; /* A8 */
    for (uint64_t t = 0; t < c; t++)
      for (int k = 0; k < 4; k++)
        q[4 * (done + t) + k] = (data[4 * s + k] >> (t * BW)) & mask_bits(BW);
    done += c;
    s++;
  }
  return GCO_OK;
}

/* ------------------------------------------------------------------ */
/* Group-Scheme, §5, Table IV, Eq. (1) and (2)             */
/* ------------------------------------------------------------------ */

static uint32_t gsc_cg(uint32_t variant) { return 1u << (variant & 3); }
static uint32_t gsc_kind(uint32_t variant) { return (variant >> 2) & 3; } /* 0 B, 1 CU, 2 IU */

/* Eq. (1): ValueOfLD = ceil(width/CG) - 1 (binary) or ceil(width/CG)
 * (unary).  The outer ceiling is forced by the §5.1 example (A12). */
uint32_t gco_gsc_ld(uint32_t quadmax, uint32_t variant) {
  uint32_t CG = gsc_cg(variant);
  uint32_t units = (gco_width(quadmax) + CG - 1) / CG;
  return gsc_kind(variant) == 0 ? units - 1 : units;
}

/* Eq. (2). */
uint32_t gco_gsc_bw(uint32_t ld, uint32_t variant) {
  uint32_t CG = gsc_cg(variant);
  return gsc_kind(variant) == 0 ? CG * (ld + 1) : CG * ld;
}

static int gsc_valid_variant(uint32_t variant) {
  if (variant > 15) return 0;
  uint32_t kind = gsc_kind(variant);
  if (kind > 2) return 0;
  if (kind == 2 && gsc_cg(variant) < 4) return 0; /* IU only for CG 4 and 8 */
  return 1;
}

/* Binary LD field width 5 - log2 CG and packing (A18):
 * CG=1 three 5-bit fields per 16-bit LE unit; CG=2 two 4-bit per byte;
 * CG=4 two 3-bit per byte; CG=8 four 2-bit per byte; LSB-first. */
static void bin_field_locate(uint32_t CG, uint64_t j, uint64_t* byte, uint32_t* shift,
                             uint32_t* width16) {
  switch (CG) {
    case 1: *byte = 2 * (j / 3); *shift = 5 * (uint32_t)(j % 3); *width16 = 1; break;
    case 2: *byte = j / 2; *shift = 4 * (uint32_t)(j % 2); *width16 = 0; break;
    case 4: *byte = j / 2; *shift = 3 * (uint32_t)(j % 2); *width16 = 0; break;
    default: *byte = j / 4; *shift = 2 * (uint32_t)(j % 4); *width16 = 0; break;
  }
}

static uint64_t bin_ctrl_bytes(uint32_t CG, uint64_t Q) {
  switch (CG) {
    case 1: return 2 * ceil_div(Q, 3);
    case 2: return ceil_div(Q, 2);
    case 4: return ceil_div(Q, 2);
    default: return ceil_div(Q, 4);
  }
}

/* Unary control bit p: byte p>>3, bit 7-(p&7) (MSB-first, A16). */
static uint32_t ubit_get(const uint8_t* c, uint64_t p) { return (c[p >> 3] >> (7 - (p & 7))) & 1u; }

static int ubit_put(bytebuf* b, uint64_t* p, uint32_t bit) {
  if (bb_reserve(b, (*p >> 3) + 1)) return -1;
  if (b->n < (*p >> 3) + 1) b->n = (*p >> 3) + 1;
  if (bit) b->p[*p >> 3] |= (uint8_t)(0x80u >> (*p & 7));
  (*p)++;
  return 0;
}

static int gsc_encode(uint32_t variant, const uint32_t* x, uint32_t n, gco_stream* out) {
  uint32_t CG = gsc_cg(variant), kind = gsc_kind(variant);
  uint64_t Q = ceil_div(n, 4);
  uint32_t* q = make_quads(x, n, Q);
  uint32_t* BW = (uint32_t*)malloc((size_t)(Q ? Q : 1) * 4);
  uint32_t* LD = (uint32_t*)malloc((size_t)(Q ? Q : 1) * 4);
  if (!q || !BW || !LD) return GCO_ERR_NOMEM;
  uint64_t total_bits = 0;
  for (uint64_t j = 0; j < Q; j++) {
    LD[j] = gco_gsc_ld(gco_quad_max(q + 4 * j), variant); /* Eq. (1) */
    BW[j] = gco_gsc_bw(LD[j], variant);                    /* low ceil(w/CG)*CG bits */
    total_bits += BW[j];
  }
  /* control area (§5.2.1) */
  bytebuf cb = {0, 0, 0};
  if (kind == 0) {
    uint64_t nb = bin_ctrl_bytes(CG, Q);
    if (bb_reserve(&cb, nb ? nb : 1)) return GCO_ERR_NOMEM;
    cb.n = nb;
    for (uint64_t j = 0; j < Q; j++) {
      uint64_t byte; uint32_t sh, w16;
      bin_field_locate(CG, j, &byte, &sh, &w16);
      uint32_t unit = w16 ? (uint32_t)cb.p[byte] | ((uint32_t)cb.p[byte + 1] << 8) : cb.p[byte];
      unit |= LD[j] << sh;
      cb.p[byte] = (uint8_t)(unit & 0xFF);
      if (w16) cb.p[byte + 1] = (uint8_t)(unit >> 8);
    }
  } else if (kind == 1) {
    /* complete unary: (LD-1) ones then a 0, may cross bytes (A15). */
    uint64_t p = 0;
    for (uint64_t j = 0; j < Q; j++) {
      for (uint32_t t = 0; t + 1 < LD[j]; t++)
        if (ubit_put(&cb, &p, 1)) return GCO_ERR_NOMEM;
      if (ubit_put(&cb, &p, 0)) return GCO_ERR_NOMEM;
    }
  } else {
    /* incomplete unary: a code never crosses a byte; the rest of a byte is
     * filled with 1s (A17). */
    uint64_t p = 0;
    for (uint64_t j = 0; j < Q; j++) {
      uint32_t used = (uint32_t)(p & 7);
      if (used != 0 && used + LD[j] > 8) {
        while ((p & 7) != 0)
          if (ubit_put(&cb, &p, 1)) return GCO_ERR_NOMEM;
      }
      for (uint32_t t = 0; t + 1 < LD[j]; t++)
        if (ubit_put(&cb, &p, 1)) return GCO_ERR_NOMEM;
      if (ubit_put(&cb, &p, 0)) return GCO_ERR_NOMEM;
    }
    while ((p & 7) != 0)
      if (ubit_put(&cb, &p, 1)) return GCO_ERR_NOMEM;
  }
  out->ctrl = cb.p ? cb.p : (uint8_t*)calloc(1, 1);
  out->ctrl_bytes = cb.n;
  /* data area: one continuous lane bitstream, whole vectors (A19). */
  out->nvec = ceil_div(total_bits, 32);
  out->data = (uint32_t*)calloc((size_t)(4 * (out->nvec + 1)), 4);
  if (!out->data) return GCO_ERR_NOMEM;
  uint64_t pos = 0;
  for (uint64_t j = 0; j < Q; j++) {
    put_quad(out->data, 0, pos, BW[j], q + 4 * j);
    pos += BW[j];
  }
  free(q);
  free(BW);
  free(LD);
  return GCO_OK;
}

/* §5.2.3: read an LD, BW = Eq. (2), extract four BW-bit ints. */
static int gsc_decode(uint32_t variant, uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes,
                      const uint32_t* data, uint64_t nvec, uint32_t* q) {
  uint32_t CG = gsc_cg(variant), kind = gsc_kind(variant);
  uint64_t Q = ceil_div(n, 4);
  uint64_t p = 0, pos = 0;
  uint32_t max_units = 32 / CG;
  for (uint64_t j = 0; j < Q; j++) {
    uint32_t ld;
    if (kind == 0) {
      uint64_t byte; uint32_t sh, w16;
      bin_field_locate(CG, j, &byte, &sh, &w16);
      if (byte + (w16 ? 1 : 0) >= ctrl_bytes) return GCO_ERR_TRUNCATED;
      uint32_t unit = w16 ? (uint32_t)ctrl[byte] | ((uint32_t)ctrl[byte + 1] << 8) : ctrl[byte];
      uint32_t fw = 5 - (variant & 3);
      ld = (unit >> sh) & mask_bits(fw);
    } else if (kind == 1) {
      uint32_t ones = 0;
      for (;;) {
        if ((p >> 3) >= ctrl_bytes) return GCO_ERR_TRUNCATED;
        uint32_t bit = ubit_get(ctrl, p);
        p++;
        if (bit == 0) break;
        ones++;
        if (ones >= max_units) return GCO_ERR_MALFORMED;
      }
      ld = ones + 1;
    } else {
      uint32_t o = (uint32_t)(p & 7);
      if (o != 0) {
        if ((p >> 3) >= ctrl_bytes) return GCO_ERR_TRUNCATED;
        uint32_t rest_all_ones = 1;
        for (uint32_t t = o; t < 8; t++)
          if (ubit_get(ctrl, (p & ~(uint64_t)7) + t) == 0) rest_all_ones = 0;
        if (rest_all_ones) p += 8 - o; /* padding to the byte end */
      }
      uint32_t ones = 0;
      for (;;) {
        if ((p >> 3) >= ctrl_bytes) return GCO_ERR_TRUNCATED;
        uint32_t bit = ubit_get(ctrl, p);
        p++;
        if (bit == 0) break;
        ones++;
        if ((p & 7) == 0) return GCO_ERR_MALFORMED; /* a code may not cross a byte */
      }
      ld = ones + 1;
      if (ld > max_units) return GCO_ERR_MALFORMED;
    }
    uint32_t bw = gco_gsc_bw(ld, variant); /* Eq. (2) */
    uint64_t end_vec = ceil_div(pos + bw, 32);
    if (end_vec > nvec) return GCO_ERR_TRUNCATED;
    get_quad(data, 0, pos, bw, q + 4 * j);
    pos += bw;
  }
  return GCO_OK;
}

/* ------------------------------------------------------------------ */
/* Group-AFOR, §6.1                                        */
/* ------------------------------------------------------------------ */

/* Frames of {8,16,32} quads ({32,64,128} ints), one bw per frame, chosen by
 * dynamic programming over the quad max array.  Objective (A23):
 * 8 header bits + 128*ceil(L*bw/32) data bits per frame.  Frames start at
 * multiples of 8 quads; L tried in the order 32, 16, 8, replaced only on a
 * strict improvement (A24).  widths[] has Qp = 8*ceil(Q/8) entries (A25). */
uint64_t gco_afor_partition(const uint32_t* widths, uint64_t Qp, uint8_t* frame_len,
                            uint8_t* frame_bw, uint64_t* n_frames) {
  uint64_t nslots = Qp / 8 + 1;
  uint64_t* C = (uint64_t*)malloc((size_t)nslots * 8);
  uint8_t* choice = (uint8_t*)malloc((size_t)nslots);
  if (!C || !choice) {
    free(C);
    free(choice);
    return (uint64_t)-1;
  }
  C[Qp / 8] = 0;
  for (int64_t i = (int64_t)Qp - 8; i >= 0; i -= 8) {
    uint64_t best = (uint64_t)-1;
    uint8_t bl = 8;
    static const uint32_t Ls[3] = {32, 16, 8};
    for (int t = 0; t < 3; t++) {
      uint32_t L = Ls[t];
      if ((uint64_t)i + L > Qp) continue;
      uint32_t bw = 1;
      for (uint32_t u = 0; u < L; u++)
        if (widths[i + u] > bw) bw = widths[i + u];
      uint64_t c = 8 + 128 * ceil_div((uint64_t)L * bw, 32) + C[(i + L) / 8];
      if (c < best) {
        best = c;
        bl = (uint8_t)L;
      }
    }
    C[i / 8] = best;
    choice[i / 8] = bl;
  }
  uint64_t f = 0;
  for (uint64_t i = 0; i < Qp; i += choice[i / 8]) {
    uint32_t L = choice[i / 8], bw = 1;
    for (uint32_t u = 0; u < L; u++)
      if (widths[i + u] > bw) bw = widths[i + u];
    if (frame_len) frame_len[f] = (uint8_t)L;
    if (frame_bw) frame_bw[f] = (uint8_t)bw;
    f++;
  }
  if (n_frames) *n_frames = f;
  uint64_t cost = C[0];
  free(C);
  free(choice);
  return cost;
}

static int afor_encode(const uint32_t* x, uint32_t n, gco_stream* out) {
  uint64_t Q = ceil_div(n, 4), Qp = 8 * ceil_div(Q, 8);
  uint32_t* q = make_quads(x, n, Qp); /* padded quads are zero (A25) */
  uint32_t* w = (uint32_t*)malloc((size_t)(Qp ? Qp : 1) * 4);
  uint8_t* fl = (uint8_t*)malloc((size_t)(Qp / 8 + 1));
  uint8_t* fb = (uint8_t*)malloc((size_t)(Qp / 8 + 1));
  if (!q || !w || !fl || !fb) return GCO_ERR_NOMEM;
  for (uint64_t j = 0; j < Qp; j++) w[j] = gco_width(gco_quad_max(q + 4 * j));
  uint64_t nf = 0;
  gco_afor_partition(w, Qp, fl, fb, &nf);
  uint64_t nvec = 0;
  for (uint64_t f = 0; f < nf; f++) nvec += ceil_div((uint64_t)fl[f] * fb[f], 32);
  out->ctrl_bytes = nf;
  out->ctrl = (uint8_t*)calloc((size_t)(nf ? nf : 1), 1);
  out->nvec = nvec;
  out->data = (uint32_t*)calloc((size_t)(4 * (nvec + 1)), 4);
  if (!out->ctrl || !out->data) return GCO_ERR_NOMEM;
  uint64_t j = 0, vec = 0;
  for (uint64_t f = 0; f < nf; f++) {
    uint32_t L = fl[f], bw = fb[f];
    uint32_t code = L == 8 ? 0 : (L == 16 ? 1 : 2);
    out->ctrl[f] = (uint8_t)(code | ((bw - 1) << 2)); /* A22 header byte */
    for (uint32_t t = 0; t < L; t++) put_quad(out->data, vec, (uint64_t)t * bw, bw, q + 4 * (j + t));
    j += L;
    vec += ceil_div((uint64_t)L * bw, 32); /* each frame starts a fresh vector */
  }
  free(q);
  free(w);
  free(fl);
  free(fb);
  return GCO_OK;
}

static int afor_decode(uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes, const uint32_t* data,
                       uint64_t nvec, uint32_t* q) {
  uint64_t Q = ceil_div(n, 4), covered = 0, f = 0, vec = 0;
  while (covered < Q) {
    if (f >= ctrl_bytes) return GCO_ERR_TRUNCATED;
    uint32_t h = ctrl[f];
    uint32_t code = h & 3;
    if (code == 3 || (h & 0x80)) return GCO_ERR_MALFORMED;
    uint32_t L = 8u << code, bw = ((h >> 2) & 31) + 1;
    uint64_t fv = ceil_div((uint64_t)L * bw, 32);
    if (vec + fv > nvec) return GCO_ERR_TRUNCATED;
    for (uint32_t t = 0; t < L; t++)
      if (covered + t < Q) get_quad(data, vec, (uint64_t)t * bw, bw, q + 4 * (covered + t));
    covered += L;
    vec += fv;
    f++;
  }
  return GCO_OK;
}

/* ------------------------------------------------------------------ */
/* Group-PFD, §6.2                                         */
/* ------------------------------------------------------------------ */

/* Step 2: on the frame's MaxArr entries, the minimum b such that the
 * exception ratio is below zeta; "below" read as <= with the exact rational
 * comparison cnt*den <= num*q (A28). */
uint32_t gco_pfd_choose_b(const uint32_t* frame_qmax, uint32_t q, uint32_t zeta_num,
                          uint32_t zeta_den) {
  for (uint32_t b = 1; b <= 32; b++) {
    uint64_t cnt = 0;
    for (uint32_t j = 0; j < q; j++)
      if (gco_width(frame_qmax[j]) > b) cnt++;
    if (cnt * (uint64_t)zeta_den <= (uint64_t)zeta_num * q) return b;
  }
  return 32;
}

static uint32_t pfd_pos_bytes(uint32_t F) { return 4 * F <= 256 ? 1 : 2; }

static int pfd_encode(uint32_t F, uint32_t zn, uint32_t zd, const uint32_t* x, uint32_t n,
                      gco_stream* out) {
  uint64_t Q = ceil_div(n, 4);
  uint64_t nf = ceil_div(Q, F);
  uint32_t* q = make_quads(x, n, Q);
  uint32_t* M = (uint32_t*)malloc((size_t)(Q ? Q : 1) * 4);
  if (!q || !M) return GCO_ERR_NOMEM;
  for (uint64_t j = 0; j < Q; j++) M[j] = gco_quad_max(q + 4 * j); /* Step 1 */
  uint32_t pb = pfd_pos_bytes(F);
  bytebuf cb = {0, 0, 0}, eb = {0, 0, 0};
  uint64_t nvec = 0;
  uint32_t* bs = (uint32_t*)malloc((size_t)(nf ? nf : 1) * 4);
  if (!bs) return GCO_ERR_NOMEM;
  for (uint64_t f = 0; f < nf; f++) {
    uint32_t qf = (uint32_t)((Q - f * F) < F ? (Q - f * F) : F); /* A33 tail frame */
    bs[f] = gco_pfd_choose_b(M + f * F, qf, zn, zd);             /* Step 2 */
    nvec += ceil_div((uint64_t)qf * bs[f], 32);
  }
  out->nvec = nvec;
  out->data = (uint32_t*)calloc((size_t)(4 * (nvec + 1)), 4);
  if (!out->data) return GCO_ERR_NOMEM;
  uint64_t vec = 0;
  for (uint64_t f = 0; f < nf; f++) {
    uint32_t qf = (uint32_t)((Q - f * F) < F ? (Q - f * F) : F), b = bs[f];
    const uint32_t* fq = q + 4 * f * F;
    /* Step 3: every int of the frame whose width exceeds b is an
     * exception (A29), in ascending in-frame position p = 4j+k. */
    uint32_t count = 0, maxv = 0;
    for (uint32_t p = 0; p < 4 * qf; p++)
      if (gco_width(fq[p]) > b) {
        count++;
        if (fq[p] > maxv) maxv = fq[p];
      }
    /* Step 4: exceptions stored at the most economical of 8/16/32. */
    uint32_t wcode = 0, wbytes = 0;
    if (count > 0) {
      if (maxv <= 0xFFu) { wcode = 1; wbytes = 1; }
      else if (maxv <= 0xFFFFu) { wcode = 2; wbytes = 2; }
      else { wcode = 3; wbytes = 4; }
    }
    /* batch-form header {b, wcode, count16} (A31) */
    if (bb_push(&cb, (uint8_t)b) || bb_push(&cb, (uint8_t)wcode) ||
        bb_push(&cb, (uint8_t)(count & 0xFF)) || bb_push(&cb, (uint8_t)(count >> 8)))
      return GCO_ERR_NOMEM;
    for (uint32_t p = 0; p < 4 * qf; p++)
      if (gco_width(fq[p]) > b) {
        if (bb_push(&eb, (uint8_t)(p & 0xFF))) return GCO_ERR_NOMEM;
        if (pb == 2 && bb_push(&eb, (uint8_t)(p >> 8))) return GCO_ERR_NOMEM;
      }
    for (uint32_t p = 0; p < 4 * qf; p++)
      if (gco_width(fq[p]) > b)
        for (uint32_t t = 0; t < wbytes; t++)
          if (bb_push(&eb, (uint8_t)((fq[p] >> (8 * t)) & 0xFF))) return GCO_ERR_NOMEM;
    /* the normal array: low b bits of all 4q ints, fresh vector per frame */
    for (uint32_t j = 0; j < qf; j++) {
      uint32_t lowq[4];
      for (int k = 0; k < 4; k++) lowq[k] = fq[4 * j + k] & mask_bits(b);
      put_quad(out->data, vec, (uint64_t)j * b, b, lowq);
    }
    vec += ceil_div((uint64_t)qf * b, 32);
  }
  out->ctrl = cb.p ? cb.p : (uint8_t*)calloc(1, 1);
  out->ctrl_bytes = cb.n;
  out->exc = eb.p ? eb.p : (uint8_t*)calloc(1, 1);
  out->exc_bytes = eb.n;
  free(q);
  free(M);
  free(bs);
  return GCO_OK;
}

/* Decoding: read b and the exception info, unpack the normal
 * array, write each exception into its position (overwrite, A30). */
static int pfd_decode(uint32_t F, uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes,
                      const uint32_t* data, uint64_t nvec, const uint8_t* exc, uint64_t exc_bytes,
                      uint32_t* q) {
  uint64_t Q = ceil_div(n, 4), nf = ceil_div(Q, F), vec = 0, e = 0;
  uint32_t pb = pfd_pos_bytes(F);
  for (uint64_t f = 0; f < nf; f++) {
    if (4 * f + 3 >= ctrl_bytes) return GCO_ERR_TRUNCATED;
    uint32_t b = ctrl[4 * f], wcode = ctrl[4 * f + 1];
    uint32_t count = (uint32_t)ctrl[4 * f + 2] | ((uint32_t)ctrl[4 * f + 3] << 8);
    uint32_t qf = (uint32_t)((Q - f * F) < F ? (Q - f * F) : F);
    if (b < 1 || b > 32 || wcode > 3 || count > 4 * qf || (count > 0 && wcode == 0))
      return GCO_ERR_MALFORMED;
    uint64_t fv = ceil_div((uint64_t)qf * b, 32);
    if (vec + fv > nvec) return GCO_ERR_TRUNCATED;
    for (uint32_t j = 0; j < qf; j++) get_quad(data, vec, (uint64_t)j * b, b, q + 4 * (f * F + j));
    uint32_t wbytes = wcode == 0 ? 0 : (wcode == 1 ? 1 : (wcode == 2 ? 2 : 4));
    uint64_t need = (uint64_t)count * (pb + wbytes);
    if (e + need > exc_bytes) return GCO_ERR_TRUNCATED;
    uint32_t prev = 0;
    for (uint32_t i = 0; i < count; i++) {
      uint32_t p = exc[e + (uint64_t)i * pb];
      if (pb == 2) p |= (uint32_t)exc[e + (uint64_t)i * pb + 1] << 8;
      if (p >= 4 * qf || (i > 0 && p <= prev)) return GCO_ERR_MALFORMED;
      prev = p;
      uint32_t v = 0;
      for (uint32_t t = 0; t < wbytes; t++)
        v |= (uint32_t)exc[e + (uint64_t)count * pb + (uint64_t)i * wbytes + t] << (8 * t);
      q[4 * f * F + p] = v; /* Step 3: overwrite */
    }
    e += need;
    vec += fv;
  }
  return GCO_OK;
}

/* ------------------------------------------------------------------ */
/* per-list dispatch                                                    */
/* ------------------------------------------------------------------ */

/* ------------------------------------------------------------------ */
/* Variable Byte, §2.3: 7-bit groups, least significant */
/* first; "the most significant bit of a byte is the continuation bit":  */
/* MSB = 1 marks the LAST byte of an integer.  The byte stream is the     */
/* control area; there is no data area.                                   */
/* ------------------------------------------------------------------ */
static int vb_encode(const uint32_t* x, uint32_t n, gco_stream* out) {
  bytebuf cb = {0, 0, 0};
  for (uint32_t i = 0; i < n; i++) {
    uint32_t v = x[i];
    while (v >= 128) {
      if (bb_push(&cb, (uint8_t)(v & 127))) return GCO_ERR_NOMEM; /* continuation */
      v >>= 7;
    }
    if (bb_push(&cb, (uint8_t)(v | 128))) return GCO_ERR_NOMEM;   /* last byte */
  }
  out->ctrl = cb.p ? cb.p : (uint8_t*)calloc(1, 1);
  out->ctrl_bytes = cb.n;
  out->nvec = 0;
  out->data = (uint32_t*)calloc(4, 4);
  return out->data ? GCO_OK : GCO_ERR_NOMEM;
}

static int vb_decode(uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes, uint32_t* q) {
  uint64_t p = 0;
  for (uint32_t i = 0; i < n; i++) {
    uint64_t v = 0;
    uint32_t k = 0;
    for (;;) {
      if (p >= ctrl_bytes) return GCO_ERR_TRUNCATED; /* stream ends mid-integer */
      if (k == 5) return GCO_ERR_MALFORMED;          /* > 5 bytes without terminator */
      uint8_t b = ctrl[p++];
      v |= (uint64_t)(b & 127) << (7 * k);
      k++;
      if (b & 128) break;
    }
    q[i] = (uint32_t)v;
  }
  return GCO_OK;
}

static int check_params(const gco_params* p) {
  if (!p) return GCO_ERR_ARG;
  switch (p->codec) {
    case GCO_VARBYTE:
    case GCO_GROUP_SIMPLE:
    case GCO_GROUP_AFOR:
      return GCO_OK;
    case GCO_GROUP_SCHEME:
      return gsc_valid_variant(p->variant) ? GCO_OK : GCO_ERR_VARIANT;
    case GCO_GROUP_PFD:
      if (p->frame_quads == 0 || p->frame_quads > 16384) return GCO_ERR_ARG;
      if (p->zeta_den == 0) return GCO_ERR_ARG;
      return GCO_OK;
    default:
      return GCO_ERR_CODEC;
  }
}

int gco_encode_list(const gco_params* p, const uint32_t* x, uint32_t n, gco_stream* out) {
  int rc = check_params(p);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  switch (p->codec) {
    case GCO_VARBYTE: rc = vb_encode(x, n, out); break;
    case GCO_GROUP_SIMPLE: rc = gs_encode(x, n, out); break;
    case GCO_GROUP_SCHEME: rc = gsc_encode(p->variant, x, n, out); break;
    case GCO_GROUP_AFOR: rc = afor_encode(x, n, out); break;
    default: rc = pfd_encode(p->frame_quads, p->zeta_num, p->zeta_den, x, n, out); break;
  }
  if (!out->exc) out->exc = (uint8_t*)calloc(1, 1);
  return rc;
}

int gco_decode_list(const gco_params* p, uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes,
                    const uint32_t* data, uint64_t nvec, const uint8_t* exc, uint64_t exc_bytes,
                    uint32_t* out) {
  int rc = check_params(p);
  if (rc) return rc;
  uint64_t Q = ceil_div(n, 4);
  uint32_t* q = (uint32_t*)calloc((size_t)(4 * (Q ? Q : 1)), 4);
  if (!q) return GCO_ERR_NOMEM;
  switch (p->codec) {
    case GCO_VARBYTE: rc = vb_decode(n, ctrl, ctrl_bytes, q); break;
    case GCO_GROUP_SIMPLE: rc = gs_decode(n, ctrl, ctrl_bytes, data, nvec, q); break;
    case GCO_GROUP_SCHEME: rc = gsc_decode(p->variant, n, ctrl, ctrl_bytes, data, nvec, q); break;
    case GCO_GROUP_AFOR: rc = afor_decode(n, ctrl, ctrl_bytes, data, nvec, q); break;
    default: rc = pfd_decode(p->frame_quads, n, ctrl, ctrl_bytes, data, nvec, exc, exc_bytes, q); break;
  }
  if (rc == GCO_OK)
    for (uint32_t i = 0; i < n; i++) out[i] = q[i]; /* emit exactly n (A5) */
  free(q);
  return rc;
}

void gco_stream_free(gco_stream* s) {
  if (!s) return;
  free(s->ctrl);
  free(s->data);
  free(s->exc);
  memset(s, 0, sizeof(*s));
}

void gco_free(void* ptr) { free(ptr); }

/* ------------------------------------------------------------------ */
/* SPEC-compatible block: 16-byte header, control, data     */
/* ------------------------------------------------------------------ */

static void put_le32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static uint32_t get_le32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

int gco_encode_block(const gco_params* p, int delta, const uint32_t* x, uint32_t n,
                     uint8_t** block, uint64_t* block_bytes) {
  int rc = check_params(p);
  if (rc) return rc;
  uint32_t* g = (uint32_t*)malloc((size_t)(n ? n : 1) * 4);
  if (!g) return GCO_ERR_NOMEM;
  for (uint32_t i = 0; i < n; i++) {
    if (delta) {
      if (i > 0 && x[i] <= x[i - 1]) {
        free(g);
        return GCO_ERR_NOT_INCREASING;
      }
      g[i] = i == 0 ? x[0] : x[i] - x[i - 1]; /* P:L57 d-gap */
    } else {
      g[i] = x[i];
    }
  }
  gco_stream s;
  rc = gco_encode_list(p, g, n, &s);
  free(g);
  if (rc) return rc;
  /* PFD's SPEC control record interleaves the exception payload per frame
   * (S:L471): [b][wcode][count16][positions][values]. */
  bytebuf c = {0, 0, 0};
  if (p->codec == GCO_GROUP_PFD) {
    uint64_t e = 0, pb = pfd_pos_bytes(p->frame_quads);
    for (uint64_t f = 0; 4 * f < s.ctrl_bytes; f++) {
      uint32_t wcode = s.ctrl[4 * f + 1];
      uint32_t count = (uint32_t)s.ctrl[4 * f + 2] | ((uint32_t)s.ctrl[4 * f + 3] << 8);
      uint32_t wbytes = wcode == 0 ? 0 : (wcode == 1 ? 1 : (wcode == 2 ? 2 : 4));
      for (int t = 0; t < 4; t++) bb_push(&c, s.ctrl[4 * f + t]);
      for (uint64_t t = 0; t < (uint64_t)count * (pb + wbytes); t++) bb_push(&c, s.exc[e + t]);
      e += (uint64_t)count * (pb + wbytes);
    }
  } else {
    for (uint64_t t = 0; t < s.ctrl_bytes; t++) bb_push(&c, s.ctrl[t]);
  }
  uint64_t data_offset = 16 * ceil_div(16 + c.n, 16);
  uint64_t total = data_offset + 16 * s.nvec;
  uint8_t* blk = (uint8_t*)calloc((size_t)total, 1);
  if (!blk) return GCO_ERR_NOMEM;
  memcpy(blk, "GCM1", 4);
  blk[4] = 1;
  blk[5] = (uint8_t)p->codec;
  blk[6] = (uint8_t)(delta ? 1 : 0);
  blk[7] = (uint8_t)(p->codec == GCO_GROUP_SCHEME ? p->variant : 0);
  put_le32(blk + 8, n);
  put_le32(blk + 12, (uint32_t)data_offset);
  if (c.n) memcpy(blk + 16, c.p, (size_t)c.n);
  for (uint64_t m = 0; m < 4 * s.nvec; m++) put_le32(blk + data_offset + 4 * m, s.data[m]);
  free(c.p);
  gco_stream_free(&s);
  *block = blk;
  *block_bytes = total;
  return GCO_OK;
}

int gco_decode_block(const uint8_t* blk, uint64_t nbytes, uint32_t frame_quads, uint32_t* out,
                     uint32_t out_cap, uint32_t* n_out) {
  if (nbytes < 16) return GCO_ERR_TRUNCATED;
  if (memcmp(blk, "GCM1", 4) != 0) return GCO_ERR_BAD_MAGIC;
  if (blk[4] != 1) return GCO_ERR_VERSION;
  gco_params p;
  p.codec = blk[5];
  p.variant = blk[7];
  p.frame_quads = frame_quads ? frame_quads : 32;
  p.zeta_num = 1;
  p.zeta_den = 10;
  int rc = check_params(&p);
  if (rc) return rc;
  if (p.codec != GCO_GROUP_SCHEME && p.variant != 0) return GCO_ERR_VARIANT;
  uint32_t n = get_le32(blk + 8), data_offset = get_le32(blk + 12);
  if (data_offset < 16 || (data_offset & 15) || data_offset > nbytes) return GCO_ERR_TRUNCATED;
  if (n > out_cap) return GCO_ERR_ARG;
  uint64_t nvec = (nbytes - data_offset) / 16;
  uint32_t* data = (uint32_t*)malloc((size_t)(4 * (nvec + 1)) * 4);
  if (!data) return GCO_ERR_NOMEM;
  for (uint64_t m = 0; m < 4 * nvec; m++) data[m] = get_le32(blk + data_offset + 4 * m);
  const uint8_t* ctrl = blk + 16;
  uint64_t ctrl_bytes = data_offset - 16;
  if (p.codec == GCO_GROUP_PFD) {
    /* split the interleaved record back into header + exception streams */
    uint64_t Q = ceil_div(n, 4), nf = ceil_div(Q, p.frame_quads), pb = pfd_pos_bytes(p.frame_quads);
    uint8_t* h = (uint8_t*)calloc((size_t)(4 * nf + 1), 1);
    bytebuf e = {0, 0, 0};
    uint64_t c = 0;
    for (uint64_t f = 0; f < nf; f++) {
      if (c + 4 > ctrl_bytes) {
        free(h); free(e.p); free(data);
        return GCO_ERR_TRUNCATED;
      }
      memcpy(h + 4 * f, ctrl + c, 4);
      uint32_t wcode = ctrl[c + 1], count = (uint32_t)ctrl[c + 2] | ((uint32_t)ctrl[c + 3] << 8);
      uint32_t wbytes = wcode == 0 ? 0 : (wcode == 1 ? 1 : (wcode == 2 ? 2 : 4));
      uint64_t len = (uint64_t)count * (pb + wbytes);
      c += 4;
      if (c + len > ctrl_bytes) {
        free(h); free(e.p); free(data);
        return GCO_ERR_TRUNCATED;
      }
      for (uint64_t t = 0; t < len; t++) bb_push(&e, ctrl[c + t]);
      c += len;
    }
    rc = gco_decode_list(&p, n, h, 4 * nf, data, nvec, e.p, e.n, out);
    free(h);
    free(e.p);
  } else {
    rc = gco_decode_list(&p, n, ctrl, ctrl_bytes, data, nvec, NULL, 0, out);
  }
  free(data);
  if (rc) return rc;
  if (blk[6] & 1) /* flags bit0: invert the d-gap */
    for (uint32_t i = 1; i < n; i++) out[i] = out[i] + out[i - 1];
  *n_out = n;
  return GCO_OK;
}

/* ------------------------------------------------------------------ */
/* batch: lists in order, each control area 4-B aligned */
/* ------------------------------------------------------------------ */

typedef struct {
  const gco_params* p;
  const uint32_t* values;
  const uint32_t* list_n;
  const uint64_t* in_off;
  int delta;
  uint64_t l0, l1;
  gco_stream* streams;
  int rc;
} enc_job;

static void* enc_worker(void* arg) {
  enc_job* J = (enc_job*)arg;
  J->rc = GCO_OK;
  for (uint64_t l = J->l0; l < J->l1 && J->rc == GCO_OK; l++) {
    uint32_t n = J->list_n[l];
    const uint32_t* x = J->values + J->in_off[l];
    uint32_t* g = (uint32_t*)malloc((size_t)(n ? n : 1) * 4);
    if (!g) {
      J->rc = GCO_ERR_NOMEM;
      break;
    }
    for (uint32_t i = 0; i < n; i++) {
      if (J->delta) {
        if (i > 0 && x[i] <= x[i - 1]) J->rc = GCO_ERR_NOT_INCREASING;
        g[i] = i == 0 ? x[0] : x[i] - x[i - 1];
      } else {
        g[i] = x[i];
      }
    }
    if (J->rc == GCO_OK) J->rc = gco_encode_list(J->p, g, n, &J->streams[l]);
    free(g);
  }
  return NULL;
}

/* split [0, n_lists) into `threads` contiguous ranges balanced by sum(n) */
static void split_lists(const uint32_t* list_n, uint64_t n_lists, int threads, uint64_t* bounds) {
  uint64_t total = 0;
  for (uint64_t l = 0; l < n_lists; l++) total += list_n[l];
  uint64_t acc = 0, l = 0;
  bounds[0] = 0;
  for (int t = 1; t < threads; t++) {
    uint64_t target = total * (uint64_t)t / (uint64_t)threads;
    while (l < n_lists && acc < target) acc += list_n[l++];
    bounds[t] = l;
  }
  bounds[threads] = n_lists;
}

int gco_encode_batch(const gco_params* p, const uint32_t* values, const uint32_t* list_n,
                     uint64_t n_lists, int delta, int threads, gco_batch* out) {
  int rc = check_params(p);
  if (rc) return rc;
  if (threads < 1) threads = 1;
  memset(out, 0, sizeof(*out));
  uint64_t* in_off = (uint64_t*)malloc((size_t)(n_lists + 1) * 8);
  gco_stream* st = (gco_stream*)calloc((size_t)(n_lists ? n_lists : 1), sizeof(gco_stream));
  if (!in_off || !st) return GCO_ERR_NOMEM;
  in_off[0] = 0;
  for (uint64_t l = 0; l < n_lists; l++) in_off[l + 1] = in_off[l] + list_n[l];
  uint64_t* bounds = (uint64_t*)malloc((size_t)(threads + 1) * 8);
  enc_job* jobs = (enc_job*)calloc((size_t)threads, sizeof(enc_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  split_lists(list_n, n_lists, threads, bounds);
  for (int t = 0; t < threads; t++) {
    jobs[t] = (enc_job){p, values, list_n, in_off, delta, bounds[t], bounds[t + 1], st, 0};
    pthread_create(&tid[t], NULL, enc_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; t++) {
    pthread_join(tid[t], NULL);
    if (jobs[t].rc && !rc) rc = jobs[t].rc;
  }
  free(bounds);
  free(jobs);
  free(tid);
  if (rc) {
    for (uint64_t l = 0; l < n_lists; l++) gco_stream_free(&st[l]);
    free(st);
    free(in_off);
    return rc;
  }
  out->n_lists = n_lists;
  out->list_n = (uint32_t*)malloc((size_t)(n_lists ? n_lists : 1) * 4);
  out->ctrl_off = (uint64_t*)malloc((size_t)(n_lists + 1) * 8);
  out->data_off = (uint64_t*)malloc((size_t)(n_lists + 1) * 8);
  out->exc_off = (uint64_t*)malloc((size_t)(n_lists + 1) * 8);
  out->out_off = (uint64_t*)malloc((size_t)(n_lists + 1) * 8);
  out->ctrl_off[0] = out->data_off[0] = out->exc_off[0] = out->out_off[0] = 0;
  for (uint64_t l = 0; l < n_lists; l++) {
    out->list_n[l] = list_n[l];
    out->ctrl_off[l + 1] = out->ctrl_off[l] + 4 * ceil_div(st[l].ctrl_bytes, 4);
    out->data_off[l + 1] = out->data_off[l] + st[l].nvec;
    out->exc_off[l + 1] = out->exc_off[l] + st[l].exc_bytes;
    out->out_off[l + 1] = out->out_off[l] + list_n[l];
  }
  out->ctrl_bytes = 16 * ceil_div(out->ctrl_off[n_lists], 16);
  out->data_vectors = out->data_off[n_lists];
  out->exc_bytes = 16 * ceil_div(out->exc_off[n_lists], 16);
  out->total_out = out->out_off[n_lists];
  out->ctrl = (uint8_t*)calloc((size_t)(out->ctrl_bytes + 16), 1);
  out->data = (uint32_t*)calloc((size_t)(4 * (out->data_vectors + 1)), 4);
  out->exc = (uint8_t*)calloc((size_t)(out->exc_bytes + 16), 1);
  for (uint64_t l = 0; l < n_lists; l++) {
    if (st[l].ctrl_bytes) memcpy(out->ctrl + out->ctrl_off[l], st[l].ctrl, (size_t)st[l].ctrl_bytes);
    if (st[l].nvec) memcpy(out->data + 4 * out->data_off[l], st[l].data, (size_t)(16 * st[l].nvec));
    if (st[l].exc_bytes) memcpy(out->exc + out->exc_off[l], st[l].exc, (size_t)st[l].exc_bytes);
    gco_stream_free(&st[l]);
  }
  free(st);
  free(in_off);
  return GCO_OK;
}

typedef struct {
  const gco_params* p;
  const gco_batch* b;
  int dgaps;
  uint64_t l0, l1;
  uint32_t* out;
  int rc;
  uint64_t bad;
} dec_job;

static void* dec_worker(void* arg) {
  dec_job* J = (dec_job*)arg;
  const gco_batch* b = J->b;
  J->rc = GCO_OK;
  for (uint64_t l = J->l0; l < J->l1; l++) {
    uint32_t n = b->list_n[l];
    uint32_t* o = J->out + b->out_off[l];
    int rc = gco_decode_list(J->p, n, b->ctrl + b->ctrl_off[l], b->ctrl_off[l + 1] - b->ctrl_off[l],
                             b->data + 4 * b->data_off[l], b->data_off[l + 1] - b->data_off[l],
                             b->exc + b->exc_off[l], b->exc_off[l + 1] - b->exc_off[l], o);
    if (rc) {
      J->rc = rc;
      J->bad = l;
      return NULL;
    }
    if (J->dgaps) /* d_i = (d_{i-1} + g_i) mod 2^32, restarting per list (A36) */
      for (uint32_t i = 1; i < n; i++) o[i] = o[i - 1] + o[i];
  }
  return NULL;
}

int gco_decode_batch(const gco_params* p, const gco_batch* b, int dgaps, int threads,
                     uint32_t* out, uint64_t* first_bad_list) {
  int rc = check_params(p);
  if (rc) return rc;
  if (threads < 1) threads = 1;
  uint64_t* bounds = (uint64_t*)malloc((size_t)(threads + 1) * 8);
  dec_job* jobs = (dec_job*)calloc((size_t)threads, sizeof(dec_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  split_lists(b->list_n, b->n_lists, threads, bounds);
  for (int t = 0; t < threads; t++) {
    jobs[t] = (dec_job){p, b, dgaps, bounds[t], bounds[t + 1], out, 0, 0};
    pthread_create(&tid[t], NULL, dec_worker, &jobs[t]);
  }
  uint64_t bad = (uint64_t)-1;
  for (int t = 0; t < threads; t++) {
    pthread_join(tid[t], NULL);
    if (jobs[t].rc && jobs[t].bad < bad) {
      bad = jobs[t].bad;
      rc = jobs[t].rc;
    }
  }
  if (first_bad_list) *first_bad_list = bad;
  free(bounds);
  free(jobs);
  free(tid);
  return rc;
}

void gco_batch_free(gco_batch* b) {
  if (!b) return;
  free(b->list_n);
  free(b->ctrl_off);
  free(b->data_off);
  free(b->exc_off);
  free(b->out_off);
  free(b->ctrl);
  free(b->data);
  free(b->exc);
  memset(b, 0, sizeof(*b));
}

/* ------------------------------------------------------------------ */
/* Skip pointers every 512 postings (§7.5; the entry format is   */
/* in gc_oracle.h).  Each list is walked group by group in stream order;  */
/* every group records the control bit that makes its owning word, its   */
/* raw quads, data lane-bits and exception bytes.                         */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t own_bit, q0, nq, dbits, ebytes;
} skip_grp;

/* the groups of one list (at most Q + 1 of them); returns the count or -1 */
static int64_t walk_list_groups(const gco_params* p, uint32_t n, const uint8_t* ctrl,
                                uint64_t ctrl_bytes, const uint8_t* exc, uint64_t exc_bytes,
                                skip_grp* g) {
  uint64_t Q = ceil_div(n, 4), q = 0;
  int64_t k = 0;
  if (p->codec == GCO_GROUP_SIMPLE) {
    for (uint64_t s = 0; q < Q; s++) {       /* selector s: bits [4s, 4s+4), one vector */
      if ((s >> 1) >= ctrl_bytes) return -1;
      uint32_t SEL = (ctrl[s >> 1] >> (4 * (s & 1))) & 15;
      if (SEL > 9) return -1;
      g[k] = (skip_grp){4 * s, q, GS_NUM[SEL], 32, 0};  /* one vector: 32 lane-bits */
      q += GS_NUM[SEL];
      k++;
    }
  } else if (p->codec == GCO_GROUP_SCHEME) {
    uint32_t CG = gsc_cg(p->variant), kind = gsc_kind(p->variant);
    uint64_t bitp = 0;
    for (uint64_t j = 0; j < Q; j++) {
      uint32_t ld, own;
      if (kind == 0) {
        uint64_t byte; uint32_t sh, w16;
        bin_field_locate(CG, j, &byte, &sh, &w16);
        if (byte + (w16 ? 1 : 0) >= ctrl_bytes) return -1;
        uint32_t unit = w16 ? (uint32_t)ctrl[byte] | ((uint32_t)ctrl[byte + 1] << 8) : ctrl[byte];
        ld = (unit >> sh) & mask_bits(5 - (p->variant & 3));
        own = (uint32_t)(8 * byte + sh);
      } else {
        if (kind == 2 && (bitp & 7)) {       /* incomplete unary: skip the byte's padding ones */
          uint32_t rest = 1;
          for (uint64_t t = bitp & 7; t < 8; t++)
            if (ubit_get(ctrl, (bitp & ~(uint64_t)7) + t) == 0) rest = 0;
          if (rest) bitp += 8 - (bitp & 7);
        }
        uint32_t ones = 0;
        for (;;) {
          if ((bitp >> 3) >= ctrl_bytes) return -1;
          uint32_t bit = ubit_get(ctrl, bitp);
          bitp++;
          if (bit == 0) break;
          ones++;
        }
        ld = ones + 1;
        own = (uint32_t)(bitp - 1);           /* the terminating 0 */
      }
      uint32_t bw = gco_gsc_bw(ld, p->variant);
      g[k] = (skip_grp){own, j, 1, bw, 0};
      k++;
    }
  } else if (p->codec == GCO_GROUP_AFOR) {
    for (uint64_t f = 0; q < Q; f++) {       /* header byte f */
      if (f >= ctrl_bytes) return -1;
      uint32_t h = ctrl[f], code = h & 3;
      if (code == 3) return -1;
      uint32_t L = 8u << code, bw = ((h >> 2) & 31) + 1;
      g[k] = (skip_grp){8 * f, q, L, 32 * ceil_div((uint64_t)L * bw, 32), 0};
      q += L;
      k++;
    }
  } else if (p->codec == GCO_GROUP_PFD) {
    uint32_t F = p->frame_quads, pb = pfd_pos_bytes(F);
    for (uint64_t f = 0; q < Q; f++) {       /* 4-byte header f */
      if (4 * f + 3 >= ctrl_bytes) return -1;
      uint32_t b = ctrl[4 * f], wcode = ctrl[4 * f + 1];
      uint32_t count = (uint32_t)ctrl[4 * f + 2] | ((uint32_t)ctrl[4 * f + 3] << 8);
      uint64_t qf = Q - q < F ? Q - q : F;
      uint32_t wbytes = wcode == 0 ? 0 : (wcode == 1 ? 1 : (wcode == 2 ? 2 : 4));
      if (b < 1 || b > 32) return -1;
      g[k] = (skip_grp){32 * f, q, F, 32 * ceil_div(qf * b, 32), (uint64_t)count * (pb + wbytes)};
      q += F;
      k++;
    }
  } else {
    return -1;
  }
  (void)exc;
  (void)exc_bytes;
  return k;
}

uint64_t gco_skip_entries(const gco_batch* b) {
  uint64_t t = 0;
  for (uint64_t l = 0; l < b->n_lists; l++) t += ceil_div(b->list_n[l], GCO_SKIP_DIST);
  return t;
}

int gco_build_skip(const gco_params* p, const gco_batch* b, uint64_t* skip_off,
                   gco_skip_entry* entries) {
  int rc = check_params(p);
  if (rc) return rc;
  if (p->codec == GCO_VARBYTE) return GCO_ERR_CODEC;
  uint64_t e = 0;
  for (uint64_t l = 0; l < b->n_lists; l++) {
    skip_off[l] = e;
    uint32_t n = b->list_n[l];
    if (n == 0) continue;
    uint64_t Q = ceil_div(n, 4);
    const uint8_t* ctrl = b->ctrl + b->ctrl_off[l];
    uint64_t cb = b->ctrl_off[l + 1] - b->ctrl_off[l];
    skip_grp* g = (skip_grp*)malloc((size_t)(Q + 2) * sizeof(skip_grp));
    uint32_t* x = (uint32_t*)malloc((size_t)n * 4);
    if (!g || !x) {
      free(g);
      free(x);
      return GCO_ERR_NOMEM;
    }
    int64_t ng = walk_list_groups(p, n, ctrl, cb, b->exc + b->exc_off[l],
                                  b->exc_off[l + 1] - b->exc_off[l], g);
    rc = ng < 0 ? GCO_ERR_MALFORMED
                : gco_decode_list(p, n, ctrl, cb, b->data + 4 * b->data_off[l],
                                  b->data_off[l + 1] - b->data_off[l], b->exc + b->exc_off[l],
                                  b->exc_off[l + 1] - b->exc_off[l], x);
    if (rc) {
      free(g);
      free(x);
      return rc;
    }
    uint32_t docid = 0;  /* running sum of the ints before the block, mod 2^32 */
    uint64_t gi = 0, t0 = 0, cq = 0, cd = 0, ce = 0;  /* groups owned by earlier words */
    for (uint64_t blk = 0; blk < ceil_div(n, GCO_SKIP_DIST); blk++) {
      for (uint64_t i = blk ? GCO_SKIP_DIST * (blk - 1) : 0; i < GCO_SKIP_DIST * blk; i++)
        docid += x[i];
      uint64_t q0 = 128 * blk;   /* the block's first quad */
      while (!(g[gi].q0 <= q0 && q0 < g[gi].q0 + g[gi].nq)) gi++;
      uint64_t word = g[gi].own_bit / 32;
      /* owners are in stream order, so the earlier words own a prefix of the groups */
      while ((int64_t)t0 < ng && g[t0].own_bit / 32 < word) {
        cq += g[t0].nq;
        cd += g[t0].dbits;
        ce += g[t0].ebytes;
        t0++;
      }
      gco_skip_entry* s = &entries[e++];
      memset(s, 0, sizeof(*s));
      s->word = (uint32_t)word;
      s->quads = (uint32_t)cq;
      s->data_bits = cd;
      s->exc_bytes = (uint32_t)ce;
      if (p->codec == GCO_GROUP_SCHEME && gsc_kind(p->variant) == 1)  /* closed form */
        s->data_bits = (uint64_t)gsc_cg(p->variant) * 32 * word;
      s->docid = docid;
    }
    free(g);
    free(x);
  }
  skip_off[b->n_lists] = e;
  return GCO_OK;
}
