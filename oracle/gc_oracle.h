/*
 * gc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU encoder/decoder for the Group formats of
 * Zhao et al., "A General SIMD-based Approach to Accelerating Compression
 * Algorithms" (arXiv 1502.01916; PAPER.md in the reference tree).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header, table or helper with
 * the product path (paper_1502_01916_b200/csrc); neither side includes the
 * other.  Every function cites the PAPER.md line ("P:L<n>") it follows; where
 * the paper is silent the reading is the one listed in DESIGN.md §3 (A-ids
 * follow SURVEY.md §8(c)).
 */
#ifndef GC_ORACLE_H
#define GC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Codec ids. */
#define GCO_VARBYTE 1
#define GCO_GROUP_SIMPLE 2
#define GCO_GROUP_SCHEME 3
#define GCO_GROUP_AFOR 4
#define GCO_GROUP_PFD 5

/* Error codes. */
#define GCO_OK 0
#define GCO_ERR_ARG 1
#define GCO_ERR_MALFORMED 2
#define GCO_ERR_TRUNCATED 3
#define GCO_ERR_BAD_MAGIC 4
#define GCO_ERR_VERSION 5
#define GCO_ERR_CODEC 6
#define GCO_ERR_VARIANT 7
#define GCO_ERR_NOMEM 8
#define GCO_ERR_NOT_INCREASING 9

typedef struct {
  int32_t codec;         /* GCO_GROUP_* */
  uint32_t variant;      /* Group-Scheme: bits0-1 log2 CG, bits2-3 LD kind (0 B, 1 CU, 2 IU) */
  uint32_t frame_quads;  /* Group-PFD frame length F in quads (32 default, A27) */
  uint32_t zeta_num;     /* Group-PFD exception threshold zeta = num/den (1/10 default, A28) */
  uint32_t zeta_den;
} gco_params;

/* One encoded list in batch form: control area, data area (4 x u32 per
 * 128-bit vector, component k of vector m at data[4m+k]), exception area. */
typedef struct {
  uint8_t* ctrl;
  uint64_t ctrl_bytes;
  uint32_t* data;
  uint64_t nvec;
  uint8_t* exc;
  uint64_t exc_bytes;
} gco_stream;

/* A packed batch (SURVEY §8(b) directory form). All arrays malloc'd by the
 * oracle when produced by gco_encode_batch; caller-owned when passed in. */
typedef struct {
  uint64_t n_lists;
  uint32_t* list_n;    /* [n_lists] */
  uint64_t* ctrl_off;  /* [n_lists+1] bytes, each 4-B aligned */
  uint64_t* data_off;  /* [n_lists+1] 16-B vectors */
  uint64_t* exc_off;   /* [n_lists+1] bytes */
  uint64_t* out_off;   /* [n_lists+1] ints */
  uint8_t* ctrl;
  uint64_t ctrl_bytes; /* buffer size, multiple of 16, >= ctrl_off[n_lists] */
  uint32_t* data;
  uint64_t data_vectors;
  uint8_t* exc;
  uint64_t exc_bytes;  /* buffer size, multiple of 16, >= exc_off[n_lists] */
  uint64_t total_out;
} gco_batch;

/* primitives exposed for the pin tests */
uint32_t gco_width(uint32_t x);
uint32_t gco_quad_max(const uint32_t* q4);
uint32_t gco_quad_or(const uint32_t* q4);
uint64_t gco_gs_select(const uint32_t* maxarr, uint64_t L, uint8_t* mode_arr);
uint32_t gco_gsc_ld(uint32_t quadmax, uint32_t variant);
uint32_t gco_gsc_bw(uint32_t ld, uint32_t variant);
uint64_t gco_afor_partition(const uint32_t* widths, uint64_t Qp, uint8_t* frame_len_quads,
                            uint8_t* frame_bw, uint64_t* n_frames);
uint32_t gco_pfd_choose_b(const uint32_t* frame_qmax, uint32_t q, uint32_t zeta_num,
                          uint32_t zeta_den);
int gco_pack_vertical(const uint32_t* quads, uint64_t Q, uint32_t bw, uint32_t* data,
                      uint64_t nvec);
int gco_unpack_vertical(const uint32_t* data, uint64_t nvec, uint32_t bw, uint64_t Q,
                        uint32_t* quads);

/* one list */
int gco_encode_list(const gco_params* p, const uint32_t* x, uint32_t n, gco_stream* out);
int gco_decode_list(const gco_params* p, uint32_t n, const uint8_t* ctrl, uint64_t ctrl_bytes,
                    const uint32_t* data, uint64_t nvec, const uint8_t* exc, uint64_t exc_bytes,
                    uint32_t* out);
void gco_stream_free(gco_stream* s);

/* SPEC-compatible self-describing block */
int gco_encode_block(const gco_params* p, int delta, const uint32_t* x, uint32_t n,
                     uint8_t** block, uint64_t* block_bytes);
int gco_decode_block(const uint8_t* block, uint64_t block_bytes, uint32_t frame_quads,
                     uint32_t* out, uint32_t out_cap, uint32_t* n_out);
void gco_free(void* ptr);

/* batch */
int gco_encode_batch(const gco_params* p, const uint32_t* values, const uint32_t* list_n,
                     uint64_t n_lists, int delta, int threads, gco_batch* out);
int gco_decode_batch(const gco_params* p, const gco_batch* b, int dgaps, int threads,
                     uint32_t* out, uint64_t* first_bad_list);
void gco_batch_free(gco_batch* b);

/* Skip pointers (§7.5: "skip list pointers for posting blocks. The skip distance
 * ... 512 postings"): one entry per block of 512 ints of every list -- block b covers the
 * list's ints [512b, 512b+512) -- saying where decoding of the block starts with nothing
 * before it.  Every group of a list is OWNED by one 32-bit control word (the word holding
 * its descriptor: Group-Simple selector, binary LD field, AFOR / PFD frame header; the
 * terminating 0 of a unary code).  An entry names the word owning the group of the block's
 * first quad (quad 128b) and the list's prefixes before that word: raw quads of the groups
 * owned by earlier words, data lane-bits (complete unary: CG x 32 x word, its closed form),
 * exception bytes (Group-PFD), and the docID before the block (the ints [0, 512b) summed
 * mod 2^32; 0 for block 0).  skip_off[l] = sum over lists l' < l of ceil(n_l' / 512). */
#define GCO_SKIP_DIST 512
typedef struct {
  uint64_t data_bits;
  uint32_t word, quads, exc_bytes, docid, pad[2];
} gco_skip_entry;
uint64_t gco_skip_entries(const gco_batch* b);  /* = skip_off[n_lists] */
int gco_build_skip(const gco_params* p, const gco_batch* b, uint64_t* skip_off,
                   gco_skip_entry* entries);

#ifdef __cplusplus
}
#endif
#endif
