/*
 * gc.h -- C ABI of the B200-native Group-format posting-list decoder.
 *
 * Operation (PAPER.md = arXiv 1502.01916):
 *   A batch of posting lists, each encoded in one of the paper's Group formats
 *   with the 4-way vertical layout (§2.1.2, §3.1) and the
 *   control area stored apart from the data area, is decoded back to
 *   exactly the stored uint32 integers ("decoders emit exactly n"):
 *     - Group-Simple          §4   (Table III; decoding P:L262-267)
 *     - Group-Scheme          §5   (Table IV; Eq.(1)-(2) P:L330, P:L338;
 *                                   binary / complete-unary / incomplete-unary LDs P:L312-318)
 *     - Group-AFOR            §6.1 (frames of {8,16,32} quads)
 *     - Group-PFD             §6.2 (decode steps 1-3; exceptions overwrite
 *                                   their slot)
 *   gc_decode_dgaps additionally applies the inverse of the d-gap transform of
 *   P:L57 §2.1.1: d_i = (d_{i-1} + g_i) mod 2^32, restarting at every list.
 *
 * The exact byte layout (every reading of a silent or garbled passage) is
 * specified in DESIGN.md §3; it is the layout oracle/ encodes.
 *
 * Conventions
 *   - All functions are plain C; no C++, CUDA-runtime or torch types cross this
 *     boundary.  A CUDA stream is passed as `void*` (a cudaStream_t; NULL = the
 *     legacy default stream).
 *   - "device" pointers are CUDA global-memory pointers; "host" pointers are CPU
 *     pointers.  The caller owns every buffer.  The decode functions never
 *     allocate device memory and keep no global mutable state: calls on distinct
 *     workspaces are reentrant.
 *   - Decode functions validate their arguments on the host synchronously and
 *     return a gc_status; all GPU work is enqueued asynchronously on the stream.
 *     Errors found in the stream contents on the device never fault: they set
 *     sticky GC_DEV_* bits in the workspace (read them with
 *     gc_read_device_status).  The output of a batch with any such bit set is
 *     unspecified, but no access ever leaves the buffers described by the batch.
 */
#ifndef GC_H
#define GC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_ABI_VERSION 2

typedef enum {
  GC_OK = 0,
  GC_ERR_INVALID_ARGUMENT = 1,   /* null/misaligned pointer, inconsistent sizes           */
  GC_ERR_UNKNOWN_CODEC = 2,
  GC_ERR_BAD_VARIANT = 3,        /* Group-Scheme variant byte, PFD variant / frame length */
  GC_ERR_WORKSPACE_TOO_SMALL = 4,
  GC_ERR_UNSUPPORTED_DEVICE = 5, /* not a compute-capability 10.x (sm_100a) device       */
  GC_ERR_CUDA = 6,               /* a CUDA runtime call failed (launch, copy)            */
  GC_ERR_NOT_INCREASING = 7,     /* encoder: delta requested on a non-increasing list    */
  GC_ERR_NOMEM = 8               /* encoder: host allocation failed                      */
} gc_status;

/* Codec ids. */
/* GC_VARBYTE (P §2.3): the short-list fallback of P:L640 §7.5; its byte
 * stream (7-bit groups, least significant first, MSB = 1 on an int's last byte) is the
 * control area (ctrl / ctrl_off, byte offsets), there is no data area (data_off all 0);
 * decoded and encoded (host and GPU) as the other codecs. */
typedef enum { GC_VARBYTE = 1, GC_GROUP_SIMPLE = 2, GC_GROUP_SCHEME = 3, GC_GROUP_AFOR = 4,
               GC_GROUP_PFD = 5 } gc_codec;

/* Sticky device status bits, OR-ed by the kernels into the workspace. */
enum {
  GC_DEV_BAD_SELECTOR = 1u << 0,  /* Group-Simple selector nibble > 9 (Table III)               */
  GC_DEV_BAD_LD = 1u << 1,        /* unary LD longer than 32/CG units; IU byte with no code     */
  GC_DEV_BAD_FRAME = 1u << 2,     /* AFOR length code 3 or bit 7 set; PFD b not in 1..32,
                                     wcode > 3                                                  */
  GC_DEV_BAD_EXCEPTION = 1u << 3, /* PFD count > 4q, count>0 with wcode 0, position >= 4q or
                                     not strictly increasing                                    */
  GC_DEV_TRUNCATED = 1u << 4      /* a list needs control/data/exception bytes beyond its
                                     [off, next_off) range, or the directory is inconsistent   */
};

/*
 * A packed batch (layout in DESIGN.md §3.7).  The struct
 * itself is host memory, read only during the call.  Arrays are DEVICE
 * pointers for gc_decode / gc_decode_dgaps / gc_checksum and HOST pointers for
 * gc_decode_host.
 *
 *   list_n[n_lists]        logical ints of each list (0 allowed)
 *   ctrl_off[n_lists+1]    byte offset of each list's control area in ctrl;
 *                          every offset is a multiple of 4 (one 32-bit control
 *                          word never mixes two lists)
 *   data_off[n_lists+1]    offset of each list's data area in data, in 128-bit
 *                          vectors
 *   exc_off[n_lists+1]     byte offset of each list's exception area (Group-PFD;
 *                          may be NULL for other codecs)
 *   out_off[n_lists+1]     exclusive prefix sum of list_n (int offsets into out)
 *   ctrl, ctrl_bytes       control stream; 16-B aligned, ctrl_bytes % 16 == 0,
 *                          ctrl_bytes >= ctrl_off[n_lists]
 *   data, data_vectors     data stream of 128-bit vectors (component k of vector m
 *                          is the little-endian u32 at byte 16m+4k); 16-B aligned;
 *                          data_vectors < 2^42 (GC_ERR_INVALID_ARGUMENT otherwise)
 *   exc, exc_bytes         Group-PFD exception stream (positions then values per
 *                          frame); 16-B aligned, exc_bytes % 16 == 0, exc_bytes < 2^47;
 *                          NULL/0 for other codecs
 *   total_out              = out_off[n_lists] = sum of list_n
 *   variant                Group-Scheme: bits 0-1 log2 CG, bits 2-3 LD kind
 *                          (0 binary, 1 complete unary, 2 incomplete unary; IU
 *                          needs CG 4 or 8).  Group-PFD: 0, or 1 =
 *                          SIMD-BP128 as the special case of P:L424 (frames of F
 *                          quads packed at the width of the frame's largest int,
 *                          no exceptions; same frame format with count 0, a frame
 *                          with exceptions sets GC_DEV_BAD_EXCEPTION).  0 otherwise.
 *   pfd_frame_quads        Group-PFD frame length F in quadruples: 32 (default,
 *                          128 ints, u8 positions) or 128 (512 ints, u16 LE
 *                          positions).  Ignored by other codecs.
 */
typedef struct {
  int32_t codec; /* gc_codec */
  uint32_t variant;
  uint32_t pfd_frame_quads;
  uint32_t reserved;
  uint64_t n_lists;
  const uint32_t* list_n;
  const uint64_t* ctrl_off;
  const uint64_t* data_off;
  const uint64_t* exc_off;
  const uint64_t* out_off;
  const uint8_t* ctrl;
  uint64_t ctrl_bytes;
  const void* data;
  uint64_t data_vectors;
  const uint8_t* exc;
  uint64_t exc_bytes;
  uint64_t total_out;
} gc_batch;

/* Bytes of device workspace gc_decode / gc_decode_dgaps need for this batch
 * (tile descriptors, look-back words, counters, the status word).  Host only,
 * no launch.  Returns GC_ERR_INVALID_ARGUMENT on a null argument. */
gc_status gc_workspace_size(const gc_batch* b, uint64_t* bytes);

/* Decode every list of the batch into out (DEVICE, 16-B aligned, total_out
 * u32): out[out_off[l] + i] = the i-th integer of list l (the stored gaps or
 * TFs).  ws: DEVICE workspace of >= gc_workspace_size bytes, 16-B aligned,
 * exclusively owned by this call until the stream reaches it (it is reset
 * inside the call).  Asynchronous on `stream`. */
gc_status gc_decode(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes, void* stream);

/* As gc_decode, then the per-list inclusive prefix sum mod 2^32 that turns
 * d-gaps into docIDs, fused into the same pass. */
gc_status gc_decode_dgaps(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                          void* stream);

/* The same work as gc_decode (dgaps == 0) / gc_decode_dgaps (dgaps != 0) split into
 * its three stream-ordered stages, for callers that time or overlap them:
 *   GC_STAGE_RESET  zero the workspace (one cudaMemsetAsync),
 *   GC_STAGE_INDEX  the control-stream scan kernel (subsystem (a)),
 *   GC_STAGE_DECODE the fused unpack / patch / d-gap-scan / store kernel.
 * stage_mask is any OR of the three; stages run in that order.  Calling the three
 * stages one after another on one stream is exactly gc_decode / gc_decode_dgaps.
 * The decode stage is one cooperative launch of min(tiles, SMs x resident CTAs) CTAs, each
 * taking every grid-th 8192-int tile; the environment variable GC_DECODE_MAX_GRID, if set,
 * caps that grid (a test knob: many tiles per CTA at small sizes; same results).  The index
 * stage scans control tiles of 2048 words, or of 256 words for batches under 2^18 control
 * words (more CTAs for a small batch); GC_INDEX_TILE_WORDS=256|2048 forces one size (a test
 * knob: it changes gc_workspace_size too, so set it before sizing the workspace). */
enum { GC_STAGE_RESET = 1, GC_STAGE_INDEX = 2, GC_STAGE_DECODE = 4, GC_STAGE_ALL = 7 };
gc_status gc_decode_stage(const gc_batch* b, uint32_t* out, void* ws, uint64_t ws_bytes,
                          void* stream, int dgaps, int stage_mask);

/* ---------------------------------------------------------------------------
 * Skip pointers and random access (§7.5: "skip list pointers for posting blocks.
 * The skip distance ... 512 postings").
 *
 * One entry per block of GC_SKIP_DIST ints of every list -- block b of list l covers the
 * list's ints [512b, 512b+512) -- saying where decoding of the block starts with nothing
 * before it.  Every group of a list is OWNED by one 32-bit control word: the word holding
 * its descriptor (Group-Simple selector, binary LD field, AFOR / PFD frame header) or, for
 * a unary code, its terminating 0.  An entry names the word owning the group of the
 * block's first quad (quad 128b, word index relative to the list's ctrl_off / 4) and the
 * list's prefixes before that word: raw quads of the groups owned by earlier words, data
 * lane-bits (complete unary: CG x 32 x word, its closed form), exception bytes
 * (Group-PFD), and docid = the block's d-gap carry, the list's ints [0, 512b) summed
 * mod 2^32 (0 for block 0).  skip_off[l] = sum over lists l' < l of ceil(n_l' / 512) is
 * list l's first entry; skip_off[n_lists] the entry count.  The layout is byte-identical
 * to the oracle's gco_skip_entry (the tests compare the two tables). */
#define GC_SKIP_DIST 512
typedef struct {
  uint64_t data_bits;
  uint32_t word, quads, exc_bytes, docid, pad[2];
} gc_skip_entry; /* 32 bytes */

/* An upper bound of the entry count, total_out / 512 + n_lists (host only, no launch). */
gc_status gc_skip_capacity(const gc_batch* b, uint64_t* entries);

/* Build the skip table of a batch (index-building time, not the query path):
 *   docids   DEVICE, total_out u32: the batch's gc_decode_dgaps output (the carries);
 *   skip_off DEVICE, n_lists + 1 u64 (written);  entries DEVICE, room for
 *   gc_skip_capacity entries (written);  ws: a decode workspace (>= gc_workspace_size bytes).
 * Runs the control-stream scan (subsystem (a)), which knows every control word's list
 * prefixes, and writes an entry wherever a word owns a block's first quad.  Not for
 * GC_VARBYTE (GC_ERR_UNKNOWN_CODEC).  Asynchronous on `stream`. */
gc_status gc_build_skip(const gc_batch* b, const uint32_t* docids, uint64_t* skip_off,
                        gc_skip_entry* entries, void* ws, uint64_t ws_bytes, void* stream);

/* Random access: decode the output ints [first, first + count) from the skip table alone
 * -- no full decode, no index stage, no look-back: every 512-int block overlapping the
 * range is decoded on its own from its entry (one warp per block: the block's control
 * words parsed from the entry's word, its quads unpacked, the d-gap scan started from the
 * entry's docid when dgaps != 0).  Exactly out[first .. first+count) is written (`out` is
 * the batch-sized output).  ws: >= 64 bytes of DEVICE memory for the sticky GC_DEV_* bits
 * (reset inside the call; gc_read_device_status reads them).  Not for GC_VARBYTE.
 * Asynchronous on `stream`. */
gc_status gc_decode_range(const gc_batch* b, const uint64_t* skip_off,
                          const gc_skip_entry* entries, uint32_t* out, uint64_t first,
                          uint64_t count, int dgaps, void* ws, uint64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Posting store (§7.5: "we use VByte to compress posting lists with less than 64
 * postings"; §7.4: query processing decodes d-gaps and TFs).  A store keeps the
 * long lists (>= threshold ints) in a Group-codec batch and the short ones in a Variable
 * Byte batch, and optionally each list's term frequencies beside its docIDs, split and
 * encoded the same way with no d-gap.  Decoded, the long group's ints come first and the
 * short group's from short_base (a multiple of 4); list_out_off[l] locates list l.
 *
 * gc_posting_split (host, no launch): for list_n[n_lists] and the threshold, the lists of
 * each group in order (long_ids[*n_long], short_ids[*n_short]; caller arrays of n_lists),
 * list_out_off[n_lists] and *short_base.
 * gc_posting_gather (host, no launch): the values of lists ids[n_ids], concatenated in
 * that order into out (and their lengths into out_list_n), for the encoder.
 * ------------------------------------------------------------------------- */
gc_status gc_posting_split(const uint32_t* list_n, uint64_t n_lists, uint32_t threshold,
                           uint64_t* long_ids, uint64_t* n_long, uint64_t* short_ids,
                           uint64_t* n_short, uint64_t* list_out_off, uint64_t* short_base);
gc_status gc_posting_gather(const uint32_t* values, const uint32_t* list_n, uint64_t n_lists,
                            const uint64_t* ids, uint64_t n_ids, uint32_t* out,
                            uint32_t* out_list_n);

/* A store on the device: the two groups of docIDs, and (or NULL) of TFs.  long_tfs must
 * have the long docIDs' codec, variant and total_out (the same lists). */
typedef struct {
  gc_batch long_docs, short_docs;
  const gc_batch* long_tfs;
  const gc_batch* short_tfs;
  uint64_t short_base;
} gc_posting_store;

/* Workspace bytes for gc_decode_posting_store (host only). */
gc_status gc_posting_store_ws_size(const gc_posting_store* s, uint64_t* bytes);

/* Decode a whole store: docs[short_base + total of the short group] receives the docIDs
 * (dgaps != 0) or gaps, tfs (if the store has TFs) the raw TFs, both in the store's output
 * layout.  The long group's docIDs and TFs are decoded in ONE fused k_decode pass over
 * both batches (their tiles interleaved: the TF tiles' unpack fills the docID tiles'
 * look-back latency); the short groups by the Variable Byte kernels.  Sticky device status
 * bits: gc_posting_store_status.  Asynchronous on `stream`. */
gc_status gc_decode_posting_store(const gc_posting_store* s, uint32_t* docs, uint32_t* tfs,
                                  int dgaps, void* ws, uint64_t ws_bytes, void* stream);
gc_status gc_posting_store_status(const gc_posting_store* s, const void* ws, uint32_t* host_bits,
                                  void* stream);

/* Copy the sticky GC_DEV_* bits of a workspace to *host_bits.  Synchronises
 * `stream`.  0 means the last decode on this workspace saw a well-formed batch. */
gc_status gc_read_device_status(const void* ws, uint32_t* host_bits, void* stream);

/* Shard-additive checksum of a decoded batch (verification, never timed):
 * dev_sum3[0] = sum_l sum_i mix64(((l+list_base) << 32 | i) ^ (out_i * 0x9E3779B97F4A7C15)),
 * dev_sum3[1] = sum of out_i, dev_sum3[2] = sum of list_n, all mod 2^64
 * (mix64 = the splitmix64 finaliser).  dev_sum3 is DEVICE
 * memory (3 x u64), overwritten.  list_base is the global id of list 0. */
gc_status gc_checksum(const gc_batch* b, const uint32_t* out, uint64_t list_base,
                      uint64_t* dev_sum3, void* stream);

/* End-to-end decode from HOST buffers: copies the directory and streams of
 * `host_batch` (host pointers; pinned memory recommended) into `dev_scratch`,
 * decodes (dgaps != 0: docIDs) and copies the result into host_out (total_out
 * u32).  dev_scratch: DEVICE memory of >= gc_host_scratch_size bytes, 256-B
 * aligned.  Asynchronous on `stream` (synchronise before reading host_out). */
gc_status gc_host_scratch_size(const gc_batch* host_batch, uint64_t* bytes);
gc_status gc_decode_host(const gc_batch* host_batch, uint32_t* host_out, int dgaps,
                         void* dev_scratch, uint64_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Host encoder (multi-threaded C++; the bytes are identical to oracle/'s).
 *   values[sum(list_n)]  HOST, concatenated lists; docIDs when delta != 0
 *                        (each list strictly increasing; the encoder applies
 *                        the d-gap of P:L57), else the integers to store.
 *   zeta_num/zeta_den    Group-PFD exception threshold, default 1/10
 *                        (variant 1, SIMD-BP128: ignored, no exceptions).
 * gc_encode_begin encodes into encoder-owned host memory and fills the HOST
 * directory arrays ctrl_off/data_off/exc_off/out_off [n_lists+1] and
 * sizes[3] = {ctrl_bytes, data_vectors, exc_bytes} (ctrl/exc padded to 16 B).
 * gc_encode_finish copies the streams into caller HOST buffers of those sizes
 * and releases the handle (gc_encode_abort releases without copying).
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t codec;
  uint32_t variant;
  uint32_t pfd_frame_quads;
  uint32_t zeta_num;
  uint32_t zeta_den;
} gc_encode_params;

gc_status gc_encode_begin(const gc_encode_params* p, const uint32_t* values,
                          const uint32_t* list_n, uint64_t n_lists, int delta, int threads,
                          uint64_t* ctrl_off, uint64_t* data_off, uint64_t* exc_off,
                          uint64_t* out_off, uint64_t* sizes, void** handle);
gc_status gc_encode_finish(void* handle, uint8_t* ctrl, void* data, uint8_t* exc);
void gc_encode_abort(void* handle);

/* ---------------------------------------------------------------------------
 * GPU encoders: Variable Byte (P §2.3), Group-Simple (Algorithm
 * 1), Group-Scheme, all 10 variants, Group-AFOR,
 * Group-PFD (variant 0) and SIMD-BP128 (PFD variant 1); bytes
 * identical to the host encoder's and the oracle's (every codec and variant the decoder
 * takes; an invalid variant: GC_ERR_BAD_VARIANT).  sizes[3] is an internal count (frames, quads or blocks): pass
 * sizes back to gc_encode_device_write unchanged.  All arrays are DEVICE memory except
 * sizes[] and the params struct.
 *   values[total_ints], list_n[n_lists]  as for gc_encode_begin (docIDs if delta)
 *   ws, ws_bytes         workspace of at least gc_encode_device_ws_size bytes,
 *                        256-B aligned, owned by the caller; shared by the two calls
 * gc_encode_device_plan fills the DEVICE directory ctrl_off/data_off/exc_off/out_off
 * [n_lists+1] and, synchronising the stream, the HOST sizes[4] = {ctrl_bytes,
 * data_vectors, exc_bytes (16-B padded), frames}.  The caller then allocates ctrl
 * (4-B aligned), data (16-B aligned) and exc of those sizes, and
 * gc_encode_device_write fills them (asynchronously, same values/ws/sizes).
 * ------------------------------------------------------------------------- */
gc_status gc_encode_device_ws_size(const gc_encode_params* p, uint64_t n_lists, uint64_t total_ints,
                                   uint64_t* bytes);
gc_status gc_encode_device_plan(const gc_encode_params* p, const uint32_t* values,
                                const uint32_t* list_n, uint64_t n_lists, uint64_t total_ints,
                                int delta, uint64_t* ctrl_off, uint64_t* data_off,
                                uint64_t* exc_off, uint64_t* out_off, void* ws, uint64_t ws_bytes,
                                uint64_t* sizes, void* stream);
gc_status gc_encode_device_write(const gc_encode_params* p, const uint32_t* values,
                                 const uint32_t* list_n, uint64_t n_lists, uint64_t total_ints,
                                 int delta, const uint64_t* out_off, const uint64_t* sizes,
                                 uint8_t* ctrl, void* data, uint8_t* exc, void* ws,
                                 uint64_t ws_bytes, void* stream);

const char* gc_status_string(gc_status s);
int gc_abi_version(void);

/* How this library was built (host only, no launch): GC_BUILD_CHECKED when every shared-
 * and global-memory index of the decode kernels is asserted at run time (-DGC_CHECKED, a
 * debugging build: a failed check prints the kernel line and traps), GC_BUILD_TIMING when
 * the decode phases are timed into the workspace header (-DGC_TIMING).  Product builds: 0. */
enum { GC_BUILD_CHECKED = 1, GC_BUILD_TIMING = 2 };
int gc_build_flags(void);

#ifdef __cplusplus
}
#endif
#endif /* GC_H */
