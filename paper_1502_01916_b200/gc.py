"""Thin Python binding of include/gc.h (argument marshalling only).

Every step of decoding runs in libgc.so's sm_100a kernels; this module only turns
numpy arrays / torch tensors into the C structs.  There is no fallback: if libgc.so
is missing or no sm_100 device is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GC_LIB") or os.path.join(_PKG, "libgc.so")

VARBYTE, GROUP_SIMPLE, GROUP_SCHEME, GROUP_AFOR, GROUP_PFD = 1, 2, 3, 4, 5
CODEC_NAMES = {GROUP_SIMPLE: "group_simple", GROUP_SCHEME: "group_scheme",
               GROUP_AFOR: "group_afor", GROUP_PFD: "group_pfd"}
DEV_BITS = {1: "BAD_SELECTOR", 2: "BAD_LD", 4: "BAD_FRAME", 8: "BAD_EXCEPTION", 16: "TRUNCATED"}


class GcError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = _lib().gc_status_string(status).decode() if _LIB is not None else str(status)
        super().__init__(f"{what}: {msg} ({status})")


class CBatch(C.Structure):
    _fields_ = [("codec", C.c_int32), ("variant", C.c_uint32), ("pfd_frame_quads", C.c_uint32),
                ("reserved", C.c_uint32), ("n_lists", C.c_uint64),
                ("list_n", C.c_void_p), ("ctrl_off", C.c_void_p), ("data_off", C.c_void_p),
                ("exc_off", C.c_void_p), ("out_off", C.c_void_p),
                ("ctrl", C.c_void_p), ("ctrl_bytes", C.c_uint64),
                ("data", C.c_void_p), ("data_vectors", C.c_uint64),
                ("exc", C.c_void_p), ("exc_bytes", C.c_uint64), ("total_out", C.c_uint64)]


class CEncodeParams(C.Structure):
    _fields_ = [("codec", C.c_int32), ("variant", C.c_uint32), ("pfd_frame_quads", C.c_uint32),
                ("zeta_num", C.c_uint32), ("zeta_den", C.c_uint32)]


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
        sigs = {
            "gc_workspace_size": (i32, [P(CBatch), P(u64)]),
            "gc_decode": (i32, [P(CBatch), vp, vp, u64, vp]),
            "gc_decode_dgaps": (i32, [P(CBatch), vp, vp, u64, vp]),
            "gc_decode_stage": (i32, [P(CBatch), vp, vp, u64, vp, i32, i32]),
            "gc_decode_range": (i32, [P(CBatch), vp, vp, vp, u64, u64, i32, vp, u64, vp]),
            "gc_skip_capacity": (i32, [P(CBatch), P(u64)]),
            "gc_posting_split": (i32, [vp, u64, C.c_uint32, vp, P(u64), vp, P(u64), vp, P(u64)]),
            "gc_posting_gather": (i32, [vp, vp, u64, vp, u64, vp, vp]),
            "gc_posting_store_ws_size": (i32, [P(CPostingStore), P(u64)]),
            "gc_decode_posting_store": (i32, [P(CPostingStore), vp, vp, i32, vp, u64, vp]),
            "gc_posting_store_status": (i32, [P(CPostingStore), vp, P(C.c_uint32), vp]),
            "gc_build_skip": (i32, [P(CBatch), vp, vp, vp, vp, u64, vp]),
            "gc_read_device_status": (i32, [vp, P(C.c_uint32), vp]),
            "gc_checksum": (i32, [P(CBatch), vp, u64, vp, vp]),
            "gc_host_scratch_size": (i32, [P(CBatch), P(u64)]),
            "gc_decode_host": (i32, [P(CBatch), vp, i32, vp, u64, vp]),
            "gc_encode_begin": (i32, [P(CEncodeParams), vp, vp, u64, i32, i32, vp, vp, vp, vp, vp,
                                      P(vp)]),
            "gc_encode_finish": (i32, [vp, vp, vp, vp]),
            "gc_encode_abort": (None, [vp]),
            "gc_encode_device_ws_size": (i32, [P(CEncodeParams), u64, u64, P(u64)]),
            "gc_encode_device_plan": (i32, [P(CEncodeParams), vp, vp, u64, u64, i32, vp, vp, vp,
                                            vp, vp, u64, vp, vp]),
            "gc_encode_device_write": (i32, [P(CEncodeParams), vp, vp, u64, u64, i32, vp, vp, vp,
                                             vp, vp, vp, u64, vp]),
            "gc_status_string": (C.c_char_p, [i32]),
            "gc_abi_version": (i32, []),
            "gc_build_flags": (i32, []),
        }
        for name, (res, args) in sigs.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _LIB = lib
    return _LIB


def abi_version() -> int:
    return int(_lib().gc_abi_version())


def build_flags() -> int:
    """1: a checked build (bounds assertions in the kernels), 2: a timing build; 0: product."""
    return int(_lib().gc_build_flags())


def gsc_variant(cg: int, kind: str) -> int:
    """Group-Scheme variant: bits 0-1 log2 CG, bits 2-3 LD kind (B/CU/IU)."""
    return {1: 0, 2: 1, 4: 2, 8: 3}[cg] | ({"B": 0, "CU": 1, "IU": 2}[kind] << 2)


GSC_VARIANTS = [(cg, k) for cg in (1, 2, 4, 8) for k in ("B", "CU")] + [(4, "IU"), (8, "IU")]


def codec_label(codec: int, variant: int = 0, frame_quads: int = 32) -> str:
    if codec == GROUP_SCHEME:
        return f"GSC-{1 << (variant & 3)}-{('B', 'CU', 'IU')[variant >> 2]}"
    if codec == GROUP_PFD:
        name = "BP128" if variant == 1 else "G-PFD"
        return name if frame_quads == 32 else f"{name}-F{frame_quads}"
    return {VARBYTE: "VByte", GROUP_SIMPLE: "G-SIM", GROUP_AFOR: "G-AFOR"}[codec]


# ----------------------------------------------------------------------------- batches
@dataclasses.dataclass
class HostBatch:
    """A packed batch in host (numpy) memory.  Layout: include/gc.h / DESIGN.md §3.7."""
    codec: int
    variant: int
    frame_quads: int
    list_n: np.ndarray      # uint32 [L]
    ctrl_off: np.ndarray    # uint64 [L+1]
    data_off: np.ndarray    # uint64 [L+1]
    exc_off: np.ndarray     # uint64 [L+1]
    out_off: np.ndarray     # uint64 [L+1]
    ctrl: np.ndarray        # uint8, len % 16 == 0
    data: np.ndarray        # uint32 [V, 4]
    exc: np.ndarray         # uint8, len % 16 == 0

    @property
    def n_lists(self) -> int:
        return len(self.list_n)

    @property
    def total_out(self) -> int:
        return int(self.out_off[-1]) if len(self.out_off) else 0

    @property
    def compressed_bytes(self) -> int:
        """Stream bytes (ctrl + data + exc, logical extents) -- the algorithmic input bytes."""
        L = self.n_lists
        return int(self.ctrl_off[L]) + 16 * int(self.data_off[L]) + int(self.exc_off[L])

    @property
    def directory_bytes(self) -> int:
        return 4 * self.n_lists + 4 * 8 * (self.n_lists + 1)

    @staticmethod
    def from_dict(d: dict) -> "HostBatch":
        ctrl = np.ascontiguousarray(d["ctrl"], np.uint8)
        exc = np.ascontiguousarray(d["exc"], np.uint8)
        ctrl = np.concatenate([ctrl, np.zeros((-len(ctrl)) % 16, np.uint8)])
        exc = np.concatenate([exc, np.zeros((-len(exc)) % 16, np.uint8)])
        return HostBatch(int(d["codec"]), int(d.get("variant", 0)), int(d.get("frame_quads", 32)),
                         np.ascontiguousarray(d["list_n"], np.uint32),
                         np.ascontiguousarray(d["ctrl_off"], np.uint64),
                         np.ascontiguousarray(d["data_off"], np.uint64),
                         np.ascontiguousarray(d["exc_off"], np.uint64),
                         np.ascontiguousarray(d["out_off"], np.uint64),
                         ctrl, np.ascontiguousarray(d["data"], np.uint32).reshape(-1, 4), exc)

    def as_dict(self) -> dict:
        return dict(codec=self.codec, variant=self.variant, frame_quads=self.frame_quads,
                    list_n=self.list_n, ctrl_off=self.ctrl_off, data_off=self.data_off,
                    exc_off=self.exc_off, out_off=self.out_off, ctrl=self.ctrl, data=self.data,
                    exc=self.exc, total_out=self.total_out)

    def cstruct(self) -> CBatch:
        """Host-pointer gc_batch (for gc_decode_host).  Keep `self` alive while used."""
        def p(a):
            return a.ctypes.data if a.size else None
        return CBatch(self.codec, self.variant, self.frame_quads, 0, self.n_lists,
                      p(self.list_n), p(self.ctrl_off), p(self.data_off), p(self.exc_off),
                      p(self.out_off), p(self.ctrl), len(self.ctrl), p(self.data),
                      len(self.data), p(self.exc), len(self.exc), self.total_out)


@dataclasses.dataclass
class DeviceBatch:
    """The same batch resident in device memory (torch tensors used as raw buffers)."""
    codec: int
    variant: int
    frame_quads: int
    n_lists: int
    total_out: int
    tensors: dict           # name -> torch tensor
    ctrl_bytes: int
    data_vectors: int
    exc_bytes: int

    @property
    def compressed_bytes(self) -> int:
        """Stream bytes (ctrl + data + exc, logical extents; reads the offsets' last entries)."""
        L = self.n_lists
        t = self.tensors
        return (int(t["ctrl_off"][L].item()) + 16 * int(t["data_off"][L].item())
                + int(t["exc_off"][L].item()))

    @property
    def directory_bytes(self) -> int:
        return 4 * self.n_lists + 4 * 8 * (self.n_lists + 1)

    def cstruct(self) -> CBatch:
        t = self.tensors

        def p(name):
            x = t[name]
            return x.data_ptr() if x.numel() else None
        return CBatch(self.codec, self.variant, self.frame_quads, 0, self.n_lists,
                      p("list_n"), p("ctrl_off"), p("data_off"), p("exc_off"), p("out_off"),
                      p("ctrl"), self.ctrl_bytes, p("data"), self.data_vectors, p("exc"),
                      self.exc_bytes, self.total_out)


def encode_batch(values: np.ndarray, list_n: np.ndarray, codec: int, variant: int = 0,
                 delta: bool = False, frame_quads: int = 32, zeta=(1, 10),
                 threads: int = 0) -> HostBatch:
    """Host encoder of libgc.so (gc_encode_begin/finish)."""
    v = np.ascontiguousarray(values, np.uint32)
    ln = np.ascontiguousarray(list_n, np.uint32)
    L = len(ln)
    offs = [np.zeros(L + 1, np.uint64) for _ in range(4)]
    sizes = np.zeros(3, np.uint64)
    prm = CEncodeParams(codec, variant, frame_quads, zeta[0], zeta[1])
    h = C.c_void_p()
    st = _lib().gc_encode_begin(C.byref(prm), v.ctypes.data if v.size else None,
                                ln.ctypes.data if L else None, L, int(delta), threads,
                                offs[0].ctypes.data, offs[1].ctypes.data, offs[2].ctypes.data,
                                offs[3].ctypes.data, sizes.ctypes.data, C.byref(h))
    if st:
        raise GcError(st, "gc_encode_begin")
    ctrl = np.zeros(int(sizes[0]), np.uint8)
    data = np.zeros((int(sizes[1]), 4), np.uint32)
    exc = np.zeros(int(sizes[2]), np.uint8)
    st = _lib().gc_encode_finish(h, ctrl.ctypes.data if ctrl.size else None,
                                 data.ctypes.data if data.size else None,
                                 exc.ctypes.data if exc.size else None)
    if st:
        raise GcError(st, "gc_encode_finish")
    return HostBatch(codec, variant, frame_quads, ln.copy(), offs[0], offs[1], offs[2], offs[3],
                     ctrl, data, exc)


def encode_device(values, list_n, codec: int = GROUP_PFD, variant: int = 0, delta: bool = False,
                  frame_quads: int = 32, zeta=(1, 10), stream=None, ws=None) -> DeviceBatch:
    """GPU encoder of the frame codecs (gc_encode_device_plan/write): Group-PFD (variant 0)
    and SIMD-BP128 (variant 1).  values, list_n: int32/uint32 CUDA tensors.  Returns the
    batch resident on the device, ready for decode()."""
    import torch
    dev = values.device
    L, N = int(list_n.numel()), int(values.numel())
    prm = CEncodeParams(codec, variant, frame_quads, zeta[0], zeta[1])
    need = C.c_uint64()
    st = _lib().gc_encode_device_ws_size(C.byref(prm), L, N, C.byref(need))
    if st:
        raise GcError(st, "gc_encode_device_ws_size")
    if ws is None or ws.numel() < need.value:
        ws = torch.empty(max(int(need.value), 256), dtype=torch.uint8, device=dev)
    offs = [torch.zeros(L + 1, dtype=torch.int64, device=dev) for _ in range(4)]
    sizes = np.zeros(4, np.uint64)
    sp = _stream_ptr(stream)
    vp = values.data_ptr() if N else None
    lp = list_n.data_ptr() if L else None
    st = _lib().gc_encode_device_plan(C.byref(prm), vp, lp, L, N, int(delta), *[o.data_ptr() for o in offs],
                                      ws.data_ptr(), ws.numel(), sizes.ctypes.data, sp)
    if st:
        raise GcError(st, "gc_encode_device_plan")
    ctrl = torch.empty(max(int(sizes[0]), 16), dtype=torch.uint8, device=dev)
    data = torch.empty(max(int(sizes[1]), 1) * 4, dtype=torch.int32, device=dev)
    exc = torch.empty(max(int(sizes[2]), 16), dtype=torch.uint8, device=dev)
    st = _lib().gc_encode_device_write(C.byref(prm), vp, lp, L, N, int(delta), offs[3].data_ptr(),
                                       sizes.ctypes.data, ctrl.data_ptr(), data.data_ptr(),
                                       exc.data_ptr(), ws.data_ptr(), ws.numel(), sp)
    if st:
        raise GcError(st, "gc_encode_device_write")
    tensors = dict(list_n=list_n.view(torch.int32), ctrl_off=offs[0], data_off=offs[1],
                   exc_off=offs[2], out_off=offs[3], ctrl=ctrl[:int(sizes[0])],
                   data=data[:4 * int(sizes[1])], exc=exc[:int(sizes[2])])
    return DeviceBatch(codec, variant, frame_quads, L, N, tensors, int(sizes[0]), int(sizes[1]),
                       int(sizes[2]))


# ----------------------------------------------------------------------------- posting store
@dataclasses.dataclass
class PostingStore:
    """P:L640 §7.5's rule: lists shorter than `threshold` (64) are Variable Byte encoded
    whatever the codec of the others.  The lists keep their order within
    each group; the decoded output holds the long group first and the short group from the
    16-byte aligned offset `short_base`; `list_out_off[i]` locates original list i in it."""
    long: HostBatch
    short: HostBatch
    list_out_off: np.ndarray   # uint64 [L]
    short_base: int
    total: int                 # ints of the decoded output (incl. the alignment gap)
    tf_long: "HostBatch | None" = None    # term frequencies (raw, no d-gap), same split
    tf_short: "HostBatch | None" = None


def encode_posting_store(values: np.ndarray, list_n: np.ndarray, codec: int, variant: int = 0,
                         delta: bool = False, threshold: int = 64, tfs: "np.ndarray | None" = None,
                         **kw) -> PostingStore:
    """`tfs` (optional, one per posting): the lists' term frequencies, stored beside the
    docIDs with the same split and codecs but no d-gap (TFs are not sorted).  The
    split and gather are gc_posting_split / gc_posting_gather; each group is encoded by the
    host encoder."""
    v = np.ascontiguousarray(values, np.uint32)
    ln = np.ascontiguousarray(list_n, np.uint32)
    L = len(ln)
    ids = {True: np.zeros(max(L, 1), np.uint64), False: np.zeros(max(L, 1), np.uint64)}
    n_long, n_short, base = C.c_uint64(), C.c_uint64(), C.c_uint64()
    off = np.zeros(max(L, 1), np.uint64)
    st = _lib().gc_posting_split(ln.ctypes.data if L else None, L, threshold,
                                 ids[False].ctypes.data, C.byref(n_long), ids[True].ctypes.data,
                                 C.byref(n_short), off.ctypes.data, C.byref(base))
    if st:
        raise GcError(st, "gc_posting_split")
    groups = {False: ids[False][:n_long.value], True: ids[True][:n_short.value]}

    def gather(src, short):
        g = groups[short]
        n = int(ln[g.astype(np.int64)].sum()) if len(g) else 0
        out = np.zeros(max(n, 1), np.uint32)
        gl = np.zeros(max(len(g), 1), np.uint32)
        r = _lib().gc_posting_gather(src.ctypes.data if src.size else None, ln.ctypes.data if L else None,
                                     L, g.ctypes.data if len(g) else None, len(g), out.ctypes.data,
                                     gl.ctypes.data)
        if r:
            raise GcError(r, "gc_posting_gather")
        return out[:n], gl[:len(g)]
    longb = encode_batch(*gather(v, False), codec, variant, delta=delta, **kw)
    shortb = encode_batch(*gather(v, True), VARBYTE, 0, delta=delta)
    short_base = int(base.value)
    st_ = PostingStore(longb, shortb, off[:L], short_base, short_base + shortb.total_out)
    if tfs is not None:
        t = np.ascontiguousarray(tfs, np.uint32)
        assert t.size == v.size, "one TF per posting"
        st_.tf_long = encode_batch(*gather(t, False), codec, variant, **kw)
        st_.tf_short = encode_batch(*gather(t, True), VARBYTE, 0)
    return st_


class CPostingStore(C.Structure):
    _fields_ = [("long_docs", CBatch), ("short_docs", CBatch), ("long_tfs", C.POINTER(CBatch)),
                ("short_tfs", C.POINTER(CBatch)), ("short_base", C.c_uint64)]


class StoreStatus(tuple):
    """(ws of the docIDs, ws of the TFs) views of the one workspace; keeps the device
    batches alive for as long as the caller holds it."""


def decode_posting_store(store: PostingStore, dgaps: bool = True, device="cuda", stream=None):
    """gc_decode_posting_store: the long group's docIDs (and TFs: one fused k_decode pass
    over both batches) and the short group's (Variable Byte) into one output (int32 view of
    uint32).  Returns (docs, workspaces) or, with TFs in the store, (docs, tfs, workspaces);
    gc.read_device_status(w) == 0 for both workspaces means a clean decode."""
    import contextlib
    import torch
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:  # (everything allocated on the decoding stream: no early reuse of its memory)
        has_tf = store.tf_long is not None
        dbs = [to_device(b, device) for b in
               ((store.long, store.short, store.tf_long, store.tf_short) if has_tf
                else (store.long, store.short))]
        cs = [d.cstruct() for d in dbs]
        cst = CPostingStore(cs[0], cs[1], C.pointer(cs[2]) if has_tf else None,
                            C.pointer(cs[3]) if has_tf else None, store.short_base)
        need = C.c_uint64()
        _lib().gc_posting_store_ws_size(C.byref(cst), C.byref(need))
        ws = torch.empty(max(int(need.value), 256), dtype=torch.uint8, device=device)
        docs = torch.empty(max(store.total, 4), dtype=torch.int32, device=device)
        tfs = torch.empty(max(store.total, 4), dtype=torch.int32, device=device) if has_tf else None
        st = _lib().gc_decode_posting_store(C.byref(cst), docs.data_ptr(),
                                            tfs.data_ptr() if has_tf else None, int(dgaps),
                                            ws.data_ptr(), ws.numel(), _stream_ptr(stream))
        if st:
            raise GcError(st, "gc_decode_posting_store")
    off = (workspace_size(dbs[0]) + 255) & ~255
    w = StoreStatus((ws[:off], ws[off:]))
    w.batches = dbs
    if has_tf:
        return docs[:store.total], tfs[:store.total], w
    return docs[:store.total], w


def to_device(hb: HostBatch, device="cuda", pin: bool = False) -> DeviceBatch:
    import torch

    def t(a, dt):
        x = torch.from_numpy(np.ascontiguousarray(a).view(dt))
        return x.to(device, non_blocking=False)
    tensors = dict(
        list_n=t(hb.list_n, np.int32), ctrl_off=t(hb.ctrl_off, np.int64),
        data_off=t(hb.data_off, np.int64), exc_off=t(hb.exc_off, np.int64),
        out_off=t(hb.out_off, np.int64), ctrl=t(hb.ctrl, np.uint8),
        data=t(hb.data.reshape(-1), np.int32), exc=t(hb.exc, np.uint8))
    return DeviceBatch(hb.codec, hb.variant, hb.frame_quads, hb.n_lists, hb.total_out, tensors,
                       len(hb.ctrl), len(hb.data), len(hb.exc))


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def workspace_size(batch) -> int:
    b = batch.cstruct()
    n = C.c_uint64(0)
    st = _lib().gc_workspace_size(C.byref(b), C.byref(n))
    if st:
        raise GcError(st, "gc_workspace_size")
    return int(n.value)


def alloc_workspace(batch, device="cuda"):
    import torch
    return torch.empty(max(workspace_size(batch), 16), dtype=torch.uint8, device=device)


def _decode(fn_name: str, batch: DeviceBatch, out=None, ws=None, stream=None):
    import torch
    dev = batch.tensors["out_off"].device
    if out is None:
        out = torch.empty(max(batch.total_out, 4), dtype=torch.int32, device=dev)
    if ws is None:
        ws = alloc_workspace(batch, dev)
    b = batch.cstruct()
    st = getattr(_lib(), fn_name)(C.byref(b), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                  _stream_ptr(stream))
    if st:
        raise GcError(st, fn_name)
    return out[:batch.total_out], ws


def decode(batch: DeviceBatch, out=None, ws=None, stream=None):
    """gc_decode: the stored integers (d-gaps / TFs).  Returns (out int32 view, ws)."""
    return _decode("gc_decode", batch, out, ws, stream)


def decode_dgaps(batch: DeviceBatch, out=None, ws=None, stream=None):
    """gc_decode_dgaps: decode + per-list prefix sum mod 2^32 (docIDs)."""
    return _decode("gc_decode_dgaps", batch, out, ws, stream)


STAGE_RESET, STAGE_INDEX, STAGE_DECODE, STAGE_ALL = 1, 2, 4, 7


SKIP_DIST = 512
# gc_skip_entry (include/gc.h): data_bits u64, word, quads, exc_bytes, docid, pad[2] u32
SKIP_DTYPE = np.dtype([("data_bits", "<u8"), ("word", "<u4"), ("quads", "<u4"),
                       ("exc_bytes", "<u4"), ("docid", "<u4"), ("pad", "<u4", (2,))])


def build_skip(batch: DeviceBatch, docids, ws=None, stream=None):
    """gc_build_skip: the batch's skip pointers every 512 postings (§7.5) from its
    d-gap decode `docids` (device).  Returns (skip_off int64 [L+1], entries uint8 [cap, 32])
    device tensors; entries[:skip_off[L]] are valid."""
    import torch
    b = batch.cstruct()
    cap = C.c_uint64(0)
    _lib().gc_skip_capacity(C.byref(b), C.byref(cap))
    dev = batch.tensors["list_n"].device
    off = torch.empty(batch.n_lists + 1, dtype=torch.int64, device=dev)
    ent = torch.empty((max(int(cap.value), 1), 32), dtype=torch.uint8, device=dev)
    if ws is None:
        ws = alloc_workspace(batch, dev)
    st = _lib().gc_build_skip(C.byref(b), docids.data_ptr(), off.data_ptr(), ent.data_ptr(),
                              ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    if st:
        raise GcError(st, "gc_build_skip")
    return off, ent


def skip_entries_host(skip_off, entries) -> np.ndarray:
    """The valid entries of a device skip table as a SKIP_DTYPE array (for comparisons)."""
    n = int(skip_off[-1].item())
    return entries[:n].cpu().numpy().reshape(-1).view(SKIP_DTYPE)


def decode_range(batch: DeviceBatch, skip_off, entries, out, first: int, count: int,
                 dgaps: bool = True, ws=None, stream=None):
    """gc_decode_range: random access -- exactly out[first:first+count] decoded from the
    skip table alone (one warp per overlapping 512-int block).  Returns the status ws."""
    import torch
    b = batch.cstruct()
    if ws is None:
        ws = torch.empty(256, dtype=torch.uint8, device=out.device)
    st = _lib().gc_decode_range(C.byref(b), skip_off.data_ptr(), entries.data_ptr(),
                                out.data_ptr(), first, count, int(dgaps), ws.data_ptr(),
                                ws.numel(), _stream_ptr(stream))
    if st:
        raise GcError(st, "gc_decode_range")
    return ws


def decode_stage(batch: DeviceBatch, out, ws, dgaps: bool, stages: int, stream=None):
    """gc_decode_stage: run a subset of the reset / index / decode stages."""
    b = batch.cstruct()
    st = _lib().gc_decode_stage(C.byref(b), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                _stream_ptr(stream), int(dgaps), stages)
    if st:
        raise GcError(st, "gc_decode_stage")


def read_device_status(ws, stream=None) -> int:
    bits = C.c_uint32(0)
    st = _lib().gc_read_device_status(ws.data_ptr(), C.byref(bits), _stream_ptr(stream))
    if st:
        raise GcError(st, "gc_read_device_status")
    return int(bits.value)


def status_names(bits: int) -> list[str]:
    return [n for b, n in DEV_BITS.items() if bits & b]


def checksum(batch: DeviceBatch, out, list_base: int = 0, stream=None):
    import torch
    sums = torch.zeros(3, dtype=torch.int64, device=out.device)
    b = batch.cstruct()
    st = _lib().gc_checksum(C.byref(b), out.data_ptr(), list_base, sums.data_ptr(),
                            _stream_ptr(stream))
    if st:
        raise GcError(st, "gc_checksum")
    return sums


def host_scratch_size(hb: HostBatch) -> int:
    b = hb.cstruct()
    n = C.c_uint64(0)
    st = _lib().gc_host_scratch_size(C.byref(b), C.byref(n))
    if st:
        raise GcError(st, "gc_host_scratch_size")
    return int(n.value)


def decode_host(hb: HostBatch, host_out: np.ndarray, dgaps: bool, scratch, stream=None):
    """gc_decode_host: H2D copies + decode + D2H copy, all enqueued on `stream`."""
    b = hb.cstruct()
    st = _lib().gc_decode_host(C.byref(b), host_out.ctypes.data, int(dgaps), scratch.data_ptr(),
                               scratch.numel(), _stream_ptr(stream))
    if st:
        raise GcError(st, "gc_decode_host")
