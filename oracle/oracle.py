"""ctypes binding of the C oracle (oracle/gc_oracle.c).  TEST INFRASTRUCTURE ONLY.

Marshalling only: every step of encoding/decoding happens in gc_oracle.c, which
follows PAPER.md step by step (see the citations there).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gc_oracle.c")
HDR = os.path.join(HERE, "gc_oracle.h")
LIB = os.path.join(HERE, "liboracle.so")

VARBYTE, GROUP_SIMPLE, GROUP_SCHEME, GROUP_AFOR, GROUP_PFD = 1, 2, 3, 4, 5
ERRORS = {0: "ok", 1: "arg", 2: "malformed", 3: "truncated", 4: "bad_magic", 5: "version",
          6: "codec", 7: "variant", 8: "nomem", 9: "not_increasing"}


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str = ""):
        self.rc = rc
        self.kind = ERRORS.get(rc, str(rc))
        super().__init__(f"oracle error {self.kind} ({rc}) {what}")


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc -O2 (no intrinsics)."""
    stale = (not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC),
                                                                      os.path.getmtime(HDR)))
    if force or stale:
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-fPIC", "-shared", "-o", tmp,
                               SRC, "-lpthread"])
        os.replace(tmp, LIB)
    return LIB


class Params(C.Structure):
    _fields_ = [("codec", C.c_int32), ("variant", C.c_uint32), ("frame_quads", C.c_uint32),
                ("zeta_num", C.c_uint32), ("zeta_den", C.c_uint32)]


class Stream(C.Structure):
    _fields_ = [("ctrl", C.POINTER(C.c_uint8)), ("ctrl_bytes", C.c_uint64),
                ("data", C.POINTER(C.c_uint32)), ("nvec", C.c_uint64),
                ("exc", C.POINTER(C.c_uint8)), ("exc_bytes", C.c_uint64)]


class Batch(C.Structure):
    _fields_ = [("n_lists", C.c_uint64), ("list_n", C.POINTER(C.c_uint32)),
                ("ctrl_off", C.POINTER(C.c_uint64)), ("data_off", C.POINTER(C.c_uint64)),
                ("exc_off", C.POINTER(C.c_uint64)), ("out_off", C.POINTER(C.c_uint64)),
                ("ctrl", C.POINTER(C.c_uint8)), ("ctrl_bytes", C.c_uint64),
                ("data", C.POINTER(C.c_uint32)), ("data_vectors", C.c_uint64),
                ("exc", C.POINTER(C.c_uint8)), ("exc_bytes", C.c_uint64),
                ("total_out", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        sig = {
            "gco_width": (C.c_uint32, [C.c_uint32]),
            "gco_quad_max": (C.c_uint32, [P(C.c_uint32)]),
            "gco_quad_or": (C.c_uint32, [P(C.c_uint32)]),
            "gco_gs_select": (C.c_uint64, [P(C.c_uint32), C.c_uint64, P(C.c_uint8)]),
            "gco_gsc_ld": (C.c_uint32, [C.c_uint32, C.c_uint32]),
            "gco_gsc_bw": (C.c_uint32, [C.c_uint32, C.c_uint32]),
            "gco_afor_partition": (C.c_uint64, [P(C.c_uint32), C.c_uint64, P(C.c_uint8),
                                                P(C.c_uint8), P(C.c_uint64)]),
            "gco_pfd_choose_b": (C.c_uint32, [P(C.c_uint32), C.c_uint32, C.c_uint32, C.c_uint32]),
            "gco_pack_vertical": (C.c_int, [P(C.c_uint32), C.c_uint64, C.c_uint32, P(C.c_uint32),
                                            C.c_uint64]),
            "gco_unpack_vertical": (C.c_int, [P(C.c_uint32), C.c_uint64, C.c_uint32, C.c_uint64,
                                              P(C.c_uint32)]),
            "gco_encode_list": (C.c_int, [P(Params), P(C.c_uint32), C.c_uint32, P(Stream)]),
            "gco_decode_list": (C.c_int, [P(Params), C.c_uint32, P(C.c_uint8), C.c_uint64,
                                          P(C.c_uint32), C.c_uint64, P(C.c_uint8), C.c_uint64,
                                          P(C.c_uint32)]),
            "gco_stream_free": (None, [P(Stream)]),
            "gco_encode_block": (C.c_int, [P(Params), C.c_int, P(C.c_uint32), C.c_uint32,
                                           P(P(C.c_uint8)), P(C.c_uint64)]),
            "gco_decode_block": (C.c_int, [P(C.c_uint8), C.c_uint64, C.c_uint32, P(C.c_uint32),
                                           C.c_uint32, P(C.c_uint32)]),
            "gco_free": (None, [C.c_void_p]),
            "gco_encode_batch": (C.c_int, [P(Params), P(C.c_uint32), P(C.c_uint32), C.c_uint64,
                                           C.c_int, C.c_int, P(Batch)]),
            "gco_decode_batch": (C.c_int, [P(Params), P(Batch), C.c_int, C.c_int, P(C.c_uint32),
                                           P(C.c_uint64)]),
            "gco_batch_free": (None, [P(Batch)]),
            "gco_skip_entries": (C.c_uint64, [P(Batch)]),
            "gco_build_skip": (C.c_int, [P(Params), P(Batch), P(C.c_uint64), C.c_void_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u8p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def params(codec: int, variant: int = 0, frame_quads: int = 32, zeta=(1, 10)) -> Params:
    return Params(codec, variant, frame_quads, zeta[0], zeta[1])


def gsc_variant(cg: int, kind: str) -> int:
    """Group-Scheme variant byte: bits0-1 log2 CG, bits2-3 LD kind."""
    k = {"B": 0, "CU": 1, "IU": 2}[kind]
    return {1: 0, 2: 1, 4: 2, 8: 3}[cg] | (k << 2)


# ---------------------------------------------------------------- primitives
def width(x: int) -> int:
    return int(lib().gco_width(x))


def quad_max(q) -> int:
    a = np.ascontiguousarray(q, dtype=np.uint32)
    return int(lib().gco_quad_max(_u32p(a)))


def quad_or(q) -> int:
    a = np.ascontiguousarray(q, dtype=np.uint32)
    return int(lib().gco_quad_or(_u32p(a)))


def gs_select(maxarr) -> list[int]:
    m = np.ascontiguousarray(maxarr, dtype=np.uint32)
    modes = np.zeros(max(len(m), 1), np.uint8)
    t = lib().gco_gs_select(_u32p(m), len(m), _u8p(modes))
    return [int(v) for v in modes[:t]]


def gsc_ld(quadmax: int, variant: int) -> int:
    return int(lib().gco_gsc_ld(quadmax, variant))


def gsc_bw(ld: int, variant: int) -> int:
    return int(lib().gco_gsc_bw(ld, variant))


def afor_partition(widths):
    w = np.ascontiguousarray(widths, dtype=np.uint32)
    assert len(w) % 8 == 0
    fl = np.zeros(len(w) // 8 + 1, np.uint8)
    fb = np.zeros(len(w) // 8 + 1, np.uint8)
    nf = C.c_uint64(0)
    cost = lib().gco_afor_partition(_u32p(w), len(w), _u8p(fl), _u8p(fb), C.byref(nf))
    return int(cost), [(int(fl[i]), int(fb[i])) for i in range(nf.value)]


def pfd_choose_b(frame_qmax, zeta=(1, 10)) -> int:
    m = np.ascontiguousarray(frame_qmax, dtype=np.uint32)
    return int(lib().gco_pfd_choose_b(_u32p(m), len(m), zeta[0], zeta[1]))


def pack_vertical(quads, bw: int) -> np.ndarray:
    q = np.ascontiguousarray(quads, dtype=np.uint32).reshape(-1, 4)
    nvec = -(-len(q) * bw // 32)
    out = np.zeros((max(nvec, 1), 4), np.uint32)
    rc = lib().gco_pack_vertical(_u32p(q), len(q), bw, _u32p(out), nvec)
    if rc:
        raise OracleError(rc)
    return out[:nvec]


def unpack_vertical(data, bw: int, Q: int) -> np.ndarray:
    d = np.ascontiguousarray(data, dtype=np.uint32).reshape(-1, 4)
    out = np.zeros((max(Q, 1), 4), np.uint32)
    rc = lib().gco_unpack_vertical(_u32p(d), len(d), bw, Q, _u32p(out))
    if rc:
        raise OracleError(rc)
    return out[:Q]


# ---------------------------------------------------------------- one list
def encode_list(x, codec: int, variant: int = 0, frame_quads: int = 32, zeta=(1, 10)):
    """Returns dict(ctrl=uint8[], data=uint32[nvec,4], exc=uint8[])."""
    a = np.ascontiguousarray(x, dtype=np.uint32)
    p = params(codec, variant, frame_quads, zeta)
    s = Stream()
    rc = lib().gco_encode_list(C.byref(p), _u32p(a), len(a), C.byref(s))
    if rc:
        lib().gco_stream_free(C.byref(s))
        raise OracleError(rc)
    out = dict(
        ctrl=np.ctypeslib.as_array(s.ctrl, (max(s.ctrl_bytes, 1),))[:s.ctrl_bytes].copy(),
        data=np.ctypeslib.as_array(s.data, (max(4 * s.nvec, 1),))[:4 * s.nvec].copy().reshape(-1, 4),
        exc=np.ctypeslib.as_array(s.exc, (max(s.exc_bytes, 1),))[:s.exc_bytes].copy(),
    )
    lib().gco_stream_free(C.byref(s))
    return out


def decode_list(n: int, ctrl, data, exc=None, codec: int = GROUP_SIMPLE, variant: int = 0,
                frame_quads: int = 32) -> np.ndarray:
    c = np.ascontiguousarray(ctrl, dtype=np.uint8)
    d = np.ascontiguousarray(data, dtype=np.uint32).reshape(-1)
    e = np.ascontiguousarray(exc if exc is not None else np.zeros(0, np.uint8), dtype=np.uint8)
    p = params(codec, variant, frame_quads)
    out = np.zeros(max(n, 1), np.uint32)
    cz = c if len(c) else np.zeros(1, np.uint8)
    dz = d if len(d) else np.zeros(4, np.uint32)
    ez = e if len(e) else np.zeros(1, np.uint8)
    rc = lib().gco_decode_list(C.byref(p), n, _u8p(cz), len(c), _u32p(dz), len(d) // 4,
                               _u8p(ez), len(e), _u32p(out))
    if rc:
        raise OracleError(rc)
    return out[:n]


def encode_block(x, codec: int, variant: int = 0, delta: bool = False, frame_quads: int = 32,
                 zeta=(1, 10)) -> bytes:
    a = np.ascontiguousarray(x, dtype=np.uint32)
    p = params(codec, variant, frame_quads, zeta)
    ptr = C.POINTER(C.c_uint8)()
    nb = C.c_uint64(0)
    rc = lib().gco_encode_block(C.byref(p), int(delta), _u32p(a), len(a), C.byref(ptr), C.byref(nb))
    if rc:
        raise OracleError(rc)
    b = bytes(np.ctypeslib.as_array(ptr, (nb.value,)))
    lib().gco_free(ptr)
    return b


def decode_block(block: bytes, frame_quads: int = 32, cap: int | None = None) -> np.ndarray:
    buf = np.frombuffer(block, np.uint8).copy() if len(block) else np.zeros(1, np.uint8)
    cap = cap if cap is not None else max(16, 8 * len(block) + 64)
    out = np.zeros(cap, np.uint32)
    n = C.c_uint32(0)
    rc = lib().gco_decode_block(_u8p(buf), len(block), frame_quads, _u32p(out), cap, C.byref(n))
    if rc:
        raise OracleError(rc)
    return out[:n.value]


# ---------------------------------------------------------------- batch
BATCH_KEYS = ("list_n", "ctrl_off", "data_off", "exc_off", "out_off", "ctrl", "data", "exc")


def encode_batch(values, list_n, codec: int, variant: int = 0, delta: bool = False,
                 frame_quads: int = 32, zeta=(1, 10), threads: int = 1) -> dict:
    """Encode + pack a batch of lists.  Returns numpy arrays."""
    v = np.ascontiguousarray(values, dtype=np.uint32)
    ln = np.ascontiguousarray(list_n, dtype=np.uint32)
    vz = v if len(v) else np.zeros(1, np.uint32)
    lz = ln if len(ln) else np.zeros(1, np.uint32)
    if codec == GROUP_PFD and variant == 1:
        # SIMD-BP128: each frame of 4F ints packed at "the minimum number of bits to
        # hold the largest integer" of the frame, no exceptions -- the b rule of P:L404 with
        # zeta = 0 (no quad may exceed b); same frame format, exception count 0
        zeta = (0, 1)
    p = params(codec, variant, frame_quads, zeta)
    b = Batch()
    rc = lib().gco_encode_batch(C.byref(p), _u32p(vz), _u32p(lz), len(ln), int(delta), threads,
                                C.byref(b))
    if rc:
        raise OracleError(rc)
    L = b.n_lists

    def arr(ptr, n, dt):
        return np.ctypeslib.as_array(ptr, (max(n, 1),))[:n].astype(dt, copy=True)

    out = dict(
        codec=codec, variant=variant, frame_quads=frame_quads,
        list_n=arr(b.list_n, L, np.uint32),
        ctrl_off=arr(b.ctrl_off, L + 1, np.uint64), data_off=arr(b.data_off, L + 1, np.uint64),
        exc_off=arr(b.exc_off, L + 1, np.uint64), out_off=arr(b.out_off, L + 1, np.uint64),
        ctrl=arr(b.ctrl, b.ctrl_bytes, np.uint8),
        data=arr(b.data, 4 * b.data_vectors, np.uint32).reshape(-1, 4),
        exc=arr(b.exc, b.exc_bytes, np.uint8),
        total_out=int(b.total_out),
    )
    lib().gco_batch_free(C.byref(b))
    return out


def _as_batch_struct(bt: dict):
    keep = {}

    def ptr(name, dt, ctype):
        a = np.ascontiguousarray(bt[name], dtype=dt).reshape(-1)
        if len(a) == 0:
            a = np.zeros(4, dt)
        keep[name] = a
        return a.ctypes.data_as(C.POINTER(ctype))

    L = len(bt["list_n"])
    b = Batch(L, ptr("list_n", np.uint32, C.c_uint32), ptr("ctrl_off", np.uint64, C.c_uint64),
              ptr("data_off", np.uint64, C.c_uint64), ptr("exc_off", np.uint64, C.c_uint64),
              ptr("out_off", np.uint64, C.c_uint64), ptr("ctrl", np.uint8, C.c_uint8),
              len(bt["ctrl"]), ptr("data", np.uint32, C.c_uint32), len(bt["data"]),
              ptr("exc", np.uint8, C.c_uint8), len(bt["exc"]), int(bt["total_out"]))
    return b, keep


def decode_batch(bt: dict, dgaps: bool = True, threads: int = 1, out: np.ndarray | None = None):
    """Decode a packed batch on the host; raises OracleError with the first bad list."""
    p = params(bt["codec"], bt.get("variant", 0), bt.get("frame_quads", 32))
    b, keep = _as_batch_struct(bt)
    if out is None:
        out = np.zeros(max(int(bt["total_out"]), 1), np.uint32)
    bad = C.c_uint64(0)
    rc = lib().gco_decode_batch(C.byref(p), C.byref(b), int(dgaps), threads, _u32p(out),
                                C.byref(bad))
    del keep
    if rc:
        raise OracleError(rc, f"list {bad.value}")
    return out[:int(bt["total_out"])]



SKIP_DIST = 512
# gco_skip_entry (gc_oracle.h): the skip pointer of one 512-int block of a list
SKIP_DTYPE = np.dtype([("data_bits", "<u8"), ("word", "<u4"), ("quads", "<u4"),
                       ("exc_bytes", "<u4"), ("docid", "<u4"), ("pad", "<u4", (2,))])


def build_skip(bt: dict):
    """Skip pointers every 512 postings (§7.5) of a packed batch: (skip_off uint64
    [L+1], entries SKIP_DTYPE [skip_off[L]]), by gco_build_skip's group-by-group walk."""
    p = params(bt["codec"], bt.get("variant", 0), bt.get("frame_quads", 32))
    b, keep = _as_batch_struct(bt)
    n_e = int(lib().gco_skip_entries(C.byref(b)))
    off = np.zeros(len(bt["list_n"]) + 1, np.uint64)
    ent = np.zeros(max(n_e, 1), SKIP_DTYPE)
    rc = lib().gco_build_skip(C.byref(p), C.byref(b), _u64p(off), ent.ctypes.data)
    del keep
    if rc:
        raise OracleError(rc, "gco_build_skip")
    return off, ent[:n_e]
