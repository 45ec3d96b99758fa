"""QNTC named-tensor container (the reference's weight / artifact exchange
format, io.hpp:33-60, io.cpp:100-171) and the weight hand-off through it.

`pack_tensors` / `unpack_tensors` are byte-for-byte the reference's
`pack_tensors` / `unpack_tensors` (same layout, same validation order, same
IoError / SchemaError messages). A parameter store packed by either side
loads onto the device with `Model.load_weights_qntc` (C ABI
`lvsg_load_weights_qntc`), bound by position like bind_params
(network.hpp:330-339). `param_names` gives the NetParams member path of
every build_params tensor (network.hpp:95-132), which `pack_param_store`
uses as entry names.
"""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import capi
from .capi import IoError
from .config import ModelConfig, SchemaError

VERSION = 1  # kTensorContainerVersion (io.hpp:44)
_DTYPES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


@dataclass
class NamedTensor:
    """io.hpp:46-60. `array` is float32 (tag 0) or float64 (tag 1)."""
    name: str
    array: np.ndarray

    @property
    def dtype_tag(self) -> int:
        return 1 if self.array.dtype == np.float64 else 0

    def as_f32(self) -> np.ndarray:
        if self.dtype_tag != 0:
            raise SchemaError(f'tensor container: entry "{self.name}" holds f64, expected f32')
        return self.array

    def as_f64(self) -> np.ndarray:
        if self.dtype_tag != 1:
            raise SchemaError(f'tensor container: entry "{self.name}" holds f32, expected f64')
        return self.array


def pack_tensors(entries: Sequence[Tuple[str, np.ndarray]]) -> bytes:
    """pack_tensors (io.cpp:100-124): float64 arrays keep tag 1, everything
    else is stored as float32."""
    out = [b"QNTC", struct.pack("<II", VERSION, len(entries))]
    for name, arr in entries:
        a = np.asarray(arr)
        a = np.ascontiguousarray(a, "<f8" if a.dtype == np.float64 else "<f4")
        nb = name.encode()
        out.append(struct.pack("<I", len(nb)) + nb)
        out.append(struct.pack("<BI", 1 if a.dtype == np.float64 else 0, a.ndim))
        out.append(struct.pack(f"<{a.ndim}Q", *a.shape))
        out.append(a.tobytes())
    return b"".join(out)


class _Reader:
    def __init__(self, buf: bytes):
        self.buf, self.pos = memoryview(buf), 0

    def take(self, n: int, what: str) -> memoryview:
        if n > len(self.buf) - self.pos:
            raise IoError(f"tensor container: truncated {what}")
        v = self.buf[self.pos:self.pos + n]
        self.pos += n
        return v

    def u(self, fmt: str, what: str) -> int:
        return struct.unpack("<" + fmt, self.take(struct.calcsize(fmt), what))[0]


def unpack_tensors(data: bytes) -> List[NamedTensor]:
    """unpack_tensors (io.cpp:126-171)."""
    r = _Reader(bytes(data))
    magic = bytes(r.take(4, "magic")).decode("latin-1")
    if magic != "QNTC":
        raise IoError(f'tensor container: bad magic "{magic}"')
    version = r.u("I", "version")
    if version != VERSION:
        raise IoError(f"tensor container: unsupported version {version}")
    count = r.u("I", "entry count")
    if count > (1 << 20):
        raise IoError("tensor container: implausible entry count")
    out = []
    for i in range(count):
        at = f"entry {i}"
        nl = r.u("I", f"{at} name length")
        if nl > (1 << 16):
            raise IoError(f"tensor container: {at}: implausible name length")
        name = bytes(r.take(nl, f"{at} name")).decode("utf-8", "surrogateescape")
        tag = r.u("B", f"{at} dtype")
        if tag > 1:
            raise IoError(f'tensor container: {at} ("{name}"): unknown dtype tag {tag}')
        rank = r.u("I", f"{at} rank")
        if rank > 16:
            raise IoError(f"tensor container: {at}: implausible rank")
        dims, n = [], 1
        for _ in range(rank):
            ext = r.u("Q", f"{at} dims")
            if ext > (1 << 32):
                raise IoError(f"tensor container: {at}: implausible extent")
            dims.append(ext)
            n *= ext
            if n > (1 << 33):
                raise IoError(f"tensor container: {at}: implausible element count")
        dt = _DTYPES[tag]
        raw = r.take(n * dt.itemsize, f'{at} ("{name}") payload')
        out.append(NamedTensor(name, np.frombuffer(raw, dt).reshape(dims).copy()))
    if r.pos != len(r.buf):
        raise IoError(f"tensor container: {len(r.buf) - r.pos} trailing bytes after the last entry")
    return out


def find_tensor(entries: Sequence[NamedTensor], name: str) -> NamedTensor:
    """find_tensor (io.cpp:181-185)."""
    for e in entries:
        if e.name == name:
            return e
    raise SchemaError(f'tensor container: missing entry "{name}"')


def param_names(cfg: ModelConfig) -> List[str]:
    """NetParams member path of every build_params tensor, in order."""
    cc = cfg.to_c()
    n, tot = ctypes.c_int64(), ctypes.c_int64()
    L = capi.lib()
    capi.raise_for(L.lvsg_param_count(cc.ptr, ctypes.byref(n), ctypes.byref(tot)), "bad config")
    buf = ctypes.create_string_buffer(256)
    out = []
    for i in range(n.value):
        capi.raise_for(L.lvsg_param_name(cc.ptr, i, buf, 256), "bad parameter index")
        out.append(buf.value.decode())
    return out


def pack_param_store(cfg: ModelConfig, seed: int) -> bytes:
    """init_param_store(cfg, seed) as a QNTC container, packed by the native
    library (lvsg_pack_param_store_qntc)."""
    cc = cfg.to_c()
    L = capi.lib()
    n = ctypes.c_size_t()
    capi.raise_for(L.lvsg_pack_param_store_qntc(cc.ptr, seed, None, 0, ctypes.byref(n)), "bad config")
    buf = ctypes.create_string_buffer(n.value)
    capi.raise_for(L.lvsg_pack_param_store_qntc(cc.ptr, seed, buf, n.value, ctypes.byref(n)),
                   "bad config")
    return buf.raw[:n.value]
