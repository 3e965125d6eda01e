"""Diagnostic: compare a tensor map encoded the way the library does with the
one Triton's launcher builds for the same plane (Triton is not used by the
product)."""
import ctypes
import torch
import triton

a = torch.arange(480 * 640, dtype=torch.float64, device="cuda").reshape(480, 640)
util = triton.runtime.driver.active.utils
obj = util.fill_tma_descriptor(a.data_ptr(), 0, 8, 8, [16, 16], [480, 640], [640, 1], 0)
tri = ctypes.string_at(id(obj) + 128, 128)
cuda = ctypes.CDLL("libcuda.so.1")
buf = ctypes.create_string_buffer(128 + 256)
addr = (ctypes.addressof(buf) + 127) & ~127
u64 = ctypes.c_uint64
dims = (u64 * 2)(640, 480)
strides = (u64 * 1)(640 * 8)
box = (ctypes.c_uint32 * 2)(16, 16)
es = (ctypes.c_uint32 * 2)(1, 1)
r = cuda.cuTensorMapEncodeTiled(ctypes.c_void_p(addr), 8, 2, ctypes.c_void_p(a.data_ptr()), dims,
                                strides, box, es, 0, 0, 2, 0)
mine = ctypes.string_at(addr, 128)
print("encode", r)
print("triton", tri.hex())
print("mine  ", mine.hex())
print("equal", tri == mine)
