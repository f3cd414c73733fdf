"""Does cuTensorMapEncodeTiled accept a dimension whose stride overlaps the
previous dimension's extent (a 'tap' view: stride = one 16-byte pixel)?"""
import ctypes as C

cuda = C.CDLL("libcuda.so.1")
cuda.cuInit(0)
enc = cuda.cuTensorMapEncodeTiled
tm = (C.c_uint8 * 128)()
dims = (C.c_uint64 * 5)(2 * 34, 4, 512 * 34, 2, 6)
strides = (C.c_uint64 * 4)(16, 34 * 16 * 2, 34 * 16, 512 * 34 * 2 * 34 * 16)
box = (C.c_uint32 * 5)(64, 4, 1, 2, 6)
es = (C.c_uint32 * 5)(1, 1, 1, 1, 1)
# need a device pointer: allocate with cuMemAlloc after a context
ctx = C.c_void_p()
dev = C.c_int()
cuda.cuDeviceGet(C.byref(dev), 0)
cuda.cuDevicePrimaryCtxRetain(C.byref(ctx), dev)
cuda.cuCtxSetCurrent(ctx)
ptr = C.c_uint64()
print("alloc", cuda.cuMemAlloc_v2(C.byref(ptr), C.c_size_t(1 << 30)))
# CU_TENSOR_MAP_DATA_TYPE_UINT64 = 4? enumerate: UINT8=0, UINT16=1, UINT32=2, INT32=3, UINT64=4
for dt in (4,):
    r = enc(tm, dt, 5, C.c_void_p(ptr.value), dims, strides, box, es, 0, 0, 3, 0)
    print("overlapping kx dim (stride 16 B): rc =", r)
strides2 = (C.c_uint64 * 4)(34 * 16 * 2 * 4, 34 * 16 * 2, 34 * 16, 512 * 34 * 2 * 34 * 16)
print("non-overlapping control: rc =", enc(tm, 4, 5, C.c_void_p(ptr.value), dims, strides2, box, es, 0, 0, 3, 0))
