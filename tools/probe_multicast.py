"""Tools only: does this GPU support multicast objects (NVLS) for a one-device group?"""
from cuda import cuda
cuda.cuInit(0)
err, dev = cuda.cuDeviceGet(0)
err, v = cuda.cuDeviceGetAttribute(cuda.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("multicast supported:", err, v)
err, ctx = cuda.cuDevicePrimaryCtxRetain(dev)
cuda.cuCtxSetCurrent(ctx)
prop = cuda.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = cuda.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
err, gran = cuda.cuMulticastGetGranularity(prop, cuda.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
print("granularity:", err, gran)
prop.size = max(gran, 2 << 20)
err, mc = cuda.cuMulticastCreate(prop)
print("create:", err)
if err == cuda.CUresult.CUDA_SUCCESS:
    print("addDevice:", cuda.cuMulticastAddDevice(mc, dev)[0])
