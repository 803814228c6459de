"""Probe: can a CUDA multicast object (NVLS) be created with one device here? (cuda-python driver API)"""
import torch
from cuda.bindings import driver as cu

torch.zeros(1, device="cuda")
ok, dev = cu.cuDeviceGet(0)
for ht in (0, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
    for nd in (1, 2):
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.size = 2 << 20
        prop.handleTypes = ht
        err, mc = cu.cuMulticastCreate(prop)
        print("handleTypes", int(ht) if not isinstance(ht, int) else ht, "numDevices", nd, "->", err)
        if err == cu.CUresult.CUDA_SUCCESS:
            print("  add device:", cu.cuMulticastAddDevice(mc, dev))
