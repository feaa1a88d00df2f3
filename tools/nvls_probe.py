#!/usr/bin/env python
"""Probe NVLink SHARP / multicast (NVLS) on this box: the device attribute,
and whether a multicast object spanning every visible GPU can be created,
bound to each GPU's memory and mapped (one process, driver API through
cuda-python).  Prints one JSON line."""

import json
import subprocess

from cuda.bindings import driver as cu


def ok(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return res[1:] if isinstance(res, tuple) and len(res) > 2 else (res[1] if isinstance(res, tuple) and len(res) == 2 else None)


def main():
    out = {}
    ok(cu.cuInit(0))
    n = ok(cu.cuDeviceGetCount())
    out["devices"] = n
    attrs = []
    for d in range(n):
        dev = ok(cu.cuDeviceGet(d))
        attrs.append(ok(cu.cuDeviceGetAttribute(
            cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)))
    out["multicast_supported"] = attrs
    try:
        out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True,
                                     text=True, timeout=20).stdout[:1500]
    except Exception as exc:  # noqa: BLE001
        out["topo"] = repr(exc)
    if n >= 2 and all(attrs):
        try:
            ctx = ok(cu.cuDevicePrimaryCtxRetain(ok(cu.cuDeviceGet(0))))
            ok(cu.cuCtxSetCurrent(ctx))
            prop = cu.CUmulticastObjectProp()
            prop.numDevices = n
            prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
            prop.size = 1 << 21
            gran = ok(cu.cuMulticastGetGranularity(
                prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
            size = max(gran, 1 << 21)
            prop.size = size
            mc = ok(cu.cuMulticastCreate(prop))
            for d in range(n):
                ok(cu.cuMulticastAddDevice(mc, ok(cu.cuDeviceGet(d))))
            for d in range(n):
                ap = cu.CUmemAllocationProp()
                ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
                ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
                ap.location.id = d
                mem = ok(cu.cuMemCreate(size, ap, 0))
                ok(cu.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
            va = ok(cu.cuMemAddressReserve(size, 0, 0, 0))
            ok(cu.cuMemMap(va, size, 0, mc, 0))
            acc = cu.CUmemAccessDesc()
            acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            acc.location.id = 0
            acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            ok(cu.cuMemSetAccess(va, size, [acc], 1))
            out["multicast_object"] = {"ok": True, "granularity": int(gran), "size": int(size)}
        except Exception as exc:  # noqa: BLE001
            out["multicast_object"] = {"ok": False, "error": repr(exc)[:300]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
