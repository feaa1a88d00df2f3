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
        stage = "start"
        try:
            ctx = ok(cu.cuDevicePrimaryCtxRetain(ok(cu.cuDeviceGet(0))))
            ok(cu.cuCtxSetCurrent(ctx))
            prop = cu.CUmulticastObjectProp()
            prop.numDevices = n
            prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
            prop.size = 1 << 21
            stage = "granularity"
            gmin = ok(cu.cuMulticastGetGranularity(
                prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM))
            gran = ok(cu.cuMulticastGetGranularity(
                prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
            out["granularity"] = {"minimum": int(gmin), "recommended": int(gran)}
            size = int(gran)
            prop.size = size
            stage = "create"
            mc = ok(cu.cuMulticastCreate(prop))
            for d in range(n):
                stage = "add_device %d" % d
                ok(cu.cuMulticastAddDevice(mc, ok(cu.cuDeviceGet(d))))
            for d in range(n):
                ap = cu.CUmemAllocationProp()
                ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
                ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
                ap.location.id = d
                ap.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
                stage = "mem_create %d" % d
                mem = ok(cu.cuMemCreate(size, ap, 0))
                stage = "bind %d" % d
                ok(cu.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
            stage = "reserve"
            va = ok(cu.cuMemAddressReserve(size, int(gran), 0, 0))
            stage = "map"
            ok(cu.cuMemMap(va, size, 0, mc, 0))
            acc = cu.CUmemAccessDesc()
            acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            acc.location.id = 0
            acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            stage = "set_access"
            ok(cu.cuMemSetAccess(va, size, [acc], 1))
            out["multicast_object"] = {"ok": True, "size": int(size)}
        except Exception as exc:  # noqa: BLE001
            out["multicast_object"] = {"ok": False, "stage": stage, "error": repr(exc)[:300]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
