"""Probe the GPU box: devices, P2P, NVLink, multicast support, host cores."""
import os, subprocess, torch, json
out = {}
out["ngpu"] = torch.cuda.device_count()
out["cores"] = len(os.sched_getaffinity(0))
out["names"] = [torch.cuda.get_device_name(i) for i in range(out["ngpu"])]
out["p2p"] = [[torch.cuda.can_device_access_peer(i, j) if i != j else True for j in range(out["ngpu"])] for i in range(out["ngpu"])]
try:
    from cuda.bindings import driver as drv
    drv.cuInit(0)
    res = {}
    for i in range(out["ngpu"]):
        _, dev = drv.cuDeviceGet(i)
        for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
                     "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", "CU_DEVICE_ATTRIBUTE_MULTI_PROCESSOR_COUNT",
                     "CU_DEVICE_ATTRIBUTE_COOPERATIVE_LAUNCH"]:
            a = getattr(drv.CUdevice_attribute, name)
            _, v = drv.cuDeviceGetAttribute(a, dev)
            res.setdefault(i, {})[name] = v
    out["attrs"] = res
except Exception as e:
    out["attrs_err"] = repr(e)
print(json.dumps(out, indent=1))
