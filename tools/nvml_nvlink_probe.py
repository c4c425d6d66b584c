"""Probe the NVML NVLink data counters on a multi-GPU box: copy 1 GiB GPU0 -> GPU1 and print the
per-link counter deltas (field ids 138/139 = NVLINK_THROUGHPUT_DATA_TX/RX, KiB)."""
import pynvml as nv
import torch

nv.nvmlInit()
h = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(torch.cuda.device_count())]


def read(dev):
    out = {}
    for l in range(18):
        try:
            st = nv.nvmlDeviceGetNvLinkState(h[dev], l)
        except Exception as ex:
            continue
        vals = nv.nvmlDeviceGetFieldValues(h[dev], [(138, l), (139, l)])
        out[l] = [(v.nvmlReturn, v.value.ullVal) for v in vals]
    vals = nv.nvmlDeviceGetFieldValues(h[dev], [138, 139])
    out["all"] = [(v.nvmlReturn, v.value.ullVal) for v in vals]
    return out


a = torch.ones(256 * 1024 * 1024, device="cuda:0")
b = torch.empty_like(a, device="cuda:1")
r0 = [read(0), read(1)]
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize()
r1 = [read(0), read(1)]
for d in (0, 1):
    for k in r0[d]:
        print(d, k, r0[d][k], r1[d][k])
