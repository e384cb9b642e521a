#!/usr/bin/env python3
"""Dev probe: which NVML NVLink counters this driver exposes (return code and
value per field / link), read before and after a 1 GiB peer copy 0 -> 1."""
import pynvml as nv
import torch

nv.nvmlInit()
FIELDS = {138: "THROUGHPUT_DATA_TX", 139: "THROUGHPUT_DATA_RX", 140: "THROUGHPUT_RAW_TX", 141: "THROUGHPUT_RAW_RX",
          201: "COUNT_XMIT_PACKETS", 202: "COUNT_XMIT_BYTES", 203: "COUNT_RCV_PACKETS", 204: "COUNT_RCV_BYTES"}


def read(dev):
    h = nv.nvmlDeviceGetHandleByIndex(dev)
    out = {}
    for f in FIELDS:
        vals = nv.nvmlDeviceGetFieldValues(h, [(f, l) for l in range(18)])
        out[f] = [(v.nvmlReturn, v.value.ullVal) for v in vals]
    return out


def link_util(dev):
    h = nv.nvmlDeviceGetHandleByIndex(dev)
    res = []
    for l in range(18):
        try:
            res.append(nv.nvmlDeviceGetNvLinkState(h, l))
        except nv.NVMLError as e:
            res.append(str(e))
    return res


print("link states gpu0:", link_util(0))
a = read(0)
b1 = read(1)
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
for _ in range(4):
    y.copy_(x)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
import time
time.sleep(1.0)
a2 = read(0)
b2 = read(1)
for f, name in FIELDS.items():
    rc0 = sorted(set(r for r, _ in a[f]))
    d0 = sum(v2 - v1 for (_, v1), (_, v2) in zip(a[f], a2[f]))
    d1 = sum(v2 - v1 for (_, v1), (_, v2) in zip(b1[f], b2[f]))
    print(f"{f} {name}: rc {rc0} gpu0 delta {d0} gpu1 delta {d1} (4 GiB copied 0->1); sample {a2[f][:4]}")
