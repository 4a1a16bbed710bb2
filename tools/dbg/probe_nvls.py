"""Probe (measurement only): does this box expose NVLS multicast to one process?
Driver attribute, and torch symmetric memory's multicast pointer at world size 1."""
import ctypes
import os

import torch
import torch.distributed as dist

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
v = ctypes.c_int()
for name, a in (("MULTICAST_SUPPORTED", 132), ("FABRIC_HANDLE", 128), ("POSIX_FD_HANDLE", 103)):
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), a, dev)
    print(name, r, v.value)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, dtype=torch.float32, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("symm ok; multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", h.buffer_ptrs)
except Exception as e:  # noqa: BLE001
    print("symm failed:", repr(e))
dist.destroy_process_group()
