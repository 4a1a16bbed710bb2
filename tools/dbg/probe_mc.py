"""Probe (measurement only): which cuMulticastCreate arguments this box accepts."""
import ctypes as ct

import torch

torch.cuda.init()
torch.empty(1, device="cuda")  # a current context
cu = ct.CDLL("libcuda.so.1")


class Prop(ct.Structure):
    _fields_ = [("numDevices", ct.c_uint), ("size", ct.c_size_t), ("handleTypes", ct.c_ulonglong),
                ("flags", ct.c_ulonglong)]


for nd in (1, 2):
    for ht in (0, 1, 8):
        p = Prop(nd, 2 << 20, ht, 0)
        g = ct.c_size_t(0)
        r0 = cu.cuMulticastGetGranularity(ct.byref(g), ct.byref(p), 1)
        p.size = max(g.value, 2 << 20)
        h = ct.c_ulonglong(0)
        r = cu.cuMulticastCreate(ct.byref(h), ct.byref(p))
        print(f"numDevices={nd} handleTypes={ht} gran_rc={r0} gran={g.value} create_rc={r}")
        if r == 0:
            rr = cu.cuMulticastAddDevice(h, 0)
            print("   add_device rc", rr)
            cu.cuMemRelease(h)
