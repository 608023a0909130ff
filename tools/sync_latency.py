"""Host-side latency of observing a finished CUDA event (diagnostic):
cudaEventSynchronize vs polling cudaEventQuery, after a short kernel chain,
and the context's scheduling flags."""
import ctypes
import time

import numpy as np
import torch

torch.cuda.init()
x = torch.zeros(1, device="cuda")
rt = ctypes.CDLL("libcudart.so.12") if False else None
try:
    import glob
    import os
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    libs += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = ctypes.CDLL(libs[0])
    flags = ctypes.c_uint()
    rt.cudaGetDeviceFlags(ctypes.byref(flags))
    print("cudaGetDeviceFlags:", hex(flags.value), "(0 auto, 1 spin, 2 yield, 4 blocking)")
except Exception as e:  # noqa: BLE001
    print("flags unavailable:", e)
s = torch.cuda.current_stream()


def chain():
    for _ in range(20):
        x.add_(1)


for mode in ("sync", "query", "sync", "query"):
    lat = []
    for _ in range(200):
        chain()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(s)
        t0 = time.perf_counter()
        if mode == "sync":
            ev.synchronize()
        else:
            while not ev.query():
                pass
        lat.append((time.perf_counter() - t0) * 1e6)
    print(f"{mode:6s}: median {np.median(lat):.1f} us  p90 {np.percentile(lat, 90):.1f} us")
