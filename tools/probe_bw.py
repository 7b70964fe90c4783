"""Measured read ceilings on this B200: LDG streaming, bulk-TMA streaming, random
256-byte row gather at the V-gather density. Usage: python tools/probe_bw.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import subprocess  # noqa: E402

_DIAG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "diag")
subprocess.run(["make", "-C", _DIAG], check=True)  # probes live outside the product .so
lib = ctypes.CDLL(os.path.join(_DIAG, "libalaya_diag.so"))
lib.alaya_diag_read.restype = ctypes.c_int
lib.alaya_diag_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
dev = torch.device("cuda")
nbytes = 8 << 30
buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
buf.random_()
sink = torch.zeros(4, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream
out = {}


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


for mode, name in [(0, "ldg_stream"), (1, "bulk_tma_stream"), (3, "tma2d_two_boxes_stream"),
                   (4, "tma3d_one_box_stream")]:
    t = timeit(lambda: lib.alaya_diag_read(buf.data_ptr(), nbytes, mode, None, 0, sink.data_ptr(), st))
    out[name + "_GBps"] = round(nbytes / t / 1e9, 1)
# size dependence: one launch over the first S bytes (fixed per-launch ramp/drain cost)
for size in (268435456, 536870912, 1073741824, 2147483648):
    for mode, name in [(0, "ldg"), (1, "bulk"), (3, "tma2d")]:
        t = timeit(lambda: lib.alaya_diag_read(buf.data_ptr(), size, mode, None, 0, sink.data_ptr(), st), reps=20)
        out[f"{name}_{size >> 20}MB_us"] = round(t * 1e6, 1)
        out[f"{name}_{size >> 20}MB_GBps"] = round(size / t / 1e9, 1)
# V-gather pattern: 24% of 256-byte rows, random positions, ascending
rows_total = nbytes // 256
g = torch.Generator(device=dev).manual_seed(0)
mask = torch.rand(rows_total, device=dev, generator=g) < 0.24
rows = torch.nonzero(mask).view(-1).to(torch.int32)
t = timeit(lambda: lib.alaya_diag_read(buf.data_ptr(), nbytes, 2, rows.data_ptr(), rows.numel(),
                                       sink.data_ptr(), st))
out["gather256_24pct_GBps"] = round(rows.numel() * 256 / t / 1e9, 1)
for ctas in (1, 2, 4):  # warps in flight per SM = 8 * ctas, 16 rows per half-warp
    t = timeit(lambda: lib.alaya_diag_read(buf.data_ptr(), nbytes, 10 + ctas, rows.data_ptr(),
                                           rows.numel(), sink.data_ptr(), st))
    out[f"gather256_{8 * ctas}warps_per_sm_GBps"] = round(rows.numel() * 256 / t / 1e9, 1)
x = buf.view(torch.bfloat16)
t = timeit(lambda: torch.sum(x, dtype=torch.float32))
out["torch_sum_GBps"] = round(nbytes / t / 1e9, 1)
print(json.dumps(out))
