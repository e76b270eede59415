"""A/B timing of the single-domain step through the bare C-ABI (works with any
build of libd2q37_b200.so, old or new): 4096 x 16384 RT init, wall bc.
usage: python tools/ab_step.py LIB [layout vl variant steps lx ly]"""
import ctypes as C
import os
import statistics
import sys
import threading
import time

lib = C.CDLL(sys.argv[1])
layout = {"aos": 0, "soa": 1, "csoa": 2, "caosoa": 3, "banded": 4}[sys.argv[2] if len(sys.argv) > 2 else "caosoa"]
vl = int(sys.argv[3]) if len(sys.argv) > 3 else 32
mode = sys.argv[4] if len(sys.argv) > 4 else "fused"  # fused | unfused | propagate (config 1 verb)
variant = {"unfused": 0, "fused": 1, "propagate": 1, "fused2": 2}[mode]
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 200
lx = int(sys.argv[6]) if len(sys.argv) > 6 else 4096
ly = int(sys.argv[7]) if len(sys.argv) > 7 else 16384
lib.d2q37_step.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int]
lib.d2q37_sync.argtypes = [C.c_void_p]
lib.d2q37_init_rt_device.argtypes = [C.c_void_p, C.c_uint64]
lib.d2q37_destroy.argtypes = [C.c_void_p]
h = C.c_void_p()
assert lib.d2q37_create(layout, lx, ly, vl if layout >= 2 else 1, 0, C.byref(h)) == 0
assert lib.d2q37_init_rt_device(h, 2018) == 0
if mode == "propagate":
    lib.d2q37_bc.argtypes = [C.c_void_p, C.c_int]
    lib.d2q37_propagate.argtypes = [C.c_void_p]
    assert lib.d2q37_bc(h, 0) == 0


def run(n):
    if mode == "propagate":
        for _ in range(n):
            assert lib.d2q37_propagate(h) == 0
    else:
        assert lib.d2q37_step(h, 0.8, n, variant, 1) == 0
run(20)
lib.d2q37_sync(h)
samples = []
stop = threading.Event()


def sample():
    try:
        import pynvml as nv
        nv.nvmlInit()
        d = nv.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            samples.append((nv.nvmlDeviceGetClockInfo(d, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(d) / 1e3))
            time.sleep(0.05)
    except Exception:
        pass


th = threading.Thread(target=sample, daemon=True)
th.start()
best = 1e30
for _ in range(3):
    t0 = time.perf_counter()
    run(steps)
    rc = lib.d2q37_sync(h)
    assert rc == 0 or os.environ.get("AB_IGNORE_ERRORS")  # timing-only variants may compute garbage
    best = min(best, time.perf_counter() - t0)
stop.set()
th.join()
sm = statistics.median(s[0] for s in samples) if samples else 0
pw = statistics.median(s[1] for s in samples) if samples else 0
print(f"{sys.argv[1].split('/')[-1]} ms/step {1e3 * best / steps:.4f} MLUPS {lx * ly * steps / best / 1e6:.1f} "
      f"sm_mhz {sm:.0f} power_w {pw:.0f}")
lib.d2q37_destroy(h)
