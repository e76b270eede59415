"""Cost of the streamed run's pitched row copies (37 x cudaMemcpy2DAsync of 4096 rows, width = chunk rows x 8 B)
against the width, both directions.  usage: python tools/pitched_copy_probe.py"""
import time

import torch
from cuda.bindings import runtime as rt

lx, ly, npop = 4096, 16384, 37
pitch_d = (ly + 16) * 8
dev = torch.empty(lx * (ly + 16), dtype=torch.float64, device="cuda")
host = torch.empty(lx * ly, dtype=torch.float64).pin_memory()
(err, st) = rt.cudaStreamCreate()
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
for rows in (4, 12, 40, 64, 96, 120, 128, 240, 480, 960, 4440):
    for up in (True, False):
        best = 1e30
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for p in range(npop):
                if up:
                    (e,) = rt.cudaMemcpy2DAsync(dev.data_ptr() + 64, pitch_d, host.data_ptr(), ly * 8, rows * 8, lx, H2D, st)
                else:
                    (e,) = rt.cudaMemcpy2DAsync(host.data_ptr(), ly * 8, dev.data_ptr() + 64, pitch_d, rows * 8, lx, D2H, st)
                assert int(e) == 0, e
            rt.cudaStreamSynchronize(st)
            best = min(best, time.perf_counter() - t0)
        gb = npop * lx * rows * 8 / 1e9
        print(f"{'H2D' if up else 'D2H'} width {rows:5d} rows ({rows * 8:6d} B): {best * 1e3:8.2f} ms  {gb / best:6.1f} GB/s", flush=True)

# Two directions at once: stream A uploads 4 x 37 wide copies; stream B downloads 37 wide copies, optionally
# behind 37 narrow ones (the sliver first download of DESIGN 3.3).  When is B done, when is everything done?
(err, st2) = rt.cudaStreamCreate()
host2 = torch.empty(lx * ly, dtype=torch.float64).pin_memory()
for narrow in (0, 40, 12, 128, 240):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(4):
            for p in range(npop):
                (e,) = rt.cudaMemcpy2DAsync(dev.data_ptr() + 64 + k * 4440 * 8, pitch_d, host.data_ptr() + k * 4440 * 8, ly * 8,
                                            4440 * 8, lx, H2D, st)
        for rows in ([narrow] if narrow else []) + [4440]:
            for p in range(npop):
                (e,) = rt.cudaMemcpy2DAsync(host2.data_ptr(), ly * 8, dev.data_ptr() + 64 + 8000 * 8, pitch_d, rows * 8, lx, D2H, st2)
        t_issue = time.perf_counter() - t0
        rt.cudaStreamSynchronize(st2)
        t_b = time.perf_counter() - t0
        rt.cudaStreamSynchronize(st)
        t_all = time.perf_counter() - t0
    print(f"concurrent: narrow first download {narrow:4d} rows: issue {t_issue * 1e3:7.1f} ms, downloads done {t_b * 1e3:7.1f} ms, "
          f"all done {t_all * 1e3:7.1f} ms", flush=True)
