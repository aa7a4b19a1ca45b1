"""FP64 / FP32 FMA peaks of this GPU ("measure FP64/FP32 peaks on the GPU box with
a DFMA/FFMA dependent-chain microbenchmark, all SMs"), through ab_peak_flops (8 independent FMA
chains per thread), median of 5, with the SM count, L2 size and the SM clock sampled by NVML
during the runs.  Prints one JSON object (committed as profiles/peaks_<round>.json)."""
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

clocks = []
stop = False


def sample():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop:
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)
    except Exception:  # NVML missing: clocks stay empty
        pass


eng = E.make(I.config(1), "fp64")
th = threading.Thread(target=sample, daemon=True)
th.start()
out = {}
for name, code in (("fp64", E.AB_FP64), ("fp32", E.AB_MIXED)):
    vals = []
    for _ in range(5):
        tf = C.c_double()
        assert eng.L.ab_peak_flops(eng.h, code, C.byref(tf)) == 0
        vals.append(tf.value)
    out[name + "_fma_tflops"] = {"median": round(statistics.median(vals), 3), "all": [round(v, 3) for v in vals]}
stop = True
th.join()
p = torch.cuda.get_device_properties(0)
out.update({"device": p.name, "sm_count": p.multi_processor_count,
            "l2_bytes": getattr(p, "L2_cache_size", None),
            "sm_mhz_median_during": statistics.median(clocks) if clocks else None,
            "sm_mhz_max_during": max(clocks) if clocks else None,
            "method": "ab_peak_flops: all SMs, 8 independent DFMA/FFMA chains per thread, 2 flops per FMA; "
                      "nominal = SMs x 64 (FP64) / 128 (FP32) FMA/clk x 2 x clock"})
if clocks:
    mhz = statistics.median(clocks)
    out["nominal_fp64_tflops_at_median_clock"] = round(p.multi_processor_count * 64 * 2 * mhz * 1e6 / 1e12, 3)
    out["nominal_fp32_tflops_at_median_clock"] = round(p.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12, 3)
print(json.dumps(out))
eng.close()
