#!/usr/bin/env python
"""Device quantize (amsq_quantize_device) vs the host quantizer: weights/s on Llama shapes.

The device run quantizes the whole tensor (CUDA events around the synchronous call); the host
run (all hardware threads, the library's bit-identical C++ quantizer) a row slice of it.
Prints one JSON line per (scheme, shape)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_16045_b200 as amsq  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for name in ("fp5.33-e2m3", "fp4.25-e2m2"):
        sid = amsq.scheme_by_name(name).id
        for rows, cols in ((28672, 4096), (57344, 8192)):
            w = torch.randn(rows, cols, device=dev)
            amsq.quantize_tensor_device(w, sid, to_host=False)  # warm-up
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                amsq.quantize_tensor_device(w, sid, to_host=False)
                ts.append(time.perf_counter() - t0)
            t_dev = min(ts)
            nh = 512
            wh = w[:nh].cpu().numpy()
            t0 = time.perf_counter()
            amsq.quantize_tensor(wh, sid, threads=0)
            t_host = time.perf_counter() - t0
            print(json.dumps({"scheme": name, "rows": rows, "cols": cols,
                              "device_s": round(t_dev, 4),
                              "device_Mweights_per_s": round(rows * cols / t_dev / 1e6, 1),
                              "host_Mweights_per_s": round(nh * cols / t_host / 1e6, 2),
                              "host_threads": os.cpu_count(),
                              "speedup": round((rows * cols / t_dev) / (nh * cols / t_host), 1)}))
            del w
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
