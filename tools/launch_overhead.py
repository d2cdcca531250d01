"""Box launch fixed cost: CUDA-event time of a 1-step / 1000-step launch with
and without the L2 flush before it, and back-to-back launches (diagnostic)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402


def main():
    ex = hb.GpuExecutor(0)
    ctx = ex.ctx
    dev = torch.device("cuda:0")
    ext = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ctx.stage(0, np.arange(16384, dtype=np.uint64))
    for steps in (1, 1000):
        for mode in ("flush", "noflush", "b2b"):
            res = []
            with torch.cuda.stream(ext):
                for rep in range(13):
                    if mode == "flush":
                        flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(ext)
                    for _ in range(20 if mode == "b2b" else 1):
                        ctx.launch(steps)
                    e1.record(ext)
                    e1.synchronize()
                    if rep >= 3:
                        res.append(e0.elapsed_time(e1) * 1e3 / (20 if mode == "b2b" else 1))
            print(f"steps {steps:5d} {mode:8s}: median {np.median(res):7.2f} us/launch")


if __name__ == "__main__":
    main()
