"""run_ea_sharded_device in a one-rank NCCL group vs the native hb_run_ea
(per-generation overhead of the multi-GPU loop; run under gpurun)."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402
from paper_2502_11129_b200 import distributed as hbd  # noqa: E402


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    ex = hb.GpuExecutor(0)
    for model in ("box", "box_and_ball"):
        kind = hb.parse_model_kind(model)
        a = hbd.run_ea_sharded_device(kind, 65536, 5, 1000, ex, dist)
        b = hb.run_ea(kind, 65536, 5, 1000, ex)
        assert np.array_equal(a.population.genomes, b.population.genomes)
        for name, fn in (("sharded_device", lambda: hbd.run_ea_sharded_device(kind, 65536, 5, 1000, ex, dist)),
                         ("native", lambda: hb.run_ea(kind, 65536, 5, 1000, ex))):
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            print(f"{model} {name}: {1e3 * min(ts):.2f} ms per 5-generation loop")
        r = hbd.run_ea_sharded_device(kind, 65536, 5, 1000, ex, dist)
        p = r.profile
        print(f"  sharded profile: sel {1e3*p.selection_s:.2f} eval {1e3*p.evaluation_s:.2f} "
              f"book {1e3*p.bookkeeping_s:.2f} total {1e3*p.total_s:.2f} ms")
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
        hbd.run_ea_sharded_device(kind, 65536, 5, 1000, ex, dist)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(8)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
