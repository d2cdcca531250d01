"""Where a native run_ea generation loop spends its time (PhaseProfile)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2502_11129_b200 as hb  # noqa: E402
from paper_2502_11129_b200.ea import run_ea_native  # noqa: E402


def main():
    ex = hb.GpuExecutor(0)
    for model in sys.argv[1:] or ["box", "box_and_ball"]:
        kind = hb.parse_model_kind(model)
        run_ea_native(kind, 65536, 5, 1000, ex)
        for _ in range(3):
            t0 = time.perf_counter()
            r = run_ea_native(kind, 65536, 5, 1000, ex)
            w = time.perf_counter() - t0
            p = r.profile
            print(f"{model}: wall {w*1e3:.2f} ms  sel {p.selection_s*1e3:.2f}  eval {p.evaluation_s*1e3:.2f}  "
                  f"book {p.bookkeeping_s*1e3:.2f}  total {p.total_s*1e3:.2f} ms")


if __name__ == "__main__":
    main()
