"""C5 (batched) under code-generation knobs: jit.INDEX64, lower.STORE_ROOTS_EARLY.  One GPU."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    from paper_2110_12865_b200 import jit, lower

    args = bench.parse_args(["--config", "c5", "--only", "--no-cpu-baseline", "--steps", "5"])
    for idx64, early in ((True, False), (False, False), (False, True), (True, True), (True, False)):
        jit.INDEX64, lower.STORE_ROOTS_EARLY = idx64, early
        line = bench.measure_batched(args, 0, 1, None)
        print(f"index64={idx64} early={early} ms {line['ms_per_step']:.4f} parity {line['config'].get('parity')}",
              flush=True)


if __name__ == "__main__":
    main()
