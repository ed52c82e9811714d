"""C5 (batched) under jit.BATCH_VEC (value sets per lane per iteration of the batched kernels)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    from paper_2110_12865_b200 import jit

    args = bench.parse_args(["--config", "c5", "--only", "--no-cpu-baseline", "--steps", "5"])
    for bvec in (8, 4, 2, 16):
        jit.BATCH_VEC = bvec
        line = bench.measure_batched(args, 0, 1, None)
        print(f"batch_vec={bvec} ms {line['ms_per_step']:.4f} parity {line['config'].get('parity')}", flush=True)


if __name__ == "__main__":
    main()
