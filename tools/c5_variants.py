"""C5 (batched) with and without direct output stores of the window members' twins (lower.BATCH_DIRECT)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    from paper_2110_12865_b200 import lower

    args = bench.parse_args(["--config", "c5", "--only", "--no-cpu-baseline", "--steps", "5"] + sys.argv[1:])
    for direct in (False, True, False, True):
        lower.BATCH_DIRECT = direct
        line = bench.measure_batched(args, 0, 1, None)
        print(f"batch_direct={direct} ms {line['ms_per_step']:.4f} parity {line['config'].get('parity')}", flush=True)


if __name__ == "__main__":
    main()
