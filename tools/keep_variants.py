"""C2 bench measurement (graph replay, per-wave launches) with and without L2 evict_last stores for
the wave feeding the window unit (lower.KEEP_BEFORE_WINDOW)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    from paper_2110_12865_b200 import lower

    args = bench.parse_args(["--only", "--no-cpu-baseline", "--steps", "20"])
    for keep in (1, 2, 3, 1):
        lower.KEEP_WAVES = keep
        line = bench.measure_eval("c2", args, 0, 1, None)
        print(f"keep={keep} ms {line['ms_per_step']:.4f} launches "
              f"{[(l_['name'], round(l_['ms'], 4)) for l_ in line['launches']]} parity {line['config'].get('parity')}",
              flush=True)


if __name__ == "__main__":
    main()
