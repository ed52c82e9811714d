"""C3 / C4 bench measurement with and without L2 evict_last stores for the last wave's output groups
(lower.KEEP_BEFORE_GATHER: the output gather reads them next)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    from paper_2110_12865_b200 import lower

    args = bench.parse_args(["--only", "--no-cpu-baseline", "--steps", "20"])
    for cfg in ("c3", "c4"):
        for keep in (False, True, False, True):
            lower.KEEP_BEFORE_GATHER = keep
            line = bench.measure_eval(cfg, args, 0, 1, None)
            print(f"{cfg} keep={keep} ms {line['ms_per_step']:.4f} launches "
                  f"{[(l_['name'], round(l_['ms'], 4)) for l_ in line['launches']]} parity "
                  f"{line['config'].get('parity')}", flush=True)


if __name__ == "__main__":
    main()
