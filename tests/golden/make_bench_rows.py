"""Golden rows of the reference's collective benchmark (cli.py:246-294):
every column but the wall times, for a few (P, m, rho).  Run in the build
container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bench_rows.py

Writes tests/golden/bench_rows.txt: `P m rho` lines followed by the
reference's CSV rows with the wall columns cut.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from gtopk import cli  # noqa: E402  (the reference)

CASES = [(1, 5000, 0.01), (2, 10000, 0.01), (3, 10000, 0.001), (4, 20000, 0.005), (8, 10000, 0.01)]


def main():
    out = []
    for P, m, rho in CASES:
        cfg = cli.RunConfig(P=P, m=m, rho=rho, repeats=2, warmup_reps=1)
        rows = cli.run_bench(cfg)
        out.append(f"# {P} {m} {rho}")
        out += [",".join(r.split(",")[:-2]) for r in rows]  # drop wall_ms, wall_ms_std
    with open(os.path.join(HERE, "bench_rows.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
