"""The reference's collective benchmark protocol (cli.py:246-294) through
paper_1901_04359_b200.bench_protocol.run_bench: every column but the wall
times equal to the reference's own rows (tests/golden/bench_rows.txt, made by
tests/golden/make_bench_rows.py from the reference itself)."""

import os

import pytest

from conftest import ROOT, cuda_ok

GOLD = os.path.join(ROOT, "tests", "golden", "bench_rows.txt")


def golden_cases():
    cases, cur = [], None
    with open(GOLD) as fh:
        for line in fh:
            line = line.strip()
            if line.startswith("#"):
                P, m, rho = line[1:].split()
                cur = (int(P), int(m), float(rho), [])
                cases.append(cur)
            elif line:
                cur[3].append(line)
    return cases


def test_golden_rows_header_and_rounds():
    """Host side: the header is the reference's; rounds per collective follow
    comm_rounds (reference collectives.py:60-74)."""
    from paper_1901_04359_b200 import bench_protocol, collectives

    assert bench_protocol.BENCH_HEADER == ("collective,P,m,k,rank,bytes_sent,bytes_recv,msgs,rounds,wall_ms,"
                                           "wall_ms_std")
    for P, m, rho, rows in golden_cases():
        assert len(rows) == 3 * P
        for r in rows:
            algo, p, *_rest, rounds = r.split(",")
            assert int(p) == P and int(rounds) == collectives.comm_rounds(algo, P)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA GPU")
@pytest.mark.parametrize("case", range(5))
def test_run_bench_rows_match_reference(case):
    from paper_1901_04359_b200 import bench_protocol

    P, m, rho, want = golden_cases()[case]
    got = bench_protocol.run_bench(P, m=m, rho=rho, warmup_reps=1, repeats=2)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        cols = g.split(",")
        assert ",".join(cols[:-2]) == w  # everything but wall_ms, wall_ms_std
        assert float(cols[-2]) > 0.0 or P == 1
