"""CLI harness (paper_2309_09072_b200/harness.py; reference SPEC.md "harness",
SURVEY.md 8(f) rank 3).  CPU: parsing, FASTA ingestion, seeded instance
generation, log-linear fit, CSV schema, exit codes (solver stubbed where a
solve is needed).  GPU: the real commands."""

import io
import math

import pytest

from paper_2309_09072_b200 import harness as H
from paper_2309_09072_b200.seqcore import LcsResult


def test_fasta_first_record():
    data = b">seq1 desc\nACGT\nAC\n>seq2\nTTTT\n"
    assert H.parse_fasta(data) == b"ACGTAC"
    assert H.parse_fasta(b">only\n\n") == b""
    with pytest.raises(H.HarnessError) as e:
        H.parse_fasta(b"ACGT\n")
    assert e.value.code == H.EXIT_IO


def test_read_input_inline_file_fasta(tmp_path):
    p = tmp_path / "a.fa"
    p.write_bytes(b">x\ngatt\ntatg\n")
    assert H.read_input(str(p), fasta=True) == b"gatttatg"
    assert H.read_input(str(p), fasta=False) == b">x\ngatt\ntatg\n"
    assert H.read_input("tcaggatt", fasta=False) == b"tcaggatt"
    with pytest.raises(H.HarnessError) as e:
        H.read_input(str(tmp_path / "missing.fa"), fasta=True)
    assert e.value.code == H.EXIT_IO


def test_parse_sizes():
    assert H.parse_sizes("2,4") == [2, 4]
    assert H.parse_sizes("2..8192x2") == [2 ** k for k in range(1, 14)]
    assert H.parse_sizes("3..30x3") == [3, 9, 27]
    assert H.parse_sizes("0,5") == [0, 5]
    for bad in ("", "4..2", "0..8", "2..8x1", "-3"):
        with pytest.raises((H.HarnessError, ValueError)):
            H.parse_sizes(bad)


def test_instance_is_pure():
    a1, b1 = H.instance(7, 10, 20, 1, 4)
    a2, b2 = H.instance(7, 10, 20, 1, 4)
    assert (a1, b1) == (a2, b2) and len(a1) == 10 and len(b1) == 20
    assert set(a1) <= set(b"abcd")
    assert H.instance(7, 10, 20, 2, 4) != (a1, b1)
    a3, _ = H.instance(1, 50, 0, 0, 200)
    assert max(a3) < 200


def test_fit_log_linear_known_answers():
    xs = [1.0, 2.0, 3.0, 4.0, 5.0]
    a, b, r2 = H.fit_log_linear(xs, [2 * math.exp(0.5 * x) for x in xs])
    assert a == pytest.approx(2.0) and b == pytest.approx(0.5) and r2 == pytest.approx(1.0)
    a, b, r2 = H.fit_log_linear(xs, [3.0] * 5)
    assert b == pytest.approx(0.0, abs=1e-12) and a == pytest.approx(3.0)
    with pytest.raises(H.HarnessError):
        H.fit_log_linear([2, 2, 2], [1, 2, 3])
    with pytest.raises(H.HarnessError):
        H.fit_log_linear([1, 2], [1, 2])


def _stub_solve(a, b, threads=1, low_memory=False):
    # host-side stand-in for the CUDA solve (harness logic only)
    return LcsResult(min(len(a), len(b)), b"", (), ())


def test_bench_records_and_csv_schema():
    recs = list(H.bench_records([2, 4], [2, 8], [1, 3], 2, 0, 4, solve=_stub_solve))
    # (threads) x (fixed x sweep, both roles) x reps
    assert len(recs) == 2 * (2 * 2 * 2) * 2
    assert {(r[1], r[2]) for r in recs} == {(2, 2), (2, 8), (4, 2), (4, 8), (8, 2), (2, 4), (8, 4)}
    buf = io.StringIO()
    H.write_csv(recs, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0].startswith("# prng:")
    assert lines[1] == "threads,size_a,size_b,rep,wall_seconds,lcs_length"
    assert len(lines) == 2 + len(recs)
    t, sa, sb, rep, sec, ln = lines[2].split(",")
    assert float(sec) >= 0 and "." in sec and int(ln) == min(int(sa), int(sb))
    with pytest.raises(H.HarnessError):
        list(H.bench_records([2], [2], [1], 0, 0, 4, solve=_stub_solve))


def test_cli_usage_errors():
    assert H.main([]) == H.EXIT_USAGE
    assert H.main(["nope"]) == H.EXIT_USAGE
    assert H.main(["bench", "--sweep", "4..2", "--csv", "/dev/null"]) == H.EXIT_USAGE
    assert H.main(["bench", "--alphabet", "1"]) == H.EXIT_USAGE
    assert H.main(["lcs", "/nonexistent/a.fa", "x", "--fasta"]) == H.EXIT_IO


@pytest.mark.gpu
def test_cli_lcs_inline_and_fasta(tmp_path):
    out = io.StringIO()
    assert H.main(["lcs", "gatttatgcagg", "tcaggatt"], out=out) == H.EXIT_OK
    text = out.getvalue()
    assert "length: 5" in text
    fa, fb = tmp_path / "a.fa", tmp_path / "b.fa"
    fa.write_bytes(b">a\ngattt\natgcagg\n")
    fb.write_bytes(b">b\ntcagg\natt\n")
    out2 = io.StringIO()
    assert H.main(["lcs", str(fa), str(fb), "--fasta"], out=out2) == H.EXIT_OK
    assert out2.getvalue() == text  # ingestion equivalence
    empty = tmp_path / "e.txt"
    empty.write_bytes(b"")
    out3 = io.StringIO()
    assert H.main(["lcs", str(empty), "abc"], out=out3) == H.EXIT_OK
    assert "length: 0" in out3.getvalue()


@pytest.mark.gpu
def test_cli_selftest_and_bench(tmp_path):
    out = io.StringIO()
    assert H.main(["selftest", "--max-len", "3", "--fuzz", "40"], out=out) == H.EXIT_OK
    assert "0 failures" in out.getvalue()
    csv_path = tmp_path / "b.csv"
    assert H.main(["bench", "--fixed", "2", "--sweep", "2..16x2", "--reps", "2",
                   "--csv", str(csv_path)]) == H.EXIT_OK
    rows = [l.split(",") for l in csv_path.read_text().splitlines()[2:]]
    assert len(rows) == 2 * 4 * 2
    # deterministic instances: same seed, same lengths
    csv2 = tmp_path / "c.csv"
    H.main(["bench", "--fixed", "2", "--sweep", "2..16x2", "--reps", "2", "--csv", str(csv2)])
    rows2 = [l.split(",") for l in csv2.read_text().splitlines()[2:]]
    assert [r[5] for r in rows] == [r[5] for r in rows2]
    for r in rows:
        a, b = H.instance(0, int(r[1]), int(r[2]), int(r[3]), 4)
        from paper_2309_09072_b200 import dp_lcs

        assert int(r[5]) == dp_lcs(a, b).length
