"""Command-line harness: ``lcs``, ``bench`` and ``selftest`` (SURVEY.md 8(f)
rank 3; the reference specifies it in SPEC.md "harness" but ships no code).

    python -m paper_2309_09072_b200 lcs gatttatgcagg tcaggatt
    python -m paper_2309_09072_b200 lcs a.fa b.fa --fasta
    python -m paper_2309_09072_b200 bench --fixed 2,4 --sweep 2..8192x2 --reps 3 --csv out.csv
    python -m paper_2309_09072_b200 selftest

Every solve goes through the package's public ``lcs()`` (the CUDA path); the
harness itself is single-threaded host code.  ``--threads`` is accepted for
parity with the reference CLI and recorded in the CSV; it does not change the
device solve.  Exit codes: 0 success, 1 usage error, 2 I/O error, 3 selftest
failure.
"""

from __future__ import annotations

import argparse
import csv
import math
import os
import sys
import time
from typing import Iterable, Iterator, List, Optional, Sequence, Tuple

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_SELFTEST = 0, 1, 2, 3
CSV_HEADER = ("threads", "size_a", "size_b", "rep", "wall_seconds", "lcs_length")
PRNG_NOTE = "# prng: numpy PCG64 (default_rng), seed = hash of (seed, size_a, size_b, rep, alphabet)"


class HarnessError(Exception):
    """An error with a CLI exit code."""

    def __init__(self, message: str, code: int):
        super().__init__(message)
        self.code = code


# ---------------------------------------------------------------- ingestion
def parse_fasta(data: bytes) -> bytes:
    """Sequence of the first FASTA record: header lines ('>') skipped, line
    breaks stripped; a file without any record is an error."""
    lines = data.splitlines()
    seq: List[bytes] = []
    seen = False
    for ln in lines:
        if ln.startswith(b">"):
            if seen:
                break
            seen = True
            continue
        if seen:
            seq.append(ln.strip())
    if not seen:
        raise HarnessError("FASTA input has no record", EXIT_IO)
    return b"".join(seq)


def read_input(arg: str, fasta: bool) -> bytes:
    """A path (read as raw bytes, or FASTA with --fasta) or an inline string."""
    if os.path.exists(arg):
        try:
            with open(arg, "rb") as f:
                data = f.read()
        except OSError as e:
            raise HarnessError(f"cannot read {arg}: {e}", EXIT_IO) from e
        return parse_fasta(data) if fasta else data
    if fasta:
        raise HarnessError(f"cannot read {arg}: no such file", EXIT_IO)
    return arg.encode()


# ---------------------------------------------------------- instance generation
def parse_sizes(spec: str) -> List[int]:
    """'2,4,8' or a geometric range 'a..bxf' (a, a*f, ... <= b)."""
    out: List[int] = []
    for part in spec.split(","):
        part = part.strip()
        if not part:
            continue
        if ".." in part:
            lo, rest = part.split("..", 1)
            hi, _, f = rest.partition("x")
            lo_i, hi_i, f_i = int(lo), int(hi), int(f or 2)
            if lo_i < 0 or hi_i < lo_i or f_i < 2 or lo_i == 0:
                raise HarnessError(f"bad size range {part!r}", EXIT_USAGE)
            v = lo_i
            while v <= hi_i:
                out.append(v)
                v *= f_i
        else:
            v = int(part)
            if v < 0:
                raise HarnessError(f"negative size {part!r}", EXIT_USAGE)
            out.append(v)
    if not out:
        raise HarnessError(f"empty size list {spec!r}", EXIT_USAGE)
    return out


def instance(seed: int, size_a: int, size_b: int, rep: int, alphabet: int) -> Tuple[bytes, bytes]:
    """Seeded random pair: a pure function of (seed, sizes, rep, alphabet)."""
    ss = np.random.SeedSequence([seed & (2**63 - 1), size_a, size_b, rep, alphabet])
    rng = np.random.default_rng(ss)
    a = rng.integers(0, alphabet, size_a, dtype=np.uint8) + 97 * (alphabet <= 26)
    b = rng.integers(0, alphabet, size_b, dtype=np.uint8) + 97 * (alphabet <= 26)
    return a.astype(np.uint8).tobytes(), b.astype(np.uint8).tobytes()


# ---------------------------------------------------------------- bench
def bench_records(fixed: Sequence[int], sweep: Sequence[int], threads: Sequence[int], reps: int,
                  seed: int, alphabet: int, low_memory: bool = False,
                  solve=None) -> Iterator[Tuple[int, int, int, int, float, int]]:
    """One record per (threads, size_a in fixed, size_b in sweep, rep), plus
    the transposed roles (size_a in sweep, size_b in fixed).  Times the
    solver call only (monotonic clock); inputs are generated outside."""
    if solve is None:
        from .solver import lcs as solve  # noqa: PLC0415  (CUDA path)
    if reps < 1:
        raise HarnessError("--reps must be >= 1", EXIT_USAGE)
    cells = [(fa, sb) for fa in fixed for sb in sweep] + [(sb, fa) for fa in fixed for sb in sweep]
    solve(b"ab", b"ba")  # untimed warm-up: library load and device context creation
    for t in threads:
        for sa, sb in cells:
            for rep in range(reps):
                a, b = instance(seed, sa, sb, rep, alphabet)
                t0 = time.perf_counter()
                r = solve(a, b, threads=t, low_memory=low_memory)
                dt = time.perf_counter() - t0
                yield (t, sa, sb, rep, dt, r.length)


def write_csv(records: Iterable[Tuple], out) -> None:
    out.write(PRNG_NOTE + "\n")
    w = csv.writer(out, lineterminator="\n")
    w.writerow(CSV_HEADER)
    for rec in records:
        t, sa, sb, rep, dt, ln = rec
        w.writerow((t, sa, sb, rep, f"{dt:.9f}", ln))
        out.flush()


def fit_log_linear(sizes: Sequence[float], seconds: Sequence[float]) -> Tuple[float, float, float]:
    """Least-squares fit of ln(time) = ln(a) + b*size: (a, b, r2) of
    time = a * exp(b * size) (SPEC fitLogLinear; for inspection only)."""
    xs = np.asarray(sizes, dtype=np.float64)
    ts = np.asarray(seconds, dtype=np.float64)
    if xs.size < 3 or np.any(ts <= 0):
        raise HarnessError("fit needs >= 3 records with positive times", EXIT_USAGE)
    if np.all(xs == xs[0]):
        raise HarnessError("fit needs at least two distinct sizes", EXIT_USAGE)
    ys = np.log(ts)
    b, ln_a = np.polyfit(xs, ys, 1)
    pred = ln_a + b * xs
    ss_res = float(np.sum((ys - pred) ** 2))
    ss_tot = float(np.sum((ys - ys.mean()) ** 2))
    r2 = 1.0 if ss_tot == 0 else 1.0 - ss_res / ss_tot
    return float(math.exp(ln_a)), float(b), r2


# ---------------------------------------------------------------- selftest
def selftest(max_len: int = 4, fuzz: int = 200, seed: int = 0, out=sys.stdout) -> List[str]:
    """Paper example, exhaustive small-alphabet sweep and fuzz, each checked
    against the package's DP (length, validity of the subsequence and
    positions) and for orientation symmetry of the length.  Returns the list
    of failures (empty = pass)."""
    import itertools

    from .dp import dp_lcs
    from .solver import lcs

    failures: List[str] = []

    def check(a: bytes, b: bytes, tag: str) -> None:
        r = lcs(a, b)
        try:
            r.validate(a, b)
        except (AssertionError, ValueError) as e:
            failures.append(f"{tag}: invalid result for {a!r}, {b!r}: {e}")
            return
        d = dp_lcs(a, b).length
        if r.length != d:
            failures.append(f"{tag}: length {r.length} != DP {d} for {a!r}, {b!r}")
        if lcs(b, a).length != r.length:
            failures.append(f"{tag}: length not symmetric for {a!r}, {b!r}")

    r = lcs(b"gatttatgcagg", b"tcaggatt")
    if r.length != 5:
        failures.append(f"paper example: length {r.length} != 5")
    check(b"gatttatgcagg", b"tcaggatt", "paper")
    check(b"", b"abc", "empty")
    words = [b""] + [bytes(p) for n in range(1, max_len + 1) for p in itertools.product(b"ab", repeat=n)]
    for a in words:
        for b in words:
            check(a, b, "exhaustive")
    rng = np.random.default_rng(seed)
    for i in range(fuzz):
        m, n = int(rng.integers(0, 70)), int(rng.integers(0, 140))
        sig = int(rng.choice([2, 4, 26, 200]))
        a = rng.integers(0, sig, m, dtype=np.uint8).tobytes()
        b = rng.integers(0, sig, n, dtype=np.uint8).tobytes()
        check(a, b, f"fuzz seed={seed} case={i}")
    out.write(f"selftest: {len(words) ** 2 + fuzz + 2} instances, {len(failures)} failures\n")
    for f in failures[:20]:
        out.write(f"  FAIL {f}\n")
    return failures


# ---------------------------------------------------------------- CLI
def _int_list(spec: str) -> List[int]:
    try:
        return [int(x) for x in spec.split(",") if x.strip()]
    except ValueError as e:
        raise HarnessError(f"bad integer list {spec!r}", EXIT_USAGE) from e


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2309_09072_b200",
                                description="Lu-Liu grid-graph LCS on B200 (lcsgrid drop-in)")
    sub = p.add_subparsers(dest="mode", required=True)
    pl = sub.add_parser("lcs", help="LCS of two inputs (inline strings or files)")
    pl.add_argument("a")
    pl.add_argument("b")
    pl.add_argument("--threads", type=int, default=int(os.environ.get("LCSGRID_THREADS", "1")))
    pl.add_argument("--fasta", action="store_true", help="inputs are FASTA files (first record)")
    pl.add_argument("--low-memory", action="store_true")
    pb = sub.add_parser("bench", help="CSV sweep (threads,size_a,size_b,rep,wall_seconds,lcs_length)")
    pb.add_argument("--fixed", default="2,4")
    pb.add_argument("--sweep", default="2..8192x2")
    pb.add_argument("--threads", default=os.environ.get("LCSGRID_THREADS", "1"))
    pb.add_argument("--reps", type=int, default=3)
    pb.add_argument("--seed", type=int, default=0)
    pb.add_argument("--alphabet", type=int, default=4)
    pb.add_argument("--csv", default=None, help="output path (default stdout)")
    pb.add_argument("--low-memory", action="store_true")
    pb.add_argument("--fit", action="store_true",
                    help="print time = a*exp(b*size) fits per (threads, fixed size) to stderr")
    ps = sub.add_parser("selftest", help="paper example + exhaustive + fuzz checks")
    ps.add_argument("--seed", type=int, default=0)
    ps.add_argument("--max-len", type=int, default=4)
    ps.add_argument("--fuzz", type=int, default=200)
    return p


def main(argv: Optional[Sequence[str]] = None, out=None) -> int:
    out = out or sys.stdout
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        if args.mode == "lcs":
            from .solver import lcs

            a = read_input(args.a, args.fasta)
            b = read_input(args.b, args.fasta)
            r = lcs(a, b, threads=args.threads, low_memory=args.low_memory)
            out.write(f"length: {r.length}\n")
            out.write(f"subsequence: {r.subsequence.decode('latin-1')}\n")
            out.write(f"positions_a: {' '.join(map(str, r.row_positions))}\n")
            out.write(f"positions_b: {' '.join(map(str, r.col_positions))}\n")
            return EXIT_OK
        if args.mode == "bench":
            if not 2 <= args.alphabet <= 256:
                raise HarnessError("--alphabet must be in 2..256", EXIT_USAGE)
            fixed, sweep = parse_sizes(args.fixed), parse_sizes(args.sweep)
            threads = _int_list(args.threads)
            ncpu = os.cpu_count() or 1
            for t in threads:
                if t > ncpu:
                    sys.stderr.write(f"warning: {t} threads exceed the {ncpu} host CPUs\n")
            recs = bench_records(fixed, sweep, threads, args.reps, args.seed, args.alphabet,
                                 args.low_memory)
            collected: List[Tuple] = []

            def tee(it):
                for rec in it:
                    collected.append(rec)
                    yield rec

            if args.csv:
                try:
                    with open(args.csv, "w", newline="") as f:
                        write_csv(tee(recs), f)
                except OSError as e:
                    raise HarnessError(f"cannot write {args.csv}: {e}", EXIT_IO) from e
            else:
                write_csv(tee(recs), out)
            if args.fit:
                for t in threads:
                    for fa in fixed:
                        grp = [r for r in collected if r[0] == t and r[1] == fa]
                        try:
                            a_, b_, r2 = fit_log_linear([r[2] for r in grp], [r[4] for r in grp])
                            sys.stderr.write(f"fit threads={t} size_a={fa}: time = {a_:.3e} * "
                                             f"exp({b_:.4g} * size_b), R2 = {r2:.4f}\n")
                        except HarnessError as e:
                            sys.stderr.write(f"fit threads={t} size_a={fa}: error: {e}\n")
            return EXIT_OK
        if args.mode == "selftest":
            fails = selftest(args.max_len, args.fuzz, args.seed, out)
            return EXIT_SELFTEST if fails else EXIT_OK
    except HarnessError as e:
        sys.stderr.write(f"error: {e}\n")
        return e.code
    return EXIT_USAGE
