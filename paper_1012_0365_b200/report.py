"""Report rows and tables (bench/report.hpp:14-154 restated): the reference's
CSV (RFC 4180) / pipe-table schema, so GPU rows sit beside CPU rows.

RPCA rows: m, method, rel_err, rank_hat, e_l0, iters, time_s, matvecs.
MC rows:   m, r, s_dr, s_m2, algorithm, time_s, iters, rel_err, matvecs.
A trailing `flag` column only if some row did not converge; a
`speedup=<baseline/blws>` line when the batch is exactly one baseline /
BLWS pair of the same scenario. Byte-stable for identical inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

RPCA, MC = "rpca", "mc"


@dataclass
class ReportRow:
    problem: str = RPCA
    m: int = 0
    method: str = ""  # "ADM", "BLWS-ADM", "SVT", "BLWS-SVT"
    rel_err: float = -1.0
    rank_hat: int = 0
    e_l0: int = 0
    iters: int = 0
    time_s: float = 0.0
    matvecs: int = 0
    r: int = 0  # MC only
    s_dr: float = 0.0
    s_m2: float = 0.0
    converged: bool = True


def _sci3(v):
    return "%.2e" % v


def _fixed2(v):
    return "%.2f" % v


def _general(v):
    return "%g" % v


def csv_escape(s: str) -> str:
    if not any(c in s for c in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def _cells(row: ReportRow, with_flag: bool):
    if row.problem == RPCA:
        cells = [str(row.m), row.method, _sci3(row.rel_err), str(row.rank_hat), str(row.e_l0), str(row.iters),
                 _fixed2(row.time_s), str(row.matvecs)]
    else:
        cells = [str(row.m), str(row.r), _general(row.s_dr), _general(row.s_m2), row.method, _fixed2(row.time_s),
                 str(row.iters), _sci3(row.rel_err), str(row.matvecs)]
    if with_flag:
        cells.append("" if row.converged else "nonconverged")
    return cells


def _header(problem: str, with_flag: bool):
    if problem == RPCA:
        cells = ["m", "method", "rel_err", "rank_hat", "e_l0", "iters", "time_s", "matvecs"]
    else:
        cells = ["m", "r", "s_dr", "s_m2", "algorithm", "time_s", "iters", "rel_err", "matvecs"]
    if with_flag:
        cells.append("flag")
    return cells


def speedup_line(rows) -> str:
    if len(rows) != 2:
        return ""
    a, b = rows
    if a.problem != b.problem or a.m != b.m or a.r != b.r:
        return ""
    a_blws, b_blws = "BLWS" in a.method, "BLWS" in b.method
    if a_blws == b_blws:
        return ""
    base, warm = (b, a) if a_blws else (a, b)
    if warm.time_s <= 0:
        return ""
    return "speedup=" + _fixed2(base.time_s / warm.time_s)


def emit_table(rows, fmt: str = "csv") -> str:
    """`fmt`: "csv" or "markdown"."""
    if not rows:
        raise ValueError("emit_table: no rows")
    kind = rows[0].problem
    if any(r.problem != kind for r in rows):
        raise ValueError("emit_table: mixed row schemas")
    with_flag = any(not r.converged for r in rows)
    header = _header(kind, with_flag)
    out = []
    if fmt == "csv":
        out.append(",".join(csv_escape(c) for c in header))
        out += [",".join(csv_escape(c) for c in _cells(r, with_flag)) for r in rows]
    else:
        out.append("|" + "".join(f" {c} |" for c in header))
        out.append("|" + " --- |" * len(header))
        out += ["|" + "".join(f" {c} |" for c in _cells(r, with_flag)) for r in rows]
    text = "\n".join(out) + "\n"
    sp = speedup_line(rows)
    return text + (sp + "\n" if sp else "")
