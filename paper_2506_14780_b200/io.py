"""CSV / JSON input and output of the reference (proj/src/io.cpp, include/sknr/io.hpp).

Formats follow io.cpp: numbers are written with %.17g (bitwise round trip),
one matrix row per line, potentials as `which,index,value`, the solver trace and
anneal trace with the reference headers, spectrum reports as JSON. The coupling
writer streams row blocks from the device (`coupling_rows`) so an n x m plan is
never held whole.
"""
from __future__ import annotations

import math
import os
from typing import Optional

import numpy as np

from . import Problem, coupling_rows

_TINY = 2.2250738585072014e-308  # smallest normal double: glibc strtod reports ERANGE below it


class CsvError(RuntimeError):
    """Parse failure with a 1-based line/column position (io.hpp:13-26)."""

    def __init__(self, path: str, line: int, column: int, what: str):
        super().__init__(f"{path}:{line}:{column}: {what}")
        self.line = line
        self.column = column


def format_double(value: float) -> str:
    """%.17g: doubles round-trip bitwise through this format (io.cpp:100-104)."""
    return "%.17g" % value


def _parse_double(cell: str) -> Optional[float]:
    """strtod semantics of parse_double (io.cpp:28-36): leading blanks skipped, trailing
    blanks/tabs/CR allowed, anything else after the number or an out-of-range value
    rejects the cell."""
    body = cell.rstrip(" \t\r")
    s = body.lstrip(" \t\n\v\f\r")
    if not s or "_" in s:
        return None
    try:
        v = float(s)
    except ValueError:
        return None
    low = s.lower().lstrip("+-")
    literal_special = low.startswith("inf") or low.startswith("nan")
    if math.isinf(v) and not literal_special:
        return None  # overflow: ERANGE
    if v != 0.0 and abs(v) < _TINY:
        return None  # underflow to a subnormal: ERANGE
    if v == 0.0 and any(ch in "123456789" for ch in s.split("e")[0].split("E")[0]):
        return None  # nonzero literal underflowed to zero: ERANGE
    return v


def _split_line(line: str):
    cells = line.split(",")
    return cells


def _read_numeric_csv(path: str):
    """(header, rows) per read_numeric_csv (io.cpp:43-83)."""
    try:
        fh = open(path, "r", newline="")
    except OSError:
        raise CsvError(path, 0, 0, "cannot open file") from None
    header: list = []
    rows: list = []
    width = 0
    line_no = 0
    with fh:
        for raw in fh:
            line_no += 1
            line = raw[:-1] if raw.endswith("\n") else raw
            if line.endswith("\r"):
                line = line[:-1]
            if not line:
                continue
            cells = _split_line(line)
            row = []
            numeric = True
            for c, cell in enumerate(cells):
                v = _parse_double(cell)
                if v is None:
                    if not rows and line_no == 1:
                        header = cells
                        numeric = False
                        break
                    raise CsvError(path, line_no, c + 1, f"not a number: '{cell}'")
                if not math.isfinite(v):
                    raise CsvError(path, line_no, c + 1, "non-finite value rejected")
                row.append(v)
            if not numeric:
                continue
            if width == 0:
                width = len(row)
            if len(row) != width:
                raise CsvError(path, line_no, len(row), "inconsistent column count")
            rows.append(row)
    if not rows:
        raise CsvError(path, line_no, 0, "no data rows")
    return header, rows


def read_csv_matrix(path: str) -> np.ndarray:
    """Numeric CSV -> column-major matrix (io.cpp:106-108)."""
    _, rows = _read_numeric_csv(path)
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def read_csv_vector(path: str) -> np.ndarray:
    """A single row or column (io.cpp:153-158)."""
    m = read_csv_matrix(path)
    if m.shape[1] == 1:
        return m[:, 0].copy()
    if m.shape[0] == 1:
        return m[0, :].copy()
    raise CsvError(path, 1, 1, "expected a single row or column")


def read_point_cloud(path: str):
    """(points n x d col-major, weights, renormalized) (io.cpp:121-151): a final column
    is a weight column only when the header's last field is `weight`."""
    header, rows = _read_numeric_csv(path)
    raw = np.array(rows, dtype=np.float64)
    has_weights = bool(header) and header[-1] == "weight"
    if raw.shape[1] < (2 if has_weights else 1):
        raise CsvError(path, 1, 1, "point cloud needs at least one coordinate column")
    renormalized = False
    if has_weights:
        pts = raw[:, :-1]
        w = raw[:, -1].copy()
        for i in range(w.size):
            if not w[i] > 0.0:
                raise CsvError(path, i + 2, raw.shape[1], "weights must be strictly positive")
        total = float(np.sum(w))
        if abs(total - 1.0) > 1e-9:
            w /= total
            renormalized = True
    else:
        pts = raw
        w = np.full(raw.shape[0], 1.0 / raw.shape[0])
    return np.asfortranarray(pts), w, renormalized


def write_csv_matrix(path: str, matrix) -> None:
    """One row per line, %.17g, comma separated (io.cpp:110-119)."""
    matrix = np.asarray(matrix, dtype=np.float64)
    with open(path, "w") as out:
        for i in range(matrix.shape[0]):
            out.write(",".join(format_double(v) for v in matrix[i]) + "\n")


def write_csv_vector(path: str, v, header: str = "") -> None:
    with open(path, "w") as out:
        if header:
            out.write(header + "\n")
        for x in np.asarray(v, dtype=np.float64):
            out.write(format_double(x) + "\n")


def write_potentials_csv(path: str, f, g) -> None:
    """`which,index,value` rows, f then g (io.cpp:167-175)."""
    with open(path, "w") as out:
        out.write("which,index,value\n")
        for i, v in enumerate(np.asarray(f, dtype=np.float64)):
            out.write(f"f,{i},{format_double(v)}\n")
        for j, v in enumerate(np.asarray(g, dtype=np.float64)):
            out.write(f"g,{j},{format_double(v)}\n")


def write_trace_csv(path: str, trace) -> None:
    """Solver trace with the reference header (io.cpp:177-190)."""
    with open(path, "w") as out:
        out.write("iter,marginal_error,marginal_error_inf,semi_dual_value,"
                  "newton_attempted,newton_accepted,time_ms\n")
        for r in trace:
            out.write(f"{r.index},{format_double(r.marginal_error)},{format_double(r.marginal_error_inf)},"
                      f"{format_double(r.semi_dual_value)},{1 if r.newton_attempted else 0},"
                      f"{1 if r.newton_accepted else 0},{format_double(r.wall_time_ms)}\n")


def write_anneal_csv(path: str, epsilons, stages) -> None:
    """Combined anneal trace (io.cpp:192-207)."""
    with open(path, "w") as out:
        out.write("stage,epsilon,iter,marginal_error,semi_dual_value,newton_accepted,time_ms\n")
        for s, st in enumerate(stages):
            for r in st.trace:
                out.write(f"{s},{format_double(epsilons[s])},{r.index},{format_double(r.marginal_error)},"
                          f"{format_double(r.semi_dual_value)},{1 if r.newton_accepted else 0},"
                          f"{format_double(r.wall_time_ms)}\n")


def spectrum_report_to_json(report: dict, k: int) -> str:
    """JSON text of a spectrum report, floats at 17 significant digits (io.cpp:238-276)."""
    lines = ["{", f'  "epsilon": {format_double(report["epsilon"])},', f'  "k": {k},']
    with_vectors = report.get("vectors_f") is not None

    def arr(name, v, trailing):
        body = ", ".join(format_double(x) for x in np.asarray(v, dtype=np.float64))
        return f'  "{name}": [{body}]' + ("," if trailing else "")

    def mat(name, m, trailing):
        m = np.asarray(m, dtype=np.float64)
        cols = ", ".join("[" + ", ".join(format_double(x) for x in m[:, c]) + "]" for c in range(m.shape[1]))
        return f'  "{name}": [{cols}]' + ("," if trailing else "")

    lines.append(arr("rho", report["rho"], True))
    lines.append(arr("hessian_eigs_low", report["hessian_eigs_low"], with_vectors))
    if with_vectors:
        lines.append(mat("vectors_f", report["vectors_f"], True))
        lines.append(mat("vectors_g", report["vectors_g"], False))
    lines.append("}")
    return "\n".join(lines) + "\n"


def write_spectrum_json(path: str, report: dict, k: int) -> None:
    with open(path, "w") as out:
        out.write(spectrum_report_to_json(report, k))


def write_coupling_csv(path: str, problem: Problem, f, g, block_bytes: int = 1 << 28) -> float:
    """coupling.csv (main.cpp:149-154) streamed from the device in row blocks; returns
    marginal_error(problem, coupling) (core.cpp:105-112) from the same blocks."""
    n, m = problem.n, problem.m
    rows_per_block = max(1, int(block_bytes // (8 * max(m, 1))))
    row_sums = np.empty(n)
    col_sums = np.zeros(m)
    with open(path, "w") as out:
        for r0 in range(0, n, rows_per_block):
            r1 = min(n, r0 + rows_per_block)
            block = coupling_rows(problem, f, g, r0, r1)
            row_sums[r0:r1] = block.sum(axis=1)
            col_sums += block.sum(axis=0)
            for i in range(block.shape[0]):
                out.write(",".join(format_double(v) for v in block[i]) + "\n")
    return float(np.linalg.norm(row_sums - problem.alpha) + np.linalg.norm(col_sums - problem.beta))


__all__ = ["CsvError", "format_double", "read_csv_matrix", "read_csv_vector", "read_point_cloud",
           "spectrum_report_to_json", "write_anneal_csv", "write_coupling_csv", "write_csv_matrix",
           "write_csv_vector", "write_potentials_csv", "write_spectrum_json", "write_trace_csv"]
