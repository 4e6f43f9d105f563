"""Record output (include/scalarmc/io.hpp, src/io.cpp): CSV with a header row
or JSON lines, every number in the shortest "%.{p}g" text that round-trips
(format_double, io.cpp:15-26) — the files the reference CLI writes."""
from __future__ import annotations

import math
from typing import IO, Sequence


def parse_record_format(name: str) -> str:
    if name in ("csv", "jsonl"):
        return name
    raise ValueError("unknown record format: " + name)


def format_double(v: float) -> str:
    """Shortest %.{1..17}g representation that parses back to v."""
    v = float(v)
    if math.isnan(v):
        return "nan"
    s = ""
    for prec in range(1, 18):
        s = "%.*g" % (prec, v)
        if float(s) == v:
            return s
    return s


class RecordWriter:
    """io.cpp:28-57: header at construction (CSV), one line per row."""

    def __init__(self, out: IO[str], fmt: str, columns: Sequence[str]):
        self.out, self.fmt, self.columns = out, parse_record_format(fmt), list(columns)
        if self.fmt == "csv":
            out.write(",".join(self.columns) + "\n")

    def write_row(self, values: Sequence[float]) -> None:
        if len(values) != len(self.columns):
            raise ValueError("RecordWriter: column count mismatch")
        if self.fmt == "csv":
            self.out.write(",".join(format_double(v) for v in values) + "\n")
        else:
            self.out.write("{" + ",".join(f'"{c}":{format_double(v)}' for c, v in zip(self.columns, values)) + "}\n")
