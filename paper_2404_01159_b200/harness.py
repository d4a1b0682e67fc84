"""Output formats of the reference's harness (so that files written here drop into its tooling).

reference: io.hpp:18-76 (fmt %.17g, ConfigEcho, CsvWriter with the `# version=` / `# config:` header lines, median,
iqr), version.hpp:5, and the `scale` sub-command's CSV (temo.cpp:229-282: median per-generation duration from the
cumulative elapsed_ms column, columns series,n,d,m,generations,tensor_ms,oracle_ms,speedup,status)."""
from __future__ import annotations

import math
import os

VERSION = "0.1.0"  # version.hpp:5: files carry the reference's format version
SCALE_COLUMNS = ["series", "n", "d", "m", "generations", "tensor_ms", "oracle_ms", "speedup", "status"]  # temo.cpp:244-246


def fmt(v) -> str:
    """io.hpp:18-24: doubles with %.17g (identical doubles give identical bytes), sizes as integers."""
    if isinstance(v, (int,)) and not isinstance(v, bool):
        return str(v)
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def config_line(cfg: dict) -> str:
    """io.hpp:29-36: `key=value` pairs in key order (ConfigEcho is a std::map)."""
    return " ".join(f"{k}={cfg[k]}" for k in sorted(cfg))


class CsvWriter:
    """io.hpp:38-59."""

    def __init__(self, path, cfg: dict, columns):
        try:
            self._fh = open(os.fspath(path), "w", newline="")
        except OSError as e:
            raise RuntimeError(f"cannot open output file: {path}") from e
        self._fh.write(f"# version={VERSION}\n")
        self._fh.write(f"# config: {config_line(cfg)}\n")
        self._fh.write(",".join(columns) + "\n")

    def row(self, cells) -> None:
        self._fh.write(",".join(str(c) for c in cells) + "\n")

    def close(self) -> None:
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def median(values) -> float:
    """io.hpp:61-66."""
    v = sorted(float(x) for x in values)
    n = len(v)
    if n == 0:
        return float("nan")
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def iqr(values) -> float:
    """io.hpp:69-76: quartiles at the medians of the two halves."""
    v = sorted(float(x) for x in values)
    n = len(v)
    if n < 2:
        return 0.0
    return median(v[(n + 1) // 2:]) - median(v[: n // 2])


def median_generation_ms(elapsed_ms) -> float:
    """temo.cpp:229-237: median of the successive differences of the cumulative elapsed_ms column."""
    prev, durations = 0.0, []
    for e in elapsed_ms:
        durations.append(float(e) - prev)
        prev = float(e)
    return median(durations)


def scale_csv(path, echo: dict) -> CsvWriter:
    """The `scale` sub-command's file (temo.cpp:239-246)."""
    return CsvWriter(path, echo, SCALE_COLUMNS)


def scale_row(series: str, n: int, d: int, m: int, generations: int, tensor_ms: float, oracle_ms: float, status: str = "ok"):
    """One row of scale.csv (temo.cpp:271-276): speedup = oracle_ms / tensor_ms (0 when tensor_ms is 0)."""
    speedup = oracle_ms / tensor_ms if tensor_ms > 0.0 else 0.0
    return [series, fmt(int(n)), fmt(int(d)), fmt(int(m)), fmt(int(generations)), fmt(float(tensor_ms)), fmt(float(oracle_ms)),
            fmt(float(speedup)), status]
