"""Host-side records around the hot path:

* solution.bin — six little-endian int64 words (nx, ny, nz, 0, 0, 0), then
  p,u,v,w,T as little-endian doubles over the global interior, i-fastest
  (write_solution / read_solution, /root/reference/proj/src/dump.cpp:51-83).
* RunRecord CSV — `np,mode,dims,strategy,overlap,size,steps,wall_time_s,
  ssspnt,speedup,efficiency,bytes_sent` (src/metrics.cpp:30-89), plus
  ScalingSeries.validate (src/metrics.cpp:115-138) and speedup_efficiency.
"""
import io
import math
import struct
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _abi as A
from .capi import InvalidArgument, ssspnt

CSV_HEADER = ("np,mode,dims,strategy,overlap,size,steps,wall_time_s,ssspnt,speedup,efficiency,"
              "bytes_sent")


def write_solution(path, fields):
    """fields: array (5, nz, ny, nx) of p,u,v,w,T."""
    f = np.asarray(fields, dtype="<f8")
    if f.ndim != 4 or f.shape[0] != 5:
        raise InvalidArgument("solution dump: field size mismatch")
    nz, ny, nx = f.shape[1:]
    with open(path, "wb") as fh:
        fh.write(struct.pack("<6q", nx, ny, nz, 0, 0, 0))
        fh.write(np.ascontiguousarray(f).tobytes())


def read_solution(path):
    with open(path, "rb") as fh:
        head = fh.read(48)
        if len(head) < 48:
            raise RuntimeError("solution file: truncated header")
        nx, ny, nz = struct.unpack("<6q", head)[:3]
        if nx <= 0 or ny <= 0 or nz <= 0:
            raise RuntimeError("solution file: bad grid size in header")
        n = nx * ny * nz
        data = fh.read(5 * n * 8)
        if len(data) < 5 * n * 8:
            raise RuntimeError("solution file: truncated variable payload")
    return np.frombuffer(data, dtype="<f8").reshape(5, nz, ny, nx).astype(np.float64)


def speedup_efficiency(t_serial, t_parallel, np_):
    if not t_serial > 0.0 or not t_parallel > 0.0:
        raise InvalidArgument("speedup: times must be positive")
    if np_ <= 0:
        raise InvalidArgument("speedup: np must be positive")
    s = t_serial / t_parallel
    return s, s / np_


def _g9(v):
    if isinstance(v, float) and math.isnan(v):
        return "nan"
    return "%.9g" % v


@dataclass
class RunRecord:
    np: int = 1
    mode: str = "3d"
    dims: str = "1x1x1"
    strategy: str = "v3"
    overlap: int = 0
    size: int = 0
    steps: int = 0
    wall_time_s: float = 0.0
    ssspnt: float = 0.0
    speedup: float = 0.0
    efficiency: float = 0.0
    bytes_sent: int = 0

    def csv_row(self):
        return ",".join([str(self.np), self.mode, self.dims, self.strategy, str(self.overlap),
                         str(self.size), str(self.steps), _g9(self.wall_time_s), _g9(self.ssspnt),
                         _g9(self.speedup), _g9(self.efficiency), str(self.bytes_sent)])

    @classmethod
    def from_result(cls, cfg, res):
        """RunRecord of a CaseResult (src/runner.cpp:317-336)."""
        size = cfg.nx * cfg.ny * cfg.nz
        return cls(np=res.np, mode=A.MODE_NAMES[cfg.mode],
                   dims="%dx%dx%d" % tuple(res.dims), strategy=A.STRATEGY_NAMES[cfg.strategy],
                   overlap=int(bool(cfg.overlap)), size=size, steps=res.steps_timed,
                   wall_time_s=res.wall_time_s,
                   ssspnt=(ssspnt(size, res.steps_timed, res.np, res.wall_time_s)
                           if res.steps_timed > 0 and res.wall_time_s > 0 else float("nan")),
                   speedup=float("nan"), efficiency=float("nan"), bytes_sent=res.bytes_sent)


def csv_text(rows):
    out = io.StringIO()
    out.write(CSV_HEADER + "\n")
    for r in rows:
        out.write(r.csv_row() + "\n")
    return out.getvalue()


def parse_csv(text):
    lines = text.splitlines()
    if not lines:
        raise RuntimeError("csv: empty input")
    if lines[0] != CSV_HEADER:
        raise RuntimeError("csv: unexpected header: " + lines[0])
    rows = []
    for line in lines[1:]:
        if not line:
            continue
        c = line.split(",")
        if len(c) != 12:
            raise RuntimeError("csv: bad row: " + line)
        rows.append(RunRecord(int(c[0]), c[1], c[2], c[3], int(c[4]), int(c[5]), int(c[6]),
                              float(c[7]), float(c[8]), float(c[9]), float(c[10]), int(c[11])))
    return rows


@dataclass
class ScalingSeries:
    label: str = ""
    scaling: str = "strong"
    rows: List[RunRecord] = field(default_factory=list)

    def validate(self):
        if not self.rows:
            return
        if self.scaling not in ("strong", "weak"):
            raise InvalidArgument("series: scaling must be strong or weak")
        base = min(self.rows, key=lambda r: r.np)
        for r in self.rows:
            if r.np <= 0:
                raise InvalidArgument("series: np must be positive")
            if self.scaling == "strong" and r.size != base.size:
                raise InvalidArgument("series: strong scaling must keep the global size fixed")
            if self.scaling == "weak" and r.size * base.np != base.size * r.np:
                raise InvalidArgument("series: weak scaling must grow size in proportion to np")

    def fill_speedups(self):
        """speedup/efficiency against the np=1 row (src/bench.cpp:51-61)."""
        serial = [r for r in self.rows if r.np == 1]
        if not serial:
            return
        s = serial[0]
        for r in self.rows:
            if self.scaling == "strong":
                r.speedup, r.efficiency = speedup_efficiency(s.wall_time_s, r.wall_time_s, r.np)
            else:
                r.efficiency = r.ssspnt / s.ssspnt
                r.speedup = r.efficiency * r.np
