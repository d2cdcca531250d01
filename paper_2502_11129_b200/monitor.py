"""Measurement helpers — mirror of /root/reference/proj/src/monitor.cpp.

* ``summarize``: mean, sample stddev, Student-t CI95, interpolated p95
  (monitor.cpp:76-105).
* ``detect_saturation_knee``: largest n whose wall stays within
  (1 + eps) of the flat-prefix minimum (monitor.cpp:184-203) — applied to
  the measured B200 variant sweeps (the paper's "constant-then-linear" law).
* ``GpuUtilSampler``: the accelerator half of the reference's utilisation
  trace (``UtilizationSample.accel_percent`` is always 0 there,
  monitor.cpp:164,177): NVML GPU utilisation sampled at 20 Hz, like the
  reference's CPU sampler (monitor.cpp:157-169).
"""
from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass
from enum import Enum
from typing import Sequence


def student_t_critical_95(df: int) -> float:
    """Two-sided 95 % Student-t critical value (monitor.cpp:60-74: bisection
    on the CDF); df = 0 returns 0."""
    if df == 0:
        return 0.0
    from scipy import stats
    return float(stats.t.ppf(0.975, df))


@dataclass
class Stats:
    n: int = 0
    mean: float = 0.0
    stddev: float = 0.0
    ci95_low: float = 0.0
    ci95_high: float = 0.0
    p95: float = 0.0

    def small_sample(self) -> bool:
        return self.n < 20


def summarize(samples: Sequence[float]) -> Stats:
    """monitor.cpp:76-105."""
    if len(samples) == 0:
        raise ValueError("summarize: empty input")
    s = Stats(n=len(samples))
    total = 0.0
    for v in samples:
        total += v
    s.mean = total / s.n
    if s.n > 1:
        ss = 0.0
        for v in samples:
            ss += (v - s.mean) * (v - s.mean)
        s.stddev = math.sqrt(ss / (s.n - 1))
        half = student_t_critical_95(s.n - 1) * s.stddev / math.sqrt(s.n)
        s.ci95_low, s.ci95_high = s.mean - half, s.mean + half
    else:
        s.ci95_low = s.ci95_high = s.mean
    srt = sorted(samples)
    h = 0.95 * (s.n - 1)
    lo = int(h)
    hi = min(lo + 1, s.n - 1)
    s.p95 = srt[lo] + (h - lo) * (srt[hi] - srt[lo])
    return s


class KneeRegime(Enum):
    Knee = 0
    AllFlat = 1
    AllLinear = 2


def detect_saturation_knee(points: Sequence[tuple[int, float]], epsilon: float = 0.05):
    """monitor.cpp:184-203.  points = [(n_variants, wall_s)] with strictly
    increasing n.  Returns (n, KneeRegime)."""
    if len(points) < 3:
        raise ValueError("detect_saturation_knee: need at least 3 points")
    for i in range(1, len(points)):
        if points[i][0] <= points[i - 1][0]:
            raise ValueError("detect_saturation_knee: n must be strictly increasing")
    t_min = min(w for _, w in points)
    threshold = (1.0 + epsilon) * t_min
    last_flat = 0
    for i, (_, w) in enumerate(points):
        if w <= threshold:
            last_flat = i
    if last_flat == len(points) - 1:
        return points[-1][0], KneeRegime.AllFlat
    if last_flat == 0:
        return points[0][0], KneeRegime.AllLinear
    return points[last_flat][0], KneeRegime.Knee


class GpuUtilSampler:
    """NVML utilisation of one GPU at ``hz`` (default 20 Hz) between start()
    and stop(); stop() returns [(t_seconds_since_start, gpu_percent)] with a
    final synchronised sample.  Degrades to an empty trace without NVML."""

    def __init__(self, device: int = 0, hz: float = 20.0):
        self.device, self.period = device, 1.0 / hz
        self.trace: list[tuple[float, float]] = []
        self._run = False
        self._th = None
        self._h = None

    def _sample(self):
        import pynvml
        return float(pynvml.nvmlDeviceGetUtilizationRates(self._h).gpu)

    def start(self):
        self.trace = []
        self.t0 = time.perf_counter()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
        except Exception:  # noqa: BLE001 - no NVML: empty trace, like monitor.cpp:153
            self._h = None
            return
        self._run = True
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()

    def _loop(self):
        while self._run:
            time.sleep(self.period)
            if not self._run:
                break
            self.trace.append((time.perf_counter() - self.t0, self._sample()))

    def stop(self):
        if self._h is None:
            return []
        self._run = False
        if self._th is not None:
            self._th.join()
        self.trace.append((time.perf_counter() - self.t0, self._sample()))
        return self.trace
