"""SM-clock / throttle-reason sampling during a timed region (NVML, the
library behind ``nvidia-smi``), for the bench's ``clocks`` record."""

from __future__ import annotations

import statistics
import threading
import time

_REASONS = (
    ("gpu_idle", "nvmlClocksEventReasonGpuIdle"),
    ("applications_clocks_setting", "nvmlClocksEventReasonApplicationsClocksSetting"),
    ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
    ("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
    ("sync_boost", "nvmlClocksEventReasonSyncBoost"),
    ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
    ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
    ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"),
)

REJECTING = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


class ClockSampler:
    """Background NVML sampler: ``with ClockSampler(idx) as s: ...`` then
    ``s.summary()``. Degrades to ``{"available": False}`` without NVML."""

    def __init__(self, device_index: int, period_s: float = 0.01):
        self.idx = device_index
        self.period = period_s
        self.samples: list[tuple[int, int, int, float]] = []
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        self._handle = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._handle = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(
                self._handle, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - telemetry is best effort
            self._nvml = None
            return self
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        return self

    def _run(self):
        p, h = self._nvml, self._handle
        while not self._stop.is_set():
            try:
                sm = p.nvmlDeviceGetClockInfo(h, p.NVML_CLOCK_SM)
                reasons = p.nvmlDeviceGetCurrentClocksEventReasons(h)
                util = p.nvmlDeviceGetUtilizationRates(h).gpu
                power = p.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.samples.append((sm, reasons, util, power))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)
        return False

    def summary(self) -> dict:
        if self._nvml is None:
            return {"available": False}
        p = self._nvml
        loaded = [s for s in self.samples if s[2] > 0] or self.samples
        if not loaded:
            return {"available": True, "samples": 0, "sm_max_mhz": self.max_mhz}
        reasons = set()
        for _, r, _, _ in loaded:
            for name, attr in _REASONS:
                bit = getattr(p, attr, 0)
                if bit and (r & bit) and name != "gpu_idle":
                    reasons.add(name)
        med = statistics.median(s[0] for s in loaded)
        rejecting = sorted(reasons & REJECTING)
        # SM clock well below max with no reason at all: a leftover clock lock
        if self.max_mhz and med < 0.8 * self.max_mhz and not reasons:
            rejecting.append("clock_stuck_low_no_reason")
        return {
            "sm_mhz": med,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(reasons),
            "samples": len(loaded),
            "power_w_max": max(s[3] for s in loaded),
            "rejecting": rejecting,
        }
