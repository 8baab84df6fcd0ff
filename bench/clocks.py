"""nvidia-smi sampling of one GPU's clocks, power and throttle reasons during a
timed region (bench.py; the driver's clocks rule).  One sampler per rank, each
on its own GPU, so a multi-GPU line carries every GPU's clocks."""
import statistics
import subprocess
import threading

THROTTLE = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms between start() and stop()."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self, wait_s=3.0):
        """Start sampling; returns once the first sample is in (nvidia-smi takes a few
        hundred ms to start), so even a sub-second timed region gets samples."""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.first = threading.Event()
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self.first.wait(wait_s)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self.first.set()

    def stop(self):
        if self.proc is None:
            return {"gpu": self.gpu, "sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0, "power_w_median": None}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        return summarise(self.lines, self.gpu)


def summarise(lines, gpu=None):
    """Median SM clock under load, max clock, throttle reasons seen, median power."""
    sm, smax, reasons, power = [], None, set(), []
    for ln in lines:
        parts = [p.strip() for p in ln.split(",")]
        if len(parts) < 9:
            continue
        try:
            sm.append(float(parts[1]))
            smax = float(parts[2])
            power.append(float(parts[3]))
        except ValueError:
            continue
        for name, val in zip(THROTTLE, parts[5:9]):
            if val.lower() == "active":
                reasons.add(name)
    busy = [v for v in sm if smax and v > 0.5 * smax] or sm
    return {"gpu": gpu, "sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
            "reasons": sorted(reasons), "samples": len(sm),
            "power_w_median": statistics.median(power) if power else None}
