"""Host-side pieces of bench.py's contract (no GPU): the nvidia-smi clocks
parser keeps only samples of the benchmarked GPUs inside the timed region
and reports the throttle reasons that void a run; peaks come from
MEASURED_PEAKS.json."""
import datetime
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class _Proc:
    def terminate(self):
        pass

    def wait(self, timeout=None):
        return 0


def _line(t, gpu, sm, mx, hw="Not Active", thermal="Not Active", swth="Not Active", pcap="Not Active"):
    ts = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
    return f"{ts}, {gpu}, {sm}, {mx}, 700.5, 0x0, {hw}, {thermal}, {swth}, {pcap}\n"


def _clocks(gpus, lines, t0, t1):
    c = bench.Clocks.__new__(bench.Clocks)
    c.gpus, c.p, c.lines, c.t0, c.t1 = set(gpus), _Proc(), lines, t0, t1
    return c


def test_clocks_window_gpu_filter_and_reasons():
    t0 = 1_700_000_000.0
    lines = [
        _line(t0 - 5, 0, 900, 1965),                       # before the timed region: dropped
        _line(t0 + 0.1, 0, 1935, 1965, pcap="Active"),     # in: sw_power_cap (kept, noted)
        _line(t0 + 0.2, 0, 1950, 1965),
        _line(t0 + 0.3, 1, 1200, 1965, hw="Active"),       # another GPU: ignored
        _line(t0 + 0.4, 0, 1965, 1965),
        _line(t0 + 9, 0, 800, 1965, thermal="Active"),     # after: dropped
        "garbage line\n",
    ]
    r = _clocks([0], lines, t0, t0 + 1.0).stop()
    assert r == {"sm_mhz": 1950.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"], "samples": 3}


def test_clocks_reports_rejecting_reasons():
    t0 = 1_700_000_000.0
    lines = [_line(t0 + 0.1, 2, 1500, 1965, hw="Active", swth="Active"),
             _line(t0 + 0.2, 3, 1600, 1965, thermal="Active")]
    r = _clocks([2, 3], lines, t0, t0 + 1).stop()
    assert r["reasons"] == ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
    assert r["samples"] == 2 and r["sm_mhz"] == 1550.0


def test_clocks_no_samples():
    r = _clocks([0], [], 0.0, 1.0).stop()
    assert r == {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}


def test_peaks_from_measured_file():
    peak, src = bench.load_peaks()
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        assert src.startswith("measured") and 4000 < peak < 9000
    else:
        assert src.startswith("fallback")


def test_bench_scripts_compile():
    """bench.py loads scripts/bench_extras.py at run time: keep it importable."""
    import py_compile
    for f in ("bench.py", os.path.join("scripts", "bench_extras.py")):
        py_compile.compile(os.path.join(ROOT, f), doraise=True)


def test_metric_bytes_definition():
    """value's bytes: world 1 = the fused step's HBM bytes (16 B/elem + 16 B/block);
    world m = every rank's AG + RS wire bytes, m * 2 (m-1) S 2."""
    assert bench.metric_bytes(1, 4096, 4096, 2) == 16 * 4096 + 32
    assert bench.metric_bytes(4, 1000, 3990, 2) == 4 * 2 * 3 * 1000 * 2
