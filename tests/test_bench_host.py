"""Host-side logic of bench.py (no GPU): the clock sampler's parsing and timed-window selection, and the CPU
baseline's thread count."""
import bench


def _line(sm, mx, pw, reasons=("Not Active",) * 4):
    return ", ".join(["0", str(sm), str(mx), str(pw), "0x0"] + list(reasons))


def test_clock_sampler_window_and_reasons():
    c = bench.ClockSampler(0)
    c.lines = [(0.0, _line(1965, 1965, 300.0)),                                   # warm-up, before the window
               (1.00, _line(1590, 1965, 900.0, ("Not Active", "Not Active", "Not Active", "Active"))),
               (1.05, _line(1575, 1965, 950.0)),
               (1.10, _line(1560, 1965, 920.0)),
               (9.0, _line(1965, 1965, 100.0)),                                   # after the window
               (1.02, "garbage line")]
    c.window(0.99, 1.11)
    s = c.summary()
    assert s["samples"] == 3 and s["sm_mhz"] == 1575 and s["sm_max_mhz"] == 1965
    assert s["reasons"] == ["sw_power_cap"] and s["power_w_max"] == 950.0


def test_clock_sampler_short_window_falls_back_to_neighbours():
    c = bench.ClockSampler(0)
    c.lines = [(0.95, _line(1600, 1965, 800.0)), (2.0, _line(1965, 1965, 100.0))]
    c.window(1.0, 1.01)  # shorter than the sampling period: no sample inside
    assert c.summary()["samples"] == 1 and c.summary()["sm_mhz"] == 1600


def test_clock_sampler_no_process():
    c = bench.ClockSampler(0)
    c.wait_first(timeout=0.01)  # no nvidia-smi started: returns at once
    assert c.summary()["samples"] == 0


def test_cpu_threads_positive():
    assert bench.cpu_threads() >= 1
