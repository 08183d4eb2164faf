"""Host-side pieces of bench.py that need no GPU: the clock sampler's parsing / window /
under-load statistics (the GPU side is exercised by every gpurun bench)."""
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def _sampler_with(lines):
    cs = bench.ClockSampler(0)
    f = tempfile.NamedTemporaryFile(mode="w", suffix=".csv", delete=False)
    f.write("".join(lines))
    f.close()
    cs.out = f
    cs.source = "nvml"
    cs.proc = subprocess.Popen([sys.executable, "-c", "import time; time.sleep(30)"])
    return cs


def test_clock_window_and_load_filter():
    # t, sm, max, power, reasons (0x4 = sw_power_cap, 0x40 = hw_thermal_slowdown)
    rows = [f"{100 + i * 0.05:.3f},1965,1965,200.0,0\n" for i in range(10)]          # idle ramp
    rows += [f"{101 + i * 0.05:.3f},{1300 + i},1965,990.0,4\n" for i in range(20)]   # loaded
    rows += ["102.500,1965,1965,150.0,64\n"]                                          # after
    cs = _sampler_with(rows)
    out = cs.stop(window=(101.0, 102.2))
    assert out["samples"] == 20 and out["samples_all"] == 31
    assert out["sm_mhz"] == 1309.5 and out["sm_max_mhz"] == 1965
    assert out["reasons"] == ["sw_power_cap"]  # the thermal sample is outside the window
    cs = _sampler_with(rows)
    whole = cs.stop()
    assert whole["reasons"] == ["sw_power_cap"]  # 150 W sample is below half peak power
    assert whole["samples_under_load"] == 20


def test_clock_window_too_small_falls_back_to_all():
    rows = [f"{100 + i:.3f},1400,1965,900.0,4\n" for i in range(5)]
    cs = _sampler_with(rows)
    out = cs.stop(window=(103.5, 104.5))  # 1 sample inside: use all 5
    assert out["samples"] == 5 and out["sm_mhz"] == 1400


def test_trace_summary_monitor_reading():
    """bench.trace_summary: per-stream end times and the reference monitor() reading
    (nano_pipeline.hpp:114-126) from per-nano-batch main / comm spans of a traced step."""
    from paper_2602_07263_b200 import capi
    op = lambda kind, stream, nano: {"kind": kind, "stream": stream, "nano": nano}  # noqa: E731
    trace = [(op(capi.OP_SHRINK, capi.STREAM_MAIN, 0), 0.1), (op(capi.OP_FWD, capi.STREAM_MAIN, 0), 2.0),
             (op(capi.OP_GRADS, capi.STREAM_SIDE, 0), 2.5), (op(capi.OP_FWD, capi.STREAM_MAIN, 1), 5.0),
             (op(capi.OP_ALLREDUCE, capi.STREAM_COMM, 1), 6.0), (op(capi.OP_ADAMW, capi.STREAM_COMM, 1), 6.5)]
    out = bench.trace_summary(trace, 7.0)
    assert out["stream_end_ms"] == {"main": 5.0, "side": 2.5, "comm": 6.5}
    assert out["t_comp_ms"] == [2.0, 3.0] and out["t_comm_ms"] == [0.0, 1.5]
    # eta = sum(t_comp) / (1 * t_iter) ; stall = t_iter - max(sum t_comp, sum t_comm)
    assert out["monitor"] == {"eta_util": round(5.0 / 7.0, 4), "delta_stall_ms": 2.0}
