"""Trace-calibrated scaling MODEL of the multi-GPU factorization (not a measurement).

The dispatch order of every plan comes from a list-schedule simulation of the DAG with a task
duration model fitted to B200 traces (tqr_host.cpp DurModel).  This tool runs that simulation
for G = 1, 2, 4, 8 ranks (148 CTAs each, 1D block-cyclic columns) with a remote-edge delay
for every dependency that crosses GPUs (peer stores of V/T + system-scope release/acquire),
and reports modelled time, efficiency T1 / (G TG) and the % of G x 37.14 TF.  The G = 1 line
is printed next to the measured bench time so the model's calibration is visible.

  python tools/scaling_model.py [--remote-us 3] [--configs C3,C4,C5]
"""
import argparse
import sys

sys.path.insert(0, ".")
import tqr_inputs  # noqa: E402
from paper_0707_3548_b200 import tqr  # noqa: E402

MEASURED_MS = {"C2": 7.08, "C3": 198.0, "C4": 52.6, "C5": 12025.0}  # r01 bench
ap = argparse.ArgumentParser()
ap.add_argument("--remote-us", type=float, default=3.0)
ap.add_argument("--configs", default="C2,C3,C4,C5")
a = ap.parse_args()
print(f"MODEL (list-schedule simulation, remote edge +{a.remote_us} us); not a measurement")
for name in a.configs.split(","):
    c = tqr_inputs.CONFIGS[name]
    fl = tqr.flops_standard(c["m"], c["n"])
    t1 = None
    for G in (1, 2, 4, 8):
        ms, busy = tqr.schedule_model(c["m"], c["n"], c["b"], c["s"], G, 148, a.remote_us * 1e3)
        t1 = ms if G == 1 else t1
        eff = t1 / (G * ms)
        pct = 100 * fl / (ms * 1e-3) / (G * 37.14e12)
        extra = f"  (measured 1 GPU: {MEASURED_MS[name]:.1f} ms)" if G == 1 and name in MEASURED_MS else ""
        print(f"{name} G={G}: {ms:10.2f} ms  busy {busy:5.3f}  efficiency {eff:5.3f}  {pct:5.1f}% of G x 37.14 TF{extra}",
              flush=True)
