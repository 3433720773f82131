"""Long parity runs of the B200 propagator against the CPU oracle.

    python scripts/parity_run.py [cfg ...] [--out gpurun_out/parity.json]

cfg1   64^3 run_bench harmonic trap, 1000 steps, populations every 50
cfg2b  128x128x256 Ioffe-floor harmonic (population-moving), 5000 steps / 25
cfg2   128x128x256 scaled-chip CTAP (configs/scaled.cfg with n_y = 128),
       25,000 steps, PopulationRecorder every 50 (V checked on all points)
cfg3   256^3 paper-chip CTAP, 1000 steps / 100
cfg4   512^3 paper-chip CTAP, 100 steps / 50 (cfg4long: 1000 steps, ~10 min of oracle)
cfg3c64 / cfg4c64  the same in complex64 mode, gate 1e-4 against the oracle
cfg5   1024x1024x512 harmonic trap, 5 steps (one GPU vs the oracle, ~50 GB host RAM)

The cases are tests/baseline_cases.py's (shared with the driver-run
tests/test_gpu_baseline_configs.py, which runs them at bounded step counts).
Gates (BASELINE north_star): psi rel L2 <= 1e-10, every trace row's p_l, p_m,
p_r within 1e-9.  The oracle is the checker only (test infrastructure).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import baseline_cases as bc  # noqa: E402

CASES = {
    "cfg1": lambda: (bc.cfg1(), 1000, "complex128"),
    "cfg2b": lambda: (bc.cfg2b(), 5000, "complex128"),
    "cfg2": lambda: (bc.cfg2(every=None), 25000, "complex128"),
    "cfg3": lambda: (bc.cfg3(every=8), 1000, "complex128"),
    "cfg4": lambda: (bc.cfg4(every=8), 100, "complex128"),
    "cfg4long": lambda: (bc.cfg4(every=16), 1000, "complex128"),
    "cfg3c64": lambda: (bc.cfg3(every=8), 1000, "complex64"),
    "cfg4c64": lambda: (bc.cfg4(every=8), 100, "complex64"),
    "cfg5": lambda: (bc.cfg5(), 5, "complex128"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["cfg1", "cfg2b", "cfg3", "cfg2"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    results = []
    for c in args.cases:
        case, steps, precision = CASES[c]()
        r = bc.run_case(case, steps, precision=precision)
        if precision != "complex128":
            r["case"] += ", " + precision
        print(json.dumps(r), flush=True)
        results.append(r)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as fh:
            json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
