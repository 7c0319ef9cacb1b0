"""SURVEY 8(d) "equal accuracy": LancSVD vs RandSVD
on C3 (sparse 4e6 x 5e5) and C4 (dense 40000 x 20000) on one B200.

  1. RandSVD at the config's q: e_max = max_i ||A v_i - s_i u_i|| / s_1
     (tsvd_residuals, the library's own kernels).
  2. LancSVD to tol = that e_max (rho_i <= tol s_1, reading R12): its TTS at
     equal accuracy.
  3. RandSVD for q = 2, 4, 8, ... 64: e_max and TTS, i.e. the q it needs to
     reach LancSVD's 1e-8 (if it does within 64).
Times are CUDA events around the solve (median of 3 after one warm-up).
One JSON line per run.

    python scripts/equal_accuracy.py [C3 C4]
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2403_06218_b200 as T  # noqa: E402


def timed(h, fn, reps=3):
    fn()
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts)


def main():
    for name in sys.argv[1:] or ["C3", "C4"]:
        cfg, seed, work = bench.make_workload(name, 0)
        dwork = bench._to_device(work)
        h = T.TruncatedSVD(**dwork)
        h.set_seed(seed)
        r, b, d = cfg["r"], cfg["b"], cfg["d"]
        p = cfg["rsvd_p"]

        def rsvd_run(q):
            t = timed(h, lambda: h.rsvd(r, p, q))
            e, _ = h.residuals()
            return t, float(e.max())
        t_r, e_r = rsvd_run(cfg["rsvd_q"])
        print(json.dumps({"config": name, "method": "rsvd", "q": cfg["rsvd_q"], "l": r + p,
                          "tts_s": round(t_r, 4), "e_max": e_r}), flush=True)
        if os.environ.get("EQ_DSWEEP"):
            # smaller Krylov dimensions at the crude tolerance: LancSVD's
            # minimum work is one cycle of d, so the equal-accuracy time
            # depends on d; thick restart (keep = r rounded up to b) so a
            # small d can still hold the r wanted Ritz pairs across cycles
            keep = -(-r // b) * b
            for dd in (keep + b, keep + 2 * b, keep + 4 * b, 2 * keep, d):
                for kp in (0, keep):
                    if kp and kp >= dd:
                        continue
                    h.set_thick_restart(kp)
                    t_l = timed(h, lambda: h.block_lanczos(r, b, max(e_r, 1e-12), 40, d=dd))
                    e, _ = h.residuals()
                    inf = h.info()
                    print(json.dumps({"config": name, "method": "lanczos", "tol": e_r,
                                      "what": "equal accuracy, d sweep", "d": dd, "keep": kp,
                                      "b": b, "tts_s": round(t_l, 4), "e_max": float(e.max()),
                                      "cycles": inf["cycles"], "nconv": inf["nconv"]}),
                          flush=True)
            h.set_thick_restart(0)
            h.close()
            continue
        for tol, label in ((max(e_r, 1e-12), "equal accuracy (tol = rSVD e_max)"),
                           (1e-8, "north_star tol 1e-8")):
            t_l = timed(h, lambda: h.block_lanczos(r, b, tol, 12, d=d))
            e, _ = h.residuals()
            inf = h.info()
            print(json.dumps({"config": name, "method": "lanczos", "tol": tol, "what": label,
                              "d": d, "b": b, "tts_s": round(t_l, 4), "e_max": float(e.max()),
                              "cycles": inf["cycles"], "nconv": inf["nconv"]}), flush=True)
        for q in (2, 4, 8, 16, 32, 64):
            t, e = rsvd_run(q)
            print(json.dumps({"config": name, "method": "rsvd", "q": q, "l": r + p,
                              "tts_s": round(t, 4), "e_max": e}), flush=True)
            if e <= 1e-8:
                break
        h.close()
        del dwork, work
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
