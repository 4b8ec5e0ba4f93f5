"""Element-stage probe: build the element ItI maps of one BASELINE config and
print the device time (and the per-label profile).  Used under ncu to list
the element kernels' launches.  Usage: python tools/element_probe.py [config] [reps]
"""
import sys
import time

sys.path.insert(0, ".")
import paper_2511_00735_b200 as hps  # noqa: E402


def main():
    cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    prob = hps.problem(2, cfgno, seed=cfgno)
    ctx = hps.Context(0)
    prof = len(sys.argv) > 3
    if prof:
        ctx.profile(True)
    for r in range(reps):
        ctx.synchronize()
        t0 = time.perf_counter()
        el = hps.build_elements(ctx, prob)
        ctx.synchronize()
        print(f"cfg{cfgno} rep {r}: element build wall {1e3 * (time.perf_counter() - t0):.2f} ms")
        del el
    if prof:
        print(ctx.profile_entries())


if __name__ == "__main__":
    main()
