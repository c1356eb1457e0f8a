"""Mutation check of the oracle pins: compile variants of oracle/crisp_oracle.c
with one plausible mistake each and show that a pin in tests/test_oracle_pins.py
fails on it (the pins would catch that mistake).  CPU only; run from the repo
root: python tools/oracle_mutations.py"""
import ctypes
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402
import test_oracle_pins as pins  # noqa: E402

SRC = open(os.path.join(ROOT, "oracle", "crisp_oracle.c")).read()
STOP = """            } else {
                cnt++;
            }
            if (ix->patience > 0 && cnt == ix->patience) break;"""
PRUNE = """                    cnt++;
                    if (ix->patience > 0 && cnt == ix->patience) break;
                    continue;"""
MUTANTS = {
    # exact patience: stop one verification late / early (O15 step 4)
    "stop_late": (STOP, STOP.replace("cnt == ix->patience)", "cnt == ix->patience + 1)"),
                  lambda: pins.test_patience_stop_is_exact(2)),
    "stop_early": (STOP, STOP.replace("cnt == ix->patience)", "cnt + 1 == ix->patience)"),
                   lambda: pins.test_patience_stop_is_exact(2)),
    # ADSampling: a prune that does not count as a non-improving verification
    "prune_not_counted": (PRUNE, "                    continue;",
                          pins.test_adsampling_prune_counts_as_non_improvement),
}


def main():
    bad = 0
    for name, (old, new, pin) in MUTANTS.items():
        assert old in SRC, name
        with tempfile.TemporaryDirectory() as d:
            c, so = os.path.join(d, "m.c"), os.path.join(d, "m.so")
            open(c, "w").write(SRC.replace(old, new))
            subprocess.check_call(["gcc", *oracle.CFLAGS, "-o", so, c, "-lm"])
            L = ctypes.CDLL(so)
            oracle._declare(L)
            saved, oracle._lib = oracle._lib, L
            try:
                pin()
                print(f"{name}: NOT caught")
                bad += 1
            except AssertionError as e:
                print(f"{name}: caught ({(str(e) or 'assert').splitlines()[0][:70]})")
            finally:
                oracle._lib = saved
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
