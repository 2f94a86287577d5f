#!/usr/bin/env python
"""Regenerate tests/golden/reference_cases.json and trainer_cases.json from the
UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY.  Runs in the dev container, where /root/reference
exists:

    make -C oracle            # builds oracle/_ref/gen_golden from /root/reference/proj/src
    python tests/golden/make_golden.py [--check]

oracle/_ref/gen_golden (oracle/gen_golden.cpp linked against the reference's
tensor.cpp / layers.cpp / gns.cpp / costmodel.cpp) replays the reference's own
known-answer tests and seeded random families (see the family list at the top
of oracle/gen_golden.cpp) and prints every case with its inputs and the
reference's outputs as JSON.  --check only verifies that the committed file is
what the reference produces today.

oracle/_ref/gen_trainer_golden (oracle/gen_trainer_golden.cpp linked against
the reference's model.cpp / dataset.cpp / trainer.cpp as well) prints
MarkovDataset streams, make_toy_model weights, scheduled_batch values and
Trainer::step logs of PerExample runs -> trainer_cases.json.
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
GEN = os.path.join(ROOT, "oracle", "_ref", "gen_golden")
OUT = os.path.join(HERE, "reference_cases.json")
GEN_T = os.path.join(ROOT, "oracle", "_ref", "gen_trainer_golden")
OUT_T = os.path.join(HERE, "trainer_cases.json")


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    if not os.path.exists(GEN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    rc = 0
    for gen, out in ((GEN, OUT), (GEN_T, OUT_T)):
        text = subprocess.run([gen], check=True, capture_output=True, text=True).stdout
        cases = json.loads(text)
        if args.check:
            with open(out) as f:
                same = json.load(f) == cases
            print(f"{os.path.basename(out)}: " + ("up to date" if same else "DIFFERS from the reference output"))
            rc |= 0 if same else 1
            continue
        with open(out, "w") as f:
            f.write(text)
        print(f"wrote {len(cases)} cases to {out}")
    return rc


if __name__ == "__main__":
    sys.exit(main())
