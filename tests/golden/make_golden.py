#!/usr/bin/env python
"""Regenerate tests/golden/reference_cases.json from the UNMODIFIED reference.

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


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    if not os.path.exists(GEN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    text = subprocess.run([GEN], check=True, capture_output=True, text=True).stdout
    cases = json.loads(text)
    if args.check:
        with open(OUT) as f:
            same = json.load(f) == cases
        print("golden up to date" if same else "golden DIFFERS from the reference output")
        return 0 if same else 1
    with open(OUT, "w") as f:
        f.write(text)
    print(f"wrote {len(cases)} cases to {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
