"""Copy the reference's small test fixtures (QAPLIB-format instances, solutions and the
manifest under proj/fixtures/) into tests/golden/fixtures.json, so the reference's own
unit tests compiled against the facade can run where /root/reference is absent (the
GPU box).  Data only; run here: python tests/golden/make_fixtures.py"""
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_FIX = "/root/reference/proj/fixtures"


def main():
    out = {}
    for name in sorted(os.listdir(REF_FIX)):
        with open(os.path.join(REF_FIX, name)) as fh:
            out[name] = fh.read()
    with open(os.path.join(HERE, "fixtures.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
