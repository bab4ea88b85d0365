"""Generate tests/golden/golden.npz from the REFERENCE build (oracle/_ref).

Run in the build container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixture is committed; tests/test_oracle_pin.py checks the plain-C
restatement against it bit for bit on any machine (including the GPU box,
where /root/reference is absent).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import oracle  # noqa: E402
import scenarios  # noqa: E402


def main():
    O = oracle.load("reference")
    data = scenarios.run_all(O)
    msgs = []
    for case in scenarios.error_cases(O):
        try:
            case()
            msgs.append("<no error>")
        except oracle.OracleError as e:
            msgs.append(str(e))
    data["errors"] = np.array(msgs)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {len(data)} arrays to {path}")


if __name__ == "__main__":
    main()
