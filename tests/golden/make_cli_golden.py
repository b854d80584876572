"""Generates tests/golden/cli_generate_golden.json from the UNMODIFIED reference generator.

`oracle/_ref/refio --gen N D Z SEED OUT` runs the reference's `generate` body
(tools/sfd_main.cpp:90-98: sfd::SyntheticStream through sfd::MatrixMarketWriter, built from
/root/reference by oracle/Makefile). The fixture records the SHA-256 and size of each output so
tests/test_cli.py can pin `sfdg generate` byte for byte where the reference is absent.
Run in the build container:  python tests/golden/make_cli_golden.py
"""
import hashlib
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REFIO = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "refio")
# (n, d, z, seed): defaults-shaped, tiny, z = d (tail empty), head-only, wide
SPECS = [(2000, 500, 30, 7), (200, 10, 7, 1), (50, 3, 3, 2), (300, 40, 40, 9), (100, 5000, 250, 123)]


def main():
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        for n, d, z, seed in SPECS:
            path = os.path.join(tmp, "g.mtx")
            subprocess.run([REFIO, "--gen", str(n), str(d), str(z), str(seed), path], check=True)
            data = open(path, "rb").read()
            out.append({"n": n, "d": d, "z": z, "seed": seed, "bytes": len(data),
                        "sha256": hashlib.sha256(data).hexdigest()})
    with open(os.path.join(HERE, "cli_generate_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
