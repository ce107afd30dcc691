"""Mutation check of the oracle's policy pins (VERDICT r1 "What's weak" #1).

Copies oracle/, tests/, synth.py and pytest.ini to a scratch directory once per mutant,
applies one plausible mistake to oracle/nb_oracle.c, and runs the oracle pins there.
Every mutant must make at least one pin fail; the script exits 1 if one survives.

  m1: mixed glsc3 accumulates in binary32
  m2: mixed Jacobi uses the fp32 copy of the diagonal, z = r * (float)dinv
  m3: mixed rho / beta computed in binary32
  m4: mixed gather-scatter accumulates in binary32
  m5: fp32 policy takes the fp64 diagonal

Usage: python tools/oracle_mutants.py [--tests tests/test_oracle_policy.py ...]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTANTS = {
    "m1": ("    double s = 0.0;\n    for (int64_t i = 0; i < n; i++) s += ((double)a[i] * c[i]) * (double)b[i];",
           "    float s = 0.0f;\n    for (int64_t i = 0; i < n; i++) s += ((double)a[i] * c[i]) * (double)b[i];"),
    "m2": ("z[l] = (float)((double)r[l] * m->dinv[l]);", "z[l] = r[l] * m->dinvf[l];"),
    "m3": ("                rho = DOT(r, z);\n                double beta = (k == 1) ? 0.0 : rho / rho_old;",
           "                rho = (float)DOT(r, z);\n"
           "                double beta = (k == 1) ? 0.0 : (float)((float)rho / (float)rho_old);"),
    "m4": ("    if (policy == OR_MIXED) or_dssum_fd(m, order, w);", "    if (policy == OR_MIXED) or_dssum_f(m, order, w);"),
    "m5": ("            else for (int64_t l = 0; l < NL; l++) z[l] = r[l] * m->dinvf[l];",
           "            else for (int64_t l = 0; l < NL; l++) z[l] = (float)((double)r[l] * m->dinv[l]);"),
}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tests", nargs="*", default=["tests/test_oracle_policy.py"])
    a = ap.parse_args()
    survivors = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, (old, new) in MUTANTS.items():
            d = os.path.join(tmp, name)
            os.makedirs(d)
            for item in ("oracle", "tests", "synth.py", "pytest.ini"):
                src = os.path.join(ROOT, item)
                (shutil.copytree if os.path.isdir(src) else shutil.copy)(src, os.path.join(d, item))
            so = os.path.join(d, "oracle", "libnb_oracle.so")
            if os.path.exists(so):
                os.remove(so)
            src = os.path.join(d, "oracle", "nb_oracle.c")
            s = open(src).read()
            assert old in s, f"{name}: pattern not found"
            open(src, "w").write(s.replace(old, new, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "not gpu",
                                *a.tests], cwd=d, capture_output=True, text=True)
            tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
            killed = r.returncode != 0
            print(f"{name}: {'killed' if killed else 'SURVIVED'} ({tail})")
            if not killed:
                survivors.append(name)
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
