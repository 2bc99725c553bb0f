"""Writes the generated kernels of the reference worked example
(3x^8-x^7+2x^6+x^5-4x^4+9x^3-3x^2-2x+1, Estrin) to docs/kernels/ so the
kernel structure can be read without running anything."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1307_5655_b200 as pe  # noqa: E402

out = os.path.join(ROOT, "docs", "kernels")
os.makedirs(out, exist_ok=True)
e = np.array([8, 7, 6, 5, 4, 3, 2, 1, 0]).reshape(-1, 1)
for name, coefs in (("f64", np.array([3, -1, 2, 1, -4, 9, -3, -2, 1], dtype=np.float64)),
                    ("i64", np.array([3, -1, 2, 1, -4, 9, -3, -2, 1], dtype=np.int64))):
    prog = pe.compile(pe.Polynomial(e, coefs), pe.builtin_scheme("estrin"))
    doms = {"f64": [("f64", pe.DOMAIN_F64), ("f64strict", pe.DOMAIN_F64_STRICT),
                    ("interval", pe.DOMAIN_INTERVAL)],
            "i64": [("i64", pe.DOMAIN_I64), ("i64f", pe.DOMAIN_I64F)]}[name]
    for tag, d in doms:
        path = os.path.join(out, f"example_estrin_{tag}.ptx")
        with open(path, "w") as f:
            f.write(prog.ptx(d))
        cubin = path.replace(".ptx", ".cubin")
        subprocess.run(["ptxas", "-arch=sm_100a", "-O3", path, "-o", cubin], check=True)
        sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
        with open(path.replace(".ptx", ".sass"), "w") as f:
            f.write(sass)
        os.remove(cubin)
        print("wrote", path)
