"""A plain-C client compiles against include/polyeval_b200.h (gcc -std=c11,
-Werror) and runs the host-only entry points through the shared library."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1307_5655_b200", "_lib")


def test_c11_client(tmp_path):
    exe = tmp_path / "abi_check"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_check.c"), "-o", str(exe), "-L", LIB,
                    "-lpolyeval_b200", f"-Wl,-rpath,{LIB}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "C ABI ok" in r.stdout
