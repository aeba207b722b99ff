"""The device ziggurat tail's log1p (csrc/glibc_log1p.h) is bit-identical
to the host C library's log1p — the function numpy's random_standard_normal
calls (npy_log1p) and so the one the reference's RNG stream depends on.
The header compiles as C; this runs it against libm on 3 x 10^7 arguments
(the tail's -u for u in [0,1), tiny, near -1, positive, huge)."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2501_05408_b200", "csrc")


def test_glibc_log1p_restatement_is_bit_exact(tmp_path):
    exe = tmp_path / "l1p"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-I", CSRC,
                           os.path.join(HERE, "csrc", "log1p_vs_libm.c"), "-o", str(exe), "-lm"])
    out = subprocess.run([str(exe), "30000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "mismatches=0" in out.stdout
