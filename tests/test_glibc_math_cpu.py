"""CPU: the device restatement of glibc's exp / log / cos (csrc/ctl_glibc.h)
is bit-identical to the host libm — the library the reference links — on the
inputs the control draws (tests/native/glibc_math_check.cpp: uniform draws for
log and cos(2*pi*u), lognormal exponents and softmax / budget weights for exp,
plus the polynomial branch of log near 1). This is what makes the device's
event logs byte-identical to the reference's (SURVEY.md §8c gate 2)."""
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_glibc_restatement_is_bit_exact(tmp_path):
    exe = tmp_path / "glibc_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", f"-I{ROOT / 'paper_2605_10195_b200' / 'csrc'}",
                    str(ROOT / "tests" / "native" / "glibc_math_check.cpp"), "-o", str(exe), "-lm"], check=True)
    p = subprocess.run([str(exe), "4000000"], capture_output=True, text=True, timeout=300)
    res = json.loads(p.stdout)
    assert p.returncode == 0 and res["bad_exp"] == res["bad_log"] == res["bad_cos"] == 0, res
