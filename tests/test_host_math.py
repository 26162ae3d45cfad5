"""Host-side checks of the kernel's SWAR mask and cut-point logic (no GPU).

csrc/dmsgm_math.cuh is compiled for the host (g++ -ffp-contract=off) and its
interval/SWAR mask is compared with the literal per-pixel predicate
fl(fl(I - mu)^2) > T (App. E, reading R14) for every intensity 0..255 on
millions of random and adversarial (mu, T) pairs ("mask as two rays").
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_swar_and_intervals(tmp_path):
    exe = tmp_path / "host_math_check"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
                           "-I", os.path.join(ROOT, "paper_1702_05156_b200", "csrc"),
                           "-o", str(exe), os.path.join(ROOT, "tests", "host_math_check.cpp")])
    out = subprocess.run([str(exe), "3000000"], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "swar_bad 0" in out.stdout
    assert "interval_fails 0 of" in out.stdout
