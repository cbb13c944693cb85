"""The closed-form repeated addition used by decode runs
(paper_2411_17651_b200/csrc/psg_fastsum.cuh) against sequential FP64
round-to-nearest stepping — the reference's per-iteration accumulation
(simulator.cpp:125-133).  Host build of the same header the kernel uses."""
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fastsum_matches_sequential_adds(tmp_path):
    exe = tmp_path / "fastsum_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    "-I", os.path.join(REPO, "paper_2411_17651_b200", "csrc"),
                    os.path.join(REPO, "tests", "native", "fastsum_check.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), "100000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad=0" in out.stdout
