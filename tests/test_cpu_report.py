"""Report writers (csrc/host/report.cpp) vs the reference's own
report_to_json / iterations_to_jsonl / report_summary_line and the CLI's
ranked.json / sweep recipes, byte for byte on random reports with edge-case
doubles (tests/native/report_check.cpp, linked against oracle/_ref)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
REF_LIB = os.path.join(REPO, "oracle", "_ref", "libplansim_ref.a")
PKG = os.path.join(REPO, "paper_2411_17651_b200")


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and os.path.exists(REF_LIB)
                         and os.path.exists(os.path.join(PKG, "libpsg.so"))),
                    reason="needs the reference headers, oracle/_ref and libpsg.so")
def test_report_writers_byte_identical(tmp_path):
    exe = tmp_path / "report_check"
    subprocess.run(["g++", "-O1", "-std=c++20", "-I", REF_INC,
                    "-I", os.path.join(REPO, "oracle", "_ref", "vendor"),
                    "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "tests", "native", "report_check.cpp"), REF_LIB,
                    "-L", PKG, "-lpsg", f"-Wl,-rpath,{PKG}", "-lpthread", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, cwd=tmp_path, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr
    assert "bad=0" in out.stdout
