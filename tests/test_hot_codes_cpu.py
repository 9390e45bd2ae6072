"""Compile-pass hot codes (evogp_internal.h HotCode, the packed interpreter's
opcodes): the branch-free mapping from a decoded node word to its code is
checked on the host against the table written case by case (g++, no GPU)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_hot_code_mapping(tmp_path):
    exe = tmp_path / "hot_codes_check"
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I/usr/local/cuda/include", "-o", str(exe),
                           os.path.join(HERE, "cpp", "hot_codes_check.cpp")])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
