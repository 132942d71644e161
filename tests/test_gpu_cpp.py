"""The C++ drop-in layer on the GPU: tests/cpp/test_rd_gpu.cpp re-expresses the
reference's hot-path test cases through include/rd_gpu.hpp."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_reference_cases(O):
    exe = os.path.join(ROOT, "tests", "cpp", "test_rd_gpu")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2102_03515_b200"), "cpptest"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    its = int(re.search(r"C1 n=32: (\d+) iterations", out.stdout).group(1))
    om = O.build_structured_cube(32)
    os_ = O.build_system(om, 1.0 / 1024.0, "smooth")
    ref = O.solve_system_amg(os_)
    assert its == ref.iterations
    m = re.search(r"C1 n=32: l2 (\S+) h1 (\S+)", out.stdout)
    l2o = O.l2_error_manufactured(om, os_, ref.u, 1.0 / 1024.0)
    h1o = O.h1_semi_error_manufactured(om, os_, ref.u, 1.0 / 1024.0)
    assert abs(float(m.group(1)) - l2o) <= 1e-9 * l2o and abs(float(m.group(2)) - h1o) <= 1e-9 * h1o
