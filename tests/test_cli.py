"""The `ssam` command line (paper_1907_06154_b200/bin/ssam) end to end.

Mirrors proj/tests/test_cli.cpp and acceptance criterion 8
(proj/tests/acceptance.cpp:273-297): exit codes 0 pass / 1 mismatch / 2
usage, the --corrupt fault-injection hook, and byte-identical --out reports
for identical flags.  Usage errors are decided before any device work, so
they run on CPU; everything that computes is -m gpu.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1907_06154_b200", "bin", "ssam")


def run(args, cwd=None):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built (make)")
    p = subprocess.run([CLI] + args.split(), capture_output=True, text=True, cwd=cwd, timeout=300)
    return p.returncode, p.stdout + p.stderr


def test_usage_errors_exit_2():
    assert run("run wat")[0] == 2
    assert run("frobnicate")[0] == 2
    assert run("run stencil2d --precision int")[0] == 2
    assert run("cost --sweep nonsense")[0] == 2
    assert run("run conv2d --w 8 --h 64 --precision int")[0] == 2  # narrower than a warp
    assert run("run conv2d --m 21 --n 3 --precision int")[0] == 2  # filter cap (kernels.hpp:192)
    assert run("run conv2d --h 400 --p 300")[0] == 2               # C > 255: length_error
    assert run("bench --suite nope")[0] == 2
    assert run("run conv2d --bogus 1")[0] == 2


@pytest.mark.gpu
def test_run_int_conv2d_passes_exactly(cuda_lib):
    rc, out = run("run conv2d --w 64 --h 64 --m 3 --n 3 --precision int --seed 1")
    assert rc == 0, out
    assert "max_rel_err=0" in out


@pytest.mark.gpu
def test_corrupt_hook_forces_mismatch(cuda_lib):
    assert run("run conv2d --w 64 --h 64 --m 3 --n 3 --precision int --corrupt")[0] == 1


@pytest.mark.gpu
def test_reports_are_byte_identical(cuda_lib, tmp_path):
    """acceptance criterion 8: two invocations, byte-identical machine reports."""
    flags = "run conv2d --w 128 --h 96 --m 5 --n 4 --precision f64 --seed 3 --out "
    a, b = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    assert run(flags + str(a))[0] == 0
    assert run(flags + str(b))[0] == 0
    ta, tb = a.read_bytes(), b.read_bytes()
    assert ta and ta == tb
    assert b'"pass":true' in ta


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    "run conv1d --len 5000 --m 9 --precision f32",
    "run conv1d --len 211 --m 32 --precision int --boundary replicate",
    "run scan --len 4096 --precision int",
    "run scan --len 4096 --precision f64",
    "run stencil2d --stencil 2d9pt --w 256 --h 256 --iters 8 --precision f32",
    "run stencil2d --stencil 2d121pt --w 128 --h 128 --precision f64",
    "run stencil3d --stencil poisson --nx 64 --ny 64 --nz 64 --precision f64",
    "run stencil3d --stencil 3d125pt --nx 48 --ny 40 --nz 36 --precision f32",
    "run conv2d --w 300 --h 200 --m 20 --n 17 --precision f32 --boundary replicate",
])
def test_run_kernels_pass(cuda_lib, args):
    rc, out = run(args)
    assert rc == 0, out


@pytest.mark.gpu
def test_input_and_dump_output(cuda_lib, tmp_path):
    import numpy as np
    dumped = tmp_path / "out.sgrd"
    assert run(f"run conv2d --w 96 --h 64 --precision f64 --seed 5 --dump-output {dumped}")[0] == 0
    g = cuda_lib.read_grid2d(str(dumped), np.float64)
    assert g.shape == (64, 96)
    # feed it back as the input of a stencil run
    assert run(f"run stencil2d --input {dumped} --precision f64")[0] == 0


@pytest.mark.gpu
def test_bench_table3_small(cuda_lib, tmp_path):
    out = tmp_path / "t3.jsonl"
    rc, text = run(f"bench --suite table3 --size 128 --size3d 32 --precision f32 --out {out}")
    assert rc == 0, text
    assert len(out.read_text().strip().splitlines()) == 15
