"""ssam_b200_measure_latency on the B200 (-m gpu): plausible cycle counts in
the order the hardware guarantees, and a profile file the reference's loader
accepts (perf_model.cpp:41-97)."""
import os

import pytest

pytestmark = pytest.mark.gpu


def test_measured_profile(cuda_lib, ref, tmp_path, monkeypatch):
    p = cuda_lib.measure_latency_profile()
    assert 2.0 <= p["t_mad"] <= 12.0
    assert p["t_shfl"] > p["t_mad"]
    assert p["t_smem_read"] > p["t_mad"]
    assert p["t_l2_read"] > p["t_smem_read"]
    assert p["t_gmem_read"] > p["t_l2_read"]
    assert p["t_gmem_write"] > 0 and p["sm_clock_mhz"] > 1000
    path = tmp_path / "B200x.profile"
    path.write_text(cuda_lib.format_profile("B200x", p))
    monkeypatch.setenv("SSAM_PROFILE_DIR", str(tmp_path))
    rc, name, vals, _ = ref.profile("B200x")
    assert rc == 0 and name == "B200x"
    assert abs(vals[1] - round(p["t_mad"])) <= 0.5
