"""The measured B200 latency profile: profiles/B200.profile is
what tools/latency_profile.py wrote on a B200, and the reference's own
loader (perf_model.cpp:41-97, resolve_profile via SSAM_PROFILE_DIR) accepts
it; its model then prices the register cache below the shared-memory cache
as on P100/V100 (perf_model.hpp:34-44)."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILE = os.path.join(ROOT, "profiles", "B200.profile")


def test_committed_profile_format(lib):
    with open(PROFILE) as fh:
        lines = [l.split() for l in fh.read().splitlines() if l.strip()]
    assert lines[0] == ["name", "B200"]
    fields = {k: int(v) for k, v in lines[1:]}
    assert tuple(fields) == lib.PROFILE_FIELDS
    assert all(v >= 1 for v in fields.values())
    assert fields["t_gmem_read"] > fields["t_smem_read"] > fields["t_mad"]
    # format_profile writes exactly this layout
    assert lib.format_profile("B200", {k: float(v) for k, v in fields.items()}) == \
        open(PROFILE).read()


def test_reference_loader_accepts_it(ref, monkeypatch):
    monkeypatch.setenv("SSAM_PROFILE_DIR", os.path.dirname(PROFILE))
    rc, name, vals, lat = ref.profile("B200", 7, 7)
    assert rc == 0 and name == "B200"
    assert np.all(vals > 0)
    l_reg, l_smem = lat
    assert l_reg < l_smem  # the register cache wins at 7x7, as the paper's model says
    rc, _, v100, _ = ref.profile("V100")
    assert rc == 0 and v100[1] == 4  # built-ins still resolve first
