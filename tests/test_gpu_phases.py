"""GPU: KV-range phases of the bf16 attention kernel (fa_phases in csrc/attention_fa.cu, the
SURVEY §8(f)2 GQA-group K/V sharing through L2).

A phased launch splits every long row's block list at the phase boundaries and carries the exact
fp32 (O, m, l) of the row between phases, so its arithmetic is the unphased kernel's, in the same
order: the bar is bit-equality with the unphased call (which the other GPU suites tie to the
reference).  Phases are forced with FPB_FA_PHASES (read once per process) in a subprocess.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2603_06199_b200 as fp
from paper_2603_06199_b200 import _abi
case, out = sys.argv[1], sys.argv[2]
exec(open({root!r} + "/tests/_phase_cases.py").read())
res = run(fp, case)
np.savez(out, **{{k: v.float().cpu().numpy() if v.is_floating_point() else v.cpu().numpy()
                 for k, v in res.items()}})
'''


def _child(case, phases, tmp_path):
    out = str(tmp_path / f"{case}_{phases}.npz")
    env = dict(os.environ, FPB_FA_PHASES=str(phases))
    code = CHILD.format(root=ROOT)
    r = subprocess.run([sys.executable, "-c", code, case, out], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(out))


@pytest.mark.parametrize("case", ["sparse", "dense", "arbitrary", "ragged_gqa"])
@pytest.mark.parametrize("phases", [2, 3])
def test_phased_equals_unphased(case, phases, tmp_path):
    a = _child(case, 1, tmp_path)
    b = _child(case, phases, tmp_path)
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k], equal_nan=True), (case, phases, k)
