"""The README's usage example runs as written (at a 64^3 grid and 100 steps
instead of 512^3 and 10,000, so it stays a seconds-long test)."""

import os
import re

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_readme_example_runs():
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.findall(r"```python\n(.*?)```", text, flags=re.S)[0]
    code = code.replace("512, 512, 512", "64, 64, 64").replace("4e-6 / 1024", "4e-6 / 128").replace("10_000", "100")
    ns = {}
    exec(compile(code, "README.md", "exec"), ns)
    rec, stats = ns["rec"], ns["stats"]
    assert stats.n_steps == 100
    rows = rec.trace.as_array()
    assert rows.shape == (3, 6)
    assert abs(rows[-1, 4] - 1.0) < 1e-10          # norm conserved
