"""CLI usage errors (no GPU): exit code 64 (SPEC.md "[MODULE] cli")."""
import subprocess
import sys

import pytest

from paper_2002_05024_b200 import cli


@pytest.mark.parametrize("argv", [[], ["frobnicate"], ["reorder", "--s", "x"], ["generate", "--kind", "nope", "--n", "3",
                                                                                "--out", "o"]])
def test_usage_errors_exit_64(argv):
    assert cli.main(argv) == 64


def test_bad_select_spec_is_a_usage_error(tmp_path):
    import numpy as np
    from paper_2002_05024_b200 import io
    p = str(tmp_path / "s.teig")
    io.write_matrix_file(p, np.eye(3), "teig")
    # selection parsing fails before any device work
    with pytest.raises(cli.UsageError):
        cli._selection(None, None, "bogus=1")


def test_module_entry_point_help():
    r = subprocess.run([sys.executable, "-m", "paper_2002_05024_b200.cli", "--help"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "generate" in r.stdout and "trace-dump" in r.stdout
