"""The GPU CLI (``paper_1604_08501_b200/cli.py``) against the reference CLI's
``bench`` / ``check`` contract (``lf/cli.py:77-162``): argument syntax,
output lines, exit codes."""

from __future__ import annotations

import pytest

from paper_1604_08501_b200.cli import _parse_int_list, build_parser, main


def test_int_list_syntax():
    assert _parse_int_list("1..8") == list(range(1, 9))
    assert _parse_int_list("2,3,4") == [2, 3, 4]
    assert _parse_int_list("1..2,5") == [1, 2, 5]


def test_parser_defaults_and_required():
    a = build_parser().parse_args(["bench", "--nq", "4", "--ne", "3"])
    assert (a.level, a.seed, a.report, a.check) == (8, 1, "text", False)
    with pytest.raises(SystemExit):
        build_parser().parse_args(["bench", "--nq", "4"])
    c = build_parser().parse_args(["check"])
    assert (c.levels, c.nq, c.ne, c.seeds) == ("1..8", "2,4,8", "1,2,5", "1")


def test_bad_configuration_exits_1(capsys):
    assert main(["bench", "--nq", "4", "--ne", "0"]) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_bench_and_check_on_gpu(cuda_device, capsys, tmp_path):
    out = tmp_path / "k.cl"
    assert main(["bench", "--nq", "4", "--ne", "64", "--report", "csv",
                 "--emit", str(out)]) == 0
    text = capsys.readouterr().out.splitlines()
    assert text[0].startswith("level,nq,ne,") and text[1].startswith("8,4,64,")
    assert "KERNEL void fused_r_s" in out.read_text()
    assert main(["check", "--levels", "6..8", "--nq", "2,4", "--ne", "2",
                 "--seeds", "1,2"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert sum("PASS" in ln for ln in lines) == 2 * 2 * 2
    assert sum("SKIP" in ln for ln in lines) == 2 * 2  # level 7
