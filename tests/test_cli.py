"""CLI host-side behaviour, no GPU: option precedence
(flag > config file > default), config-file errors and usage errors map to
exit code 2, like the reference's fmmkit command (src/cli.py)."""

import argparse

import pytest

from paper_1209_3516_b200 import cli


def _opts(argv):
    return cli.settings(cli.parser().parse_args(argv))


def test_precedence_flag_over_file_over_default(tmp_path):
    cfg = tmp_path / "opts.cfg"
    cfg.write_text("# comment\np = 6\ntheta=0.45  # trailing\nuse-rsqrt = yes\nprecision = fp32\n")
    o = _opts(["run", "--config", str(cfg), "--p", "5"])
    assert o.p == 5 and o.theta == 0.45 and o.use_rsqrt is True and o.precision == "fp32"
    assert o.ncrit == 30 and o.strategy == "dualtree"


@pytest.mark.parametrize("text", ["bogus = 1\n", "p\n", "mutual = maybe\n", "strategy = fast\n"])
def test_bad_config_files_exit_2(tmp_path, text, capsys):
    cfg = tmp_path / "bad.cfg"
    cfg.write_text(text)
    assert cli.main(["scaling", "--config", str(cfg), "--n-list", "10"]) == 2
    assert "error" in capsys.readouterr().err


def test_usage_errors_exit_2(capsys):
    assert cli.main(["scaling", "--n-list=-3,10", "--mutual"]) == 2
    assert cli.main(["run", "--n", "0"]) == 2
    assert cli.main(["run", "--input", "/nonexistent.csv"]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["run", "--strategy", "fast"])
    assert e.value.code == 2
    with pytest.raises(SystemExit):
        cli.main([])


def test_list_parsing():
    assert cli.split_list("1e3, 2000,", int, "n") == [1000, 2000]
    with pytest.raises(cli.CliError):
        cli.split_list("a,b", float, "target")
    with pytest.raises(cli.CliError):
        cli.split_list(" , ", int, "n")


def test_option_table_drives_parser_and_config():
    """Every option of the table is a flag of exactly the commands that
    take it, and a config-file key of the same name."""
    ap = cli.parser()
    sub = next(a for a in ap._actions if isinstance(a, argparse._SubParsersAction))
    for cmd, sp in sub.choices.items():
        flags = {a.dest for a in sp._actions if a.option_strings} - {"help", "config"}
        assert flags == {o.key for o in cli.OPTIONS if cmd in o.commands}, cmd
    assert set(cli.BY_KEY) == {o.key for o in cli.OPTIONS}
