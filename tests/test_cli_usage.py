"""CPU: CLI argument handling and usage exit codes (cli.cpp:306-316; test_cli.cpp usage cases)."""
from paper_2108_13162_b200.cli import main


def test_usage_errors_exit_1():
    assert main(["solve"]) == 1
    assert main(["nosuchcommand"]) == 1
    assert main([]) == 1
    assert main(["solve", "x.mtx", "--method", "qmr"]) == 1
    assert main(["spmv-bench", "x.mtx", "--block-size", "100"]) == 1


def test_version(capsys):
    assert main(["--version"]) == 0
    assert capsys.readouterr().out.strip() == "0.1.0"
