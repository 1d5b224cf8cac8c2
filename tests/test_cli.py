"""CLI argument handling and exit codes, mirroring the reference's tests/test_cli.py:186-240
(usage errors exit 1, the dilated splitting and non-tiling steps are rejected before any device
work).  Runs on the CPU: every case fails in the parser or in the argument checks."""

from paper_1403_3511_b200.cli import EXIT_USAGE, main


def run(argv, capsys):
    code = main(argv)
    out = capsys.readouterr()
    return code, out.out, out.err


def test_usage_errors_exit_one(capsys):
    cases = [[], ["frobnicate"], ["bench", "--kmax", "abc"], ["bench", "--kmax", ""], ["bench", "--kmax=-4"],
             ["propagate", "--h", "0"], ["propagate", "--h", "nonsense"], ["propagate", "--h", "1/0"],
             ["propagate", "--scheme", "euler"], ["bench", "--jobs", "0"], ["rederr", "--dims", "0"]]
    for argv in cases:
        code, _, _ = run(argv, capsys)
        assert code == EXIT_USAGE, argv


def test_dilated_splitting_is_rejected(capsys):
    code, _, err = run(["propagate", "--kmax", "6", "--scale", "2"], capsys)
    assert code == EXIT_USAGE and "--scale must be 1" in err


def test_steps_must_tile_the_interval(capsys):
    code, _, err = run(["propagate", "--kmax", "6", "--degree", "3", "--h", "2/5"], capsys)
    assert code == EXIT_USAGE and "does not divide" in err
