"""attn-verify (paper_2410_18038_b200/verify.py), the GPU port of the reference CLI's
self-check suite (attnsim_cli.cpp:92-190): exit codes and the injected-fault mode."""
import pytest
import torch

from paper_2410_18038_b200 import verify


def test_bad_configuration_exits_2():
    assert verify.main(["--max-m", "0"]) == 2
    assert verify.main(["--tolerance", "-1"]) == 2
    assert verify.main(["--no-such-flag"]) == 2


def test_without_a_device_exits_2():
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    assert verify.main(["--instances", "1"]) == 2


@pytest.mark.gpu
def test_suite_passes_on_the_gpu(capsys):
    assert verify.main(["--instances", "12", "--split-instances", "4", "--causality-instances", "6"]) == 0
    out = capsys.readouterr().out
    for name in ("oracle-equivalence", "split-invariance", "causality"):
        assert name in out
    assert "FAIL" not in out


@pytest.mark.gpu
def test_injected_mask_off_by_one_fails():
    assert verify.main(["--instances", "0", "--split-instances", "0", "--causality-instances", "4",
                        "--inject-mask-off-by-one"]) == 1
