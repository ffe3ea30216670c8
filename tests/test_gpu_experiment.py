"""The experiment harness on the GPU engine (every Simulation::run is a
device of a colo_replay_colocated fleet; TPT samples sorted on the device):
`run` in all three modes and `compare` produce files byte-identical to the
reference CLI's (tests/golden/cli/expected.json)."""
import pytest

from paper_2503_01066_b200 import colosim as cs
from paper_2503_01066_b200 import experiment as ex

from experiment_check import run_all, run_cli_profile

pytestmark = pytest.mark.gpu


def test_harness_outputs_match_reference_cli_gpu(tmp_path):
    run_all(ex.GpuEngine(cs.Context(0)), str(tmp_path))


def test_cli_profile_matches_reference_cli(tmp_path):
    run_cli_profile(str(tmp_path))
