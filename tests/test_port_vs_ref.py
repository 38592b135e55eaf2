"""The plain-C restatement (oracle/bdis_oracle.c) against the reference itself
(oracle/_ref, the unmodified reference sources) on the cases the GPU parity
tests use: the 16 randomized configurations (gray, RGB, RGBA with holes,
variance on/off) and BASELINE configs 0 and 1 at 640x480 -- every output
bit-identical, so a GPU test that falls back to the port checks the same
thing. CPU only."""
import pytest

from tests.parity import compare_oracles, random_case


@pytest.mark.parametrize("seed", range(16))
def test_randomized_configs_port_equals_reference(port, ref, seed):
    import paper_2205_03133_b200 as P

    cfg, l, r = random_case(P, seed)
    compare_oracles(port, ref, cfg, l, r)


@pytest.mark.parametrize("config", [0, 1])
def test_baseline_configs_port_equals_reference(port, ref, config):
    import paper_2205_03133_b200 as P

    l, r = P.synth_pair(config)
    compare_oracles(port, ref, P.PipelineConfig.baseline(config), l, r)
