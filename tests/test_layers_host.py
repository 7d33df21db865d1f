"""Layer-stack host logic (CPU): the network grammar, presets and shape walk
mirror layers.hpp:182-348, checked against the reference itself where the
oracle library is available."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import ConfigError, layers


def test_presets_shapes():
    small = layers.preset_network("reference-net-small")
    assert small.default_batch == 8 and small.input_maps == 3 and small.input_image == 32
    sh = small.shape()
    assert (sh.conv_count, sh.final_maps, sh.final_size, sh.fc_inputs, sh.fc_outputs) == (5, 48, 7, 2352, 1000)
    big = layers.preset_network("reference-net")
    sh = big.shape()
    assert big.default_batch == 128
    assert (sh.conv_count, sh.final_maps, sh.final_size, sh.fc_inputs) == (5, 384, 7, 18816)


@pytest.mark.parametrize("text", [
    "relu\nconv 3 8 1 1\n",                 # first stage must be a convolution
    "conv 3 8 1 2\nconv 3 8 3 2\n",         # map chaining
    "conv 2 8 1 2\npool\n",                 # odd plane size before pool (n'=7)
    "conv 3 8 1 2\nfc 10\nrelu\n",          # fc must be last
    "conv 9 8 1 2\n",                       # kernel larger than image
])
def test_invalid_networks_raise_config_error(text):
    with pytest.raises(ConfigError):
        layers.parse_network(text)


@pytest.mark.parametrize("text", ["conv 3 8 1\n", "conv 3 8 1 2 7\n", "conv 0 8 1 2\n", "blob\n", "# only a comment\n"])
def test_parse_errors(text):
    with pytest.raises(ConfigError):
        layers.parse_network(text)


def test_comments_and_blank_lines():
    spec = layers.parse_network("\n# net\nconv 3 8 2 4  # first\n\nrelu\npool # half\nfc 5\n")
    assert [s.kind for s in spec.stages] == [layers.StageKind.conv, layers.StageKind.relu, layers.StageKind.pool,
                                              layers.StageKind.fc]
    assert spec.shape().fc_inputs == 4 * 3 * 3


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("records", [
    [(0, 3, 8, 1, 2), (0, 3, 8, 3, 2)],
    [(0, 2, 8, 1, 2), (2, 0, 0, 0, 0)],
    [(0, 3, 8, 1, 2), (3, 0, 0, 0, 10), (1, 0, 0, 0, 0)],
])
def test_reference_rejects_the_same_networks(records):
    """NetworkSpec::validate of the reference raises config_error (code 3) too."""
    with pytest.raises(oracle.OracleError) as ei:
        oracle.ref_run_iteration(records, 2, 1, engine=1)
    assert ei.value.code == 3


def test_init_params_streams():
    spec = layers.preset_network("reference-net-small")
    p = layers.init_params(spec, 1234)
    assert [w.shape for w in p.conv] == [(12, 3, 11, 11), (32, 12, 7, 7), (48, 32, 5, 5), (48, 48, 5, 5),
                                         (48, 48, 3, 3)]
    # layer ci draws from stream ci of the weights role (rng.hpp:41-47, layers.hpp:364)
    from paper_1312_5851_b200.rng import uniform_at
    r = 2 | (1 << 8)
    assert p.conv[1].reshape(-1)[5] == np.float32(uniform_at(1234, r, 5))
    assert p.fc_weights.shape == (1000, 2352) and p.fc_bias.shape == (1000,)
