"""The drop-in model surface (paper_2111_04007_b200/modules.py): CutPoint
placement, the cut-point blocks and ModelSpec the reference's partitioner
consumes (sp/core.py:45-87, sp/partitioner.py:269-374), and the expansion of
a stage map over CutPoint blocks to layers."""

import pytest

from paper_2111_04007_b200 import ConfigError, assign_stages, uniform_profile
from paper_2111_04007_b200.model import CONFIGS, GPT2Stage, StageSpec
from paper_2111_04007_b200.modules import GPT2, CutPoint


def test_cutpoint_placement_and_blocks():
    cfg = CONFIGS["tiny"]
    m = GPT2(cfg)
    assert len(m.cutpoints) == cfg.n_layer - 1
    assert m.cutpoint_blocks() == [[0], [1], [2], [3]]
    m2 = GPT2(cfg, cut_every=2)
    assert m2.cutpoint_blocks() == [[0, 1], [2, 3]]
    m3 = GPT2(CONFIGS["gpt2_355m"], cut_after=[5, 11, 17])
    assert [len(b) for b in m3.cutpoint_blocks()] == [6, 6, 6, 6]
    assert [c.index for c in m3.cutpoints] == [0, 1, 2]
    with pytest.raises(ConfigError):
        GPT2(cfg, cut_after=[3])
    with pytest.raises(RuntimeError):
        m(None)


@pytest.mark.parametrize("name", ["gpt2_355m", "bert_large"])
def test_model_spec_counts_every_parameter(name):
    cfg = CONFIGS[name]
    m = GPT2(cfg, cut_every=3)
    spec = m.model_spec()
    assert spec.num_cutpoints == cfg.n_layer // 3
    # the blocks' parameters add up to the whole model (tied embedding once)
    first = GPT2Stage.memory_plan(cfg, StageSpec(0, 1, tuple(range(cfg.n_layer))), 1)
    # memory_plan counts 128-element padding per tensor: within 0.1 %
    assert abs(sum(spec.cutpoint_parameters) - first["param_count"]) < 1e-3 * first["param_count"]


def test_stage_map_over_blocks_expands_to_layers():
    cfg = CONFIGS["gpt2_355m"]
    m = GPT2(cfg, cut_every=4)
    a = assign_stages(m.model_spec(), 2, 8, uniform_profile(6, 1.0, 2.0, m_grid=(8,)))
    layers = m.layer_stage_map(a.stage_map)
    assert len(layers) == cfg.n_layer and layers[0] == 0 and layers[-1] == 1
    assert sum(c.active for c in m.cutpoints) == 1
    boundary = [i for i in range(1, 24) if layers[i] != layers[i - 1]][0]
    assert boundary % 4 == 0          # the boundary is one of the CutPoints
    with pytest.raises(ConfigError):
        m.layer_stage_map((0,) * 24)
    assert isinstance(m.cutpoints[0], CutPoint) and m.cutpoints[0](3) == 3
