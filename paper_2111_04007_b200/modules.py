"""The drop-in model surface: a GPT-2 / BERT described as an ``nn.Module``
whose ``CutPoint`` markers are the candidate pipeline boundaries, as in
Varuna (the user inserts CutPoints into the model
definition; the partitioner activates a subset of them as stage boundaries).

    model = GPT2(CONFIGS["gpt2_355m"])                 # a CutPoint after every layer
    model = GPT2(cfg, cut_every=2)                      # ... after every second layer
    model = GPT2(cfg, cut_after=[5, 11, 17])            # ... after chosen layers
    spec = model.model_spec()                           # ModelSpec over the CutPoint blocks
    a = assign_stages(spec, P, m, profile)              # sp/partitioner.py:269-374
    v = Varuna(model, ParallelConfig(P, D, m, N, a.stage_map))

The module is a STRUCTURE (layer order, CutPoint placement, hyper-
parameters), not a container of weights: Varuna instantiates only this
rank's stage, with its parameters in the executor's flat HBM buffers and its
math in the sm_100a kernels (there is no CPU or autograd path). CutPoint is
an identity in ``forward`` on a structure, and records whether the stage
map made it an active boundary.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from .core import ConfigError, ModelSpec
from .model import GPT2Config


class CutPoint(torch.nn.Module):
    """A candidate pipeline boundary. Identity in the
    forward pass; ``active`` is set by Varuna when the stage map places a
    stage boundary here (a pass-through otherwise)."""

    def __init__(self):
        super().__init__()
        self.index = -1       # position among the model's CutPoints
        self.active = False

    def forward(self, x):
        return x

    def extra_repr(self) -> str:
        return f"index={self.index}, active={self.active}"


class TransformerLayer(torch.nn.Module):
    """Descriptor of transformer layer ``index`` of the model (pre-LN GPT-2
    or post-LN BERT per the config); its weights live in the executor."""

    def __init__(self, index: int):
        super().__init__()
        self.index = index

    def extra_repr(self) -> str:
        return f"index={self.index}"


class GPT2(torch.nn.Module):
    """Structure of a GPT-2 (or BERT, ``cfg.arch == "bert"``): embedding,
    ``cfg.n_layer`` transformer layers with CutPoints between them, head."""

    def __init__(self, cfg: GPT2Config, cut_every: int = 1,
                 cut_after: Optional[Sequence[int]] = None):
        super().__init__()
        self.cfg = cfg
        L = cfg.n_layer
        if cut_after is None:
            if cut_every < 1:
                raise ConfigError("GPT2: cut_every must be >= 1")
            cut_after = [li for li in range(L - 1) if (li + 1) % cut_every == 0]
        cut_after = sorted(set(int(c) for c in cut_after))
        if any(c < 0 or c >= L - 1 for c in cut_after):
            raise ConfigError(f"GPT2: CutPoints go after layers 0..{L - 2}")
        self.body = torch.nn.ModuleList()
        k = 0
        for li in range(L):
            self.body.append(TransformerLayer(li))
            if li in cut_after:
                cp = CutPoint()
                cp.index = k
                k += 1
                self.body.append(cp)

    @property
    def cutpoints(self) -> List[CutPoint]:
        return [m for m in self.body if isinstance(m, CutPoint)]

    def cutpoint_blocks(self) -> List[List[int]]:
        """Layer indices of the K = #CutPoints + 1 blocks the CutPoints
        delimit (the reference's cut-point units, sp/core.py:45-87)."""
        blocks, cur = [], []
        for mod in self.body:
            if isinstance(mod, CutPoint):
                blocks.append(cur)
                cur = []
            else:
                cur.append(mod.index)
        blocks.append(cur)
        return blocks

    def model_spec(self, name: Optional[str] = None) -> ModelSpec:
        """ModelSpec over the CutPoint blocks: parameters per block (layers;
        the embedding with the first block, the final norm / head with the
        last, the tied embedding once) and the boundary activation h*s*2
        bytes per example — the input of assign_stages / memory_check."""
        cfg = self.cfg
        h, V, S = cfg.hidden, cfg.vocab_size, cfg.seq_len
        blocks = self.cutpoint_blocks()
        params = [len(b) * cfg.layer_param_count() for b in blocks]
        params[0] += V * h + S * h + (cfg.type_vocab * h + 2 * h if cfg.arch == "bert" else 0)
        params[-1] += (h * h + 3 * h + V) if cfg.arch == "bert" else 2 * h
        return ModelSpec(name or f"{cfg.arch}-L{cfg.n_layer}-h{h}", tuple(params),
                         (h * S * 2,) * len(blocks))

    def layer_stage_map(self, stage_map: Sequence[int]) -> tuple:
        """Per-layer stage of a stage map over the CutPoint blocks; marks the
        CutPoints the map activates."""
        blocks = self.cutpoint_blocks()
        if len(stage_map) != len(blocks):
            raise ConfigError(f"stage_map covers {len(stage_map)} cut-point blocks, the model "
                              f"has {len(blocks)} ({len(self.cutpoints)} CutPoints)")
        for cp, (a, b) in zip(self.cutpoints, zip(stage_map, stage_map[1:])):
            cp.active = a != b
        out = []
        for s, blk in zip(stage_map, blocks):
            out += [s] * len(blk)
        return tuple(out)

    def forward(self, x):
        raise RuntimeError("GPT2 is a model structure; run it with Varuna(model, config).step")
