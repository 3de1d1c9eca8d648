"""synth — seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds the counter-based random generator (C, ``csrc/synth.c``) and the model
*descriptions* (layer tables: ops, tensor shapes, activation slots) of the
paper's workload classes.  It contains none of the method's arithmetic: no
forward-pass math, no swapping, no device layout.  See DESIGN.md, "Input recipe".
"""
from .models import (  # noqa: F401
    ModelSpec, Tensor, Slot, Layer, Op, Act, Rule,
    mlp, bert, gpt2, resnet50, resnet_tiny, build_model, CONFIGS,
)
