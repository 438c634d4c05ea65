"""Seeded synthetic inputs for the five BASELINE configs.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the CUDA path
(``paper_1907_12933_b200/``).  It holds random draws and the quantisation that *defines* each
synthetic network's exact operands (readings C14-C19 in DESIGN.md); it holds
none of the method's arithmetic (no forward pass, no sign/value/distance predicate, no covering
method, no argmax/property).

Why synthetic: the paper's 5x5 vocalic dataset and trained 25-5-4-5 net (§IV.A)
are not available; MNIST/CIFAR are not in the container either.  The generators below take those
workloads' shapes and value ranges and stand in for them.
"""
from .configs import (  # noqa: F401
    NUM_FP32, NUM_BF16, NUM_Q4_12, NUM_INT8,
    ACT_SIGMOID, ACT_PL_SIGMOID, ACT_RELU,
    PERT_TUPLE_REPLACE, PERT_SUBSET_OFFSET, PERT_SUBSET_REPLACE, PERT_PHILOX_LATTICE, PERT_PHILOX_BOX,
    PERT_PHILOX_CLAMP, cfg4_lattice, eight_bit_bf16,
    PROP_ARGMAX_UNCHANGED, PROP_TARGET_NEVER, PROP_THRESHOLD_LITERAL, PROP_THRESHOLD_LITERAL_ALL,
    Config, Net, Pert, Prop, CovSpec, make_config, CONFIG_IDS,
    f32_to_bf16_bits, bf16_bits_to_f32, vowel_net, pair_images, gamma_config,
)
