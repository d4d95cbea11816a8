"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic: only model shapes,
round parameters and the generators of prompts and response-length traces
(DESIGN.md §4 "input recipe").  Both ``oracle/`` and
``paper_2509_21009_b200/`` (through tests and bench) consume what it
produces; neither imports the other.
"""
from .configs import MODELS, ROUNDS, model_config  # noqa: F401
from .gen import prompts, length_trace, trace_for_round  # noqa: F401
