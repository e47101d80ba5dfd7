#!/usr/bin/env python3
"""Experiment: build libdsft_spec.so (-DDSFT_K2_SPEC: compile-time K2 for the headline primes)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1706_02740_b200 import build as b
b.build(force=True, defines=("DSFT_K2_SPEC",), out=os.path.join(ROOT, "paper_1706_02740_b200", "libdsft_spec.so"))
