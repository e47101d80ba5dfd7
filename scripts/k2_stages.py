#!/usr/bin/env python3
"""Print the K2 stage layout (radices, twiddle-free mask, Good-Thomas dimensions) of
the bucket primes for the BASELINE configs (needs a GPU: plans upload tables)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_02740_b200 as d
for N,s in ((2**26,1000),(2**26,2000),(2**26,4000),(2**22,50),(6000011,100),(2**24,256),(4096,8)):
    p=d.Plan(N,s)
    print(N,s,[(P,)+p.dsft_plan_k2_stages(t) for t,P in enumerate(p.primes())], p.dsft_plan_k2_specialized())
