"""Seeded synthetic workload tooling (L0): circuit generator, network builder, planner.

This package produces the plan JSON that both the CUDA library (``tn_plan_load``) and the oracle
read.  It is input generation, not the product path and not the oracle.
"""
