"""Seeded synthetic input generators shared by the oracle tests and the product.

This package holds NONE of the method's arithmetic (no gate matrices, no
lowering, no noise sampling, no planning): it only emits circuit descriptions
(gate name, qubits, angles), noise-model parameters, shot counts and seeds in
the shapes of BASELINE.json's five configs.  Both `oracle/` and the CUDA path
consume these descriptions independently.
"""
from .generators import (  # noqa: F401
    GATE_KINDS, Circuit, Workload, qft_gates, basis_prep_gates, brickwork_gates,
    random_3_regular_edges, qaoa_gates, hea_gates, ghz_gates, load_config,
    config_names, make_config, make_variant, monomial_brickwork_gates, random_circuit,
    inverse_qft_gates, qpe_gates, bv_gates,
)
