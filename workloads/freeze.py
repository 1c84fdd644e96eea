"""Freeze the five BASELINE.json configs to configs/*.json (inputs only).

Run: python -m workloads.freeze
"""
import json
import os

from .generators import _CONFIG_DIR, config_names, make_config


def main() -> None:
    os.makedirs(_CONFIG_DIR, exist_ok=True)
    for name in config_names():
        w = make_config(name)
        with open(os.path.join(_CONFIG_DIR, name + ".json"), "w") as f:
            json.dump(w.to_json(), f, indent=0)
        print(name, w.circuit.n_qubits, len(w.circuit.gates))


if __name__ == "__main__":
    main()
