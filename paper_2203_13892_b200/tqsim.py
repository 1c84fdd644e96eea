"""Thin ctypes binding of include/tqsim.h (argument marshalling only).

Every step of the simulation runs in libtqsim.so (CUDA kernels for sm_100a);
this module only converts Python / numpy arguments to the C structs and back.
There is no CPU fallback: if the library is missing, importing the binding
raises, and GPU entry points return TQSIM_ECUDA without a device.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtqsim.so")

GATE_KINDS = ("x", "y", "z", "h", "s", "sdg", "t", "tdg", "rx", "ry", "rz",
              "p", "u", "cx", "cz", "swap", "cp")
KIND_ID = {k: i for i, k in enumerate(GATE_KINDS)}
MAX_LEVELS = 64

STATUS = {0: "TQSIM_OK", 2: "TQSIM_EINVAL", 3: "TQSIM_ECAPACITY", 4: "TQSIM_ECUDA",
          5: "TQSIM_ENCCL", 6: "TQSIM_EINTERNAL"}


class TqsimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class tqsim_gate(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("q0", C.c_uint32), ("q1", C.c_uint32),
                ("reserved", C.c_uint32), ("theta", C.c_double), ("phi", C.c_double),
                ("lam", C.c_double)]


class tqsim_circuit(C.Structure):
    _fields_ = [("n_qubits", C.c_uint32), ("reserved", C.c_uint32), ("n_gates", C.c_uint64),
                ("gates", C.POINTER(tqsim_gate))]


class tqsim_noise_model(C.Structure):
    _fields_ = [("p1", C.c_double), ("p2", C.c_double), ("readout_p01", C.c_double),
                ("readout_p10", C.c_double), ("amp_damping", C.c_double), ("phase_damping", C.c_double),
                ("t1", C.c_double), ("t2", C.c_double), ("gate_time_1q", C.c_double),
                ("gate_time_2q", C.c_double)]


class tqsim_options(C.Structure):
    _fields_ = [("copy_cost_gates", C.c_double), ("z", C.c_double), ("eps", C.c_double),
                ("mem_budget_bytes", C.c_uint64), ("topup", C.c_uint32),
                ("tile_qubits", C.c_uint32), ("batch_log2_amps", C.c_uint32),
                ("profile", C.c_uint32), ("no_dedup", C.c_uint32), ("trail_low", C.c_uint32),
                ("small_tree", C.c_uint32)]


class tqsim_plan(C.Structure):
    _fields_ = [("n_levels", C.c_uint32), ("n_qubits", C.c_uint32),
                ("arities", C.c_uint32 * MAX_LEVELS), ("boundaries", C.c_uint64 * (MAX_LEVELS + 1)),
                ("first_error_rate", C.c_double), ("predicted_speedup_nodes", C.c_double),
                ("predicted_speedup_gates", C.c_double), ("n_lowered_gates", C.c_uint64),
                ("n_outcomes", C.c_uint64), ("node_executions", C.c_uint64),
                ("gate_amp_updates", C.c_uint64), ("flat_gate_amp_updates", C.c_uint64),
                ("hbm_passes", C.c_uint64), ("tile_qubits", C.c_uint32), ("trail_top_bits", C.c_uint32),
                ("trail_fast", C.c_uint32), ("small_tree", C.c_uint32)]

    @property
    def arity_list(self) -> List[int]:
        return [int(self.arities[i]) for i in range(self.n_levels)]

    @property
    def boundary_list(self) -> List[int]:
        return [int(self.boundaries[i]) for i in range(self.n_levels + 1)]


class tqsim_stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("pass_launches", C.c_uint64),
                ("measure_launches", C.c_uint64), ("node_executions", C.c_uint64),
                ("gate_amp_updates", C.c_uint64), ("pass_bytes", C.c_uint64),
                ("measure_bytes", C.c_uint64), ("pass_ms", C.c_double), ("measure_ms", C.c_double),
                ("leaves", C.c_uint64), ("noise_launches", C.c_uint64), ("noise_ms", C.c_double),
                ("computed_node_executions", C.c_uint64), ("computed_gate_amp_updates", C.c_uint64),
                ("computed_pass_bytes", C.c_uint64)]


class tqsim_pass_timing(C.Structure):
    _fields_ = [("level", C.c_uint32), ("pass_", C.c_uint32), ("states_per_launch", C.c_uint32),
                ("reserved", C.c_uint32), ("launches_per_tree", C.c_double),
                ("ms_per_launch", C.c_double), ("alg_bytes_per_launch", C.c_double)]


class tqsim_kernel_timing(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("level", C.c_uint32), ("pass_", C.c_uint32),
                ("reserved", C.c_uint32), ("launches", C.c_uint64), ("states", C.c_uint64),
                ("computed_states", C.c_uint64), ("ms", C.c_double), ("alg_bytes", C.c_double),
                ("nominal_bytes", C.c_double), ("fp64_per_amp", C.c_double)]


class tqsim_result(C.Structure):
    _fields_ = [("plan", tqsim_plan), ("n_distinct", C.c_uint64),
                ("bitstrings", C.POINTER(C.c_uint64)), ("counts", C.POINTER(C.c_uint64)),
                ("leaf_outcomes", C.POINTER(C.c_uint32)), ("wall_s", C.c_double),
                ("stats", tqsim_stats)]


class tqsim_debug(C.Structure):
    _fields_ = [("n_dumps", C.c_uint32), ("reserved", C.c_uint32),
                ("dump_levels", C.POINTER(C.c_uint32)), ("dump_instances", C.POINTER(C.c_uint64)),
                ("dump_host", C.POINTER(C.c_double)), ("leaf_u", C.POINTER(C.c_double)),
                ("leaf_flagged", C.POINTER(C.c_uint8)), ("leaf_total", C.POINTER(C.c_double))]


class tqsim_op_record(C.Structure):
    _fields_ = [("level", C.c_uint32), ("pass_", C.c_uint32), ("phase", C.c_uint32),
                ("gate", C.c_uint32), ("tile_qubit_mask", C.c_uint64),
                ("reg_qubit_mask", C.c_uint64), ("role", C.c_uint32), ("reserved", C.c_uint32)]


_P = C.POINTER
_SIGS = {
    "tqsim_default_options": (None, [_P(tqsim_options)]),
    "tqsim_last_error": (C.c_char_p, []),
    "tqsim_version": (C.c_char_p, []),
    "tqsim_lower_circuit": (C.c_int, [_P(tqsim_circuit), _P(tqsim_gate), C.c_uint64, _P(C.c_uint64)]),
    "tqsim_profile_passes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                       C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32,
                                       _P(tqsim_pass_timing), C.c_uint64, _P(C.c_uint64)]),
    "tqsim_profile_tree": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                     C.c_void_p, C.c_uint64, C.c_void_p, _P(tqsim_kernel_timing),
                                     C.c_uint64, _P(C.c_uint64)]),
    "tqsim_shard_levels": (C.c_int, [_P(tqsim_plan), C.c_uint32, C.c_uint32, _P(C.c_uint32),
                                     _P(C.c_uint64), _P(C.c_uint64)]),
    "tqsim_parse_qasm": (C.c_int, [C.c_char_p, _P(tqsim_gate), C.c_uint64, _P(C.c_uint64),
                                   _P(C.c_uint32), _P(C.c_uint32)]),
    "tqsim_profile_copy_cost": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, _P(C.c_double),
                                          _P(C.c_double), _P(C.c_double)]),
    "tqsim_plan_circuit": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64,
                                     _P(C.c_uint32), C.c_uint32, _P(tqsim_options), _P(tqsim_plan)]),
    "tqsim_describe_passes": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64,
                                        _P(C.c_uint32), C.c_uint32, _P(tqsim_options),
                                        _P(tqsim_op_record), C.c_uint64, _P(C.c_uint64)]),
    "tqsim_compile_passes": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64,
                                       _P(C.c_uint32), C.c_uint32, _P(tqsim_options),
                                       _P(C.c_uint64), _P(C.c_uint64), _P(C.c_double)]),
    "tqsim_pass_source": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64,
                                    _P(C.c_uint32), C.c_uint32, _P(tqsim_options), C.c_uint32,
                                    C.c_uint32, C.c_char_p, C.c_uint64, _P(C.c_uint64)]),
    "tqsim_shard_range": (C.c_int, [_P(tqsim_plan), C.c_uint32, C.c_uint32, _P(C.c_uint64),
                                    _P(C.c_uint64), _P(C.c_uint64), _P(C.c_uint64)]),
    "tqsim_create": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64,
                               _P(C.c_uint32), C.c_uint32, _P(tqsim_options), _P(C.c_void_p)]),
    "tqsim_get_plan": (C.c_int, [C.c_void_p, _P(tqsim_plan)]),
    "tqsim_get_stats": (C.c_int, [C.c_void_p, _P(tqsim_stats)]),
    "tqsim_destroy": (None, [C.c_void_p]),
    "tqsim_workspace_bytes": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, _P(C.c_uint64)]),
    "tqsim_execute": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p,
                                C.c_void_p, C.c_uint64, C.c_void_p]),
    "tqsim_run": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64, _P(C.c_uint32),
                            C.c_uint32, C.c_uint64, _P(_P(tqsim_result))]),
    "tqsim_run_ex": (C.c_int, [_P(tqsim_circuit), _P(tqsim_noise_model), C.c_uint64,
                               _P(C.c_uint32), C.c_uint32, C.c_uint64, _P(tqsim_options),
                               _P(tqsim_debug), _P(_P(tqsim_result))]),
    "tqsim_result_free": (None, [_P(tqsim_result)]),
    "tqsim_release_run_cache": (None, []),
    "tqsim_debug_philox": (C.c_int, [_P(C.c_uint32), C.c_uint64, _P(C.c_uint32)]),
    "tqsim_debug_noise_table": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                          C.c_uint64, _P(C.c_uint8)]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Load libtqsim.so (fails loudly when the CUDA library was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libtqsim.so not built (run __graft_entry__.build() or "
                              "python -m paper_2203_13892_b200.build): " + LIB_PATH)
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise TqsimError(status, lib().tqsim_last_error().decode())


# ------------------------------------------------------------------ marshalling helpers
class CircuitArg:
    """Keeps the ctypes gate array alive with the tqsim_circuit that points at it."""

    def __init__(self, n_qubits: int, gates: Sequence[Tuple]):
        arr = (tqsim_gate * max(1, len(gates)))()
        for i, g in enumerate(gates):
            kind, a, b, th, ph, la = g
            arr[i] = tqsim_gate(KIND_ID[kind] if isinstance(kind, str) else int(kind), int(a),
                                int(b) if int(b) >= 0 else 0, 0, float(th), float(ph), float(la))
        self.arr = arr
        self.c = tqsim_circuit(int(n_qubits), 0, len(gates), C.cast(arr, C.POINTER(tqsim_gate)))


def noise_arg(p1: float, p2: float, p01: float = 0.0, p10: float = 0.0, amp_damping: float = 0.0,
              phase_damping: float = 0.0, t1: float = 0.0, t2: float = 0.0, gate_time_1q: float = 0.0,
              gate_time_2q: float = 0.0) -> tqsim_noise_model:
    """Depolarizing p1 / p2, readout p01 / p10, and the non-Pauli channels (amplitude / phase
    damping, thermal relaxation T1 / T2 with gate times), 0 = off."""
    return tqsim_noise_model(float(p1), float(p2), float(p01), float(p10), float(amp_damping),
                             float(phase_damping), float(t1), float(t2), float(gate_time_1q),
                             float(gate_time_2q))


def default_options(**kw) -> tqsim_options:
    o = tqsim_options()
    lib().tqsim_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _arities(arities):
    if arities is None:
        return None, 0
    a = (C.c_uint32 * len(arities))(*[int(x) for x in arities])
    return a, len(arities)


# ------------------------------------------------------------------ C-ABI mirrors
def tqsim_version() -> str:
    return lib().tqsim_version().decode()


def tqsim_parse_qasm(text: str):
    """OpenQASM 2.0 subset -> (n_qubits, gates, measured); gates as the tuples CircuitArg
    takes: (kind, q0, q1 or -1, theta, phi, lambda)."""
    b = text.encode()
    n, w, m = C.c_uint64(), C.c_uint32(), C.c_uint32()
    _check(lib().tqsim_parse_qasm(b, None, 0, C.byref(n), C.byref(w), C.byref(m)))
    out = (tqsim_gate * max(1, n.value))()
    _check(lib().tqsim_parse_qasm(b, out, n.value, C.byref(n), C.byref(w), C.byref(m)))
    gates = []
    for i in range(n.value):
        g = out[i]
        kind = GATE_KINDS[g.kind]
        two = kind in ("cx", "cz", "swap", "cp")
        gates.append((kind, int(g.q0), int(g.q1) if two else -1, float(g.theta), float(g.phi), float(g.lam)))
    return int(w.value), gates, bool(m.value)


def tqsim_profile_copy_cost(n_qubits: int, n_probe_gates: int = 64, seed: int = 0):
    """(copy_cost_gates, copy_ms, gate_ms) measured on this GPU."""
    c, cm, gm = C.c_double(), C.c_double(), C.c_double()
    _check(lib().tqsim_profile_copy_cost(int(n_qubits), int(n_probe_gates), int(seed), C.byref(c),
                                         C.byref(cm), C.byref(gm)))
    return c.value, cm.value, gm.value


def tqsim_lower_circuit(n_qubits: int, gates) -> List[Tuple[str, int, int]]:
    ca = CircuitArg(n_qubits, gates)
    n = C.c_uint64()
    _check(lib().tqsim_lower_circuit(C.byref(ca.c), None, 0, C.byref(n)))
    out = (tqsim_gate * max(1, n.value))()
    _check(lib().tqsim_lower_circuit(C.byref(ca.c), out, n.value, C.byref(n)))
    return [(GATE_KINDS[out[i].kind], out[i].q0, out[i].q1) for i in range(n.value)]


def tqsim_plan_circuit(n_qubits, gates, noise: tqsim_noise_model, n_shots: int, arities=None,
                       options: Optional[tqsim_options] = None) -> tqsim_plan:
    ca = CircuitArg(n_qubits, gates)
    a, L = _arities(arities)
    p = tqsim_plan()
    _check(lib().tqsim_plan_circuit(C.byref(ca.c), C.byref(noise), int(n_shots), a, L,
                                    C.byref(options) if options else None, C.byref(p)))
    return p


def tqsim_describe_passes(n_qubits, gates, noise, n_shots, arities=None, options=None):
    ca = CircuitArg(n_qubits, gates)
    a, L = _arities(arities)
    n = C.c_uint64()
    opt = C.byref(options) if options else None
    _check(lib().tqsim_describe_passes(C.byref(ca.c), C.byref(noise), int(n_shots), a, L, opt,
                                       None, 0, C.byref(n)))
    out = (tqsim_op_record * max(1, n.value))()
    _check(lib().tqsim_describe_passes(C.byref(ca.c), C.byref(noise), int(n_shots), a, L, opt,
                                       out, n.value, C.byref(n)))
    return [out[i] for i in range(n.value)]


def tqsim_compile_passes(n_qubits, gates, noise, n_shots, arities=None, options=None):
    """Compile every specialized pass kernel (host-only NVRTC): (kernels, cubin bytes, seconds)."""
    ca = CircuitArg(n_qubits, gates)
    a, L = _arities(arities)
    k, b, s = C.c_uint64(), C.c_uint64(), C.c_double()
    _check(lib().tqsim_compile_passes(C.byref(ca.c), C.byref(noise), int(n_shots), a, L,
                                      C.byref(options) if options else None, C.byref(k),
                                      C.byref(b), C.byref(s)))
    return int(k.value), int(b.value), float(s.value)


def tqsim_pass_source(n_qubits, gates, noise, n_shots, arities=None, options=None, level=0,
                      pass_=0) -> str:
    ca = CircuitArg(n_qubits, gates)
    a, L = _arities(arities)
    n = C.c_uint64()
    opt = C.byref(options) if options else None
    _check(lib().tqsim_pass_source(C.byref(ca.c), C.byref(noise), int(n_shots), a, L, opt, level,
                                   pass_, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().tqsim_pass_source(C.byref(ca.c), C.byref(noise), int(n_shots), a, L, opt, level,
                                   pass_, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def tqsim_shard_range(plan: tqsim_plan, rank: int, world: int) -> Tuple[int, int, int, int]:
    v = [C.c_uint64() for _ in range(4)]
    _check(lib().tqsim_shard_range(C.byref(plan), rank, world, *[C.byref(x) for x in v]))
    return tuple(int(x.value) for x in v)


def tqsim_shard_levels(plan: tqsim_plan, rank: int, world: int):
    """(split_level, lo[], hi[]): the rank's instance range [lo[d], hi[d]) at every level."""
    L = int(plan.n_levels)
    sp = C.c_uint32()
    lo, hi = (C.c_uint64 * L)(), (C.c_uint64 * L)()
    _check(lib().tqsim_shard_levels(C.byref(plan), rank, world, C.byref(sp), lo, hi))
    return int(sp.value), [int(v) for v in lo], [int(v) for v in hi]


class Handle:
    """tqsim_create / tqsim_execute / tqsim_destroy."""

    def __init__(self, n_qubits, gates, noise, n_shots, arities=None, options=None):
        ca = CircuitArg(n_qubits, gates)
        a, L = _arities(arities)
        h = C.c_void_p()
        _check(lib().tqsim_create(C.byref(ca.c), C.byref(noise), int(n_shots), a, L,
                                  C.byref(options) if options else None, C.byref(h)))
        self.h = h

    @property
    def plan(self) -> tqsim_plan:
        p = tqsim_plan()
        _check(lib().tqsim_get_plan(self.h, C.byref(p)))
        return p

    def stats(self) -> tqsim_stats:
        s = tqsim_stats()
        _check(lib().tqsim_get_stats(self.h, C.byref(s)))
        return s

    def workspace_bytes(self, rank: int = 0, world: int = 1) -> int:
        b = C.c_uint64()
        _check(lib().tqsim_workspace_bytes(self.h, rank, world, C.byref(b)))
        return int(b.value)

    def execute(self, seed: int, rank: int, world: int, stream: int, d_workspace: int,
                workspace_bytes: int, d_leaf_outcomes: int) -> None:
        _check(lib().tqsim_execute(self.h, int(seed), rank, world, C.c_void_p(stream),
                                   C.c_void_p(d_workspace), int(workspace_bytes),
                                   C.c_void_p(d_leaf_outcomes)))

    def profile_passes(self, seed: int, rank: int, world: int, stream: int, d_workspace: int,
                       workspace_bytes: int, d_leaf_outcomes: int, reps: int = 5):
        """Live CUDA-event timing of every gate-pass kernel (tqsim_profile_passes)."""
        n = C.c_uint64()
        args = (self.h, int(seed), rank, world, C.c_void_p(stream), C.c_void_p(d_workspace),
                int(workspace_bytes), C.c_void_p(d_leaf_outcomes), int(reps))
        _check(lib().tqsim_profile_passes(*args, None, 0, C.byref(n)))
        out = (tqsim_pass_timing * max(1, n.value))()
        _check(lib().tqsim_profile_passes(*args, out, n.value, C.byref(n)))
        return [out[i] for i in range(n.value)]

    def profile_tree(self, seed: int, rank: int, world: int, stream: int, d_workspace: int,
                     workspace_bytes: int, d_leaf_outcomes: int):
        """In-tree CUDA-event timing of every kernel family (tqsim_profile_tree)."""
        n = C.c_uint64()
        args = (self.h, int(seed), rank, world, C.c_void_p(stream), C.c_void_p(d_workspace),
                int(workspace_bytes), C.c_void_p(d_leaf_outcomes))
        cap = 1024                                   # one tree run (re-run only if it overflows)
        out = (tqsim_kernel_timing * cap)()
        _check(lib().tqsim_profile_tree(*args, out, cap, C.byref(n)))
        if n.value > cap:
            out = (tqsim_kernel_timing * n.value)()
            _check(lib().tqsim_profile_tree(*args, out, n.value, C.byref(n)))
        return [out[i] for i in range(n.value)]

    def noise_table(self, seed: int, level: int, inst_begin: int, count: int) -> np.ndarray:
        p = self.plan
        slen = p.boundaries[level + 1] - p.boundaries[level]
        out = np.zeros(count * slen, dtype=np.uint8)
        _check(lib().tqsim_debug_noise_table(self.h, int(seed), level, inst_begin, count,
                                             out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out.reshape(count, slen)

    def close(self) -> None:
        if self.h:
            lib().tqsim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tqsim_create(*args, **kw) -> Handle:
    return Handle(*args, **kw)


class Result:
    """A run's outcome: the plan, the histogram (`bitstrings`, `counts_array`, ascending;
    `counts` is the same as a dict, built on first access), the leaf-ordered outcomes,
    wall time, run statistics and (debug) dumped states."""

    def __init__(self, plan, bitstrings, counts_array, leaf_outcomes, wall_s, stats, dumps=None,
                 leaf_u=None, leaf_flagged=None, leaf_total=None):
        self.plan = plan
        self.leaf_u = leaf_u                  # debug: per-leaf u53 uniform (R9)
        self.leaf_flagged = leaf_flagged      # debug: draw within 1e-9 of a CDF boundary
        self.leaf_total = leaf_total          # debug: sum |a|^2 as the sampler summed it
        self.bitstrings = bitstrings
        self.counts_array = counts_array
        self.leaf_outcomes = leaf_outcomes
        self.wall_s = wall_s
        self.stats = stats
        self.dumps = dumps
        self._counts = None

    @property
    def counts(self) -> Dict[int, int]:
        if self._counts is None:
            self._counts = dict(zip(self.bitstrings.tolist(), self.counts_array.tolist()))
        return self._counts


def tqsim_run_ex(n_qubits, gates, noise, n_shots, arities=None, seed=0, options=None,
                 dumps: Sequence[Tuple[int, int]] = (), leaf_debug: bool = False) -> Result:
    """tqsim_run with options; `dumps` = [(level, instance)] state dumps (stored-state path);
    leaf_debug=True also returns the per-leaf u53 / flag / total (default path kept)."""
    ca = CircuitArg(n_qubits, gates)
    a, L = _arities(arities)
    dbg = None
    host = None
    lu = lf = lt = None
    if dumps or leaf_debug:
        dbg = tqsim_debug()
    if dumps:
        lv = (C.c_uint32 * len(dumps))(*[int(d) for d, _ in dumps])
        ins = (C.c_uint64 * len(dumps))(*[int(j) for _, j in dumps])
        host = np.zeros((len(dumps), 2 ** n_qubits, 2), dtype=np.float64)
        dbg.n_dumps = len(dumps)
        dbg.dump_levels = C.cast(lv, C.POINTER(C.c_uint32))
        dbg.dump_instances = C.cast(ins, C.POINTER(C.c_uint64))
        dbg.dump_host = host.ctypes.data_as(C.POINTER(C.c_double))
        dbg._keep = (lv, ins)
    if leaf_debug:
        nout = tqsim_plan_circuit(n_qubits, gates, noise, n_shots, arities, options).n_outcomes
        lu = np.zeros(nout, dtype=np.float64)
        lt = np.zeros(nout, dtype=np.float64)
        lf = np.zeros(nout, dtype=np.uint8)
        dbg.leaf_u = lu.ctypes.data_as(C.POINTER(C.c_double))
        dbg.leaf_total = lt.ctypes.data_as(C.POINTER(C.c_double))
        dbg.leaf_flagged = lf.ctypes.data_as(C.POINTER(C.c_uint8))
    r = C.POINTER(tqsim_result)()
    _check(lib().tqsim_run_ex(C.byref(ca.c), C.byref(noise), int(n_shots), a, L, int(seed),
                              C.byref(options) if options else None,
                              C.byref(dbg) if dbg is not None else None, C.byref(r)))
    try:
        res = r.contents
        n = res.plan.n_outcomes
        leaf = np.ctypeslib.as_array(res.leaf_outcomes, shape=(n,)).copy()
        nd = res.n_distinct
        bits = np.ctypeslib.as_array(res.bitstrings, shape=(max(nd, 1),))[:nd].copy()
        cnts = np.ctypeslib.as_array(res.counts, shape=(max(nd, 1),))[:nd].copy()
        plan = tqsim_plan.from_buffer_copy(res.plan)
        stats = tqsim_stats.from_buffer_copy(res.stats)
        wall = float(res.wall_s)
    finally:
        lib().tqsim_result_free(r)
    states = None
    if host is not None:
        states = host[..., 0] + 1j * host[..., 1]
    return Result(plan, bits, cnts, leaf, wall, stats, states, lu,
                  lf.astype(bool) if lf is not None else None, lt)


def tqsim_run(n_qubits, gates, noise, n_shots, arities=None, seed=0) -> Result:
    """The north_star call: returns outcome counts (and the leaf-ordered outcomes).
    `gates` is a gate list or a prebuilt CircuitArg (marshalled once, reused)."""
    ca = gates if isinstance(gates, CircuitArg) else CircuitArg(n_qubits, gates)
    a, L = _arities(arities)
    r = C.POINTER(tqsim_result)()
    _check(lib().tqsim_run(C.byref(ca.c), C.byref(noise), int(n_shots), a, L, int(seed),
                           C.byref(r)))
    try:
        res = r.contents
        n = res.plan.n_outcomes
        leaf = np.ctypeslib.as_array(res.leaf_outcomes, shape=(n,)).copy()
        nd = res.n_distinct
        bits = np.ctypeslib.as_array(res.bitstrings, shape=(max(nd, 1),))[:nd].copy()
        cnts = np.ctypeslib.as_array(res.counts, shape=(max(nd, 1),))[:nd].copy()
        out = Result(tqsim_plan.from_buffer_copy(res.plan), bits, cnts, leaf, float(res.wall_s),
                     tqsim_stats.from_buffer_copy(res.stats))
    finally:
        lib().tqsim_result_free(r)
    return out


def tqsim_release_run_cache() -> None:
    """Free tqsim_run's plan cache, workspace arena and page-locked buffer."""
    lib().tqsim_release_run_cache()


def tqsim_debug_philox(words: np.ndarray) -> np.ndarray:
    """words: (n, 6) uint32 = (c0, c1, c2, c3, k0, k1) -> (n, 4) uint32 via the device Philox."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros((w.shape[0], 4), dtype=np.uint32)
    _check(lib().tqsim_debug_philox(w.ctypes.data_as(C.POINTER(C.c_uint32)), w.shape[0],
                                    out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out


def workload_args(w):
    """(n_qubits, gates, noise, shots, arities) of a workloads.Workload."""
    return (w.circuit.n_qubits, w.circuit.gates,
            noise_arg(w.p1, w.p2, w.readout_p01, w.readout_p10), w.shots, w.arities)
