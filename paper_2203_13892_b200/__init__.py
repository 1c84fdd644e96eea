"""B200-native TQSim hot path: tree-based multi-shot noisy statevector
simulation (arXiv 2203.13892) behind the C ABI in include/tqsim.h.

The compute path is libtqsim.so (hand-written sm_100a CUDA kernels + a C++
tree scheduler); `tqsim` is its ctypes binding.  This package never imports the
test oracle.
"""
from . import tqsim  # noqa: F401
from .tqsim import (Handle, Result, TqsimError, default_options, noise_arg, tqsim_create,  # noqa: F401
                    tqsim_debug_philox, tqsim_describe_passes, tqsim_lower_circuit,
                    tqsim_plan_circuit, tqsim_run, tqsim_run_ex, tqsim_shard_range,
                    workload_args)
