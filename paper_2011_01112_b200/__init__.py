"""B200-native batched confidence-maximising depth assignment (arXiv 2011.01112).

Thin Python binding over the C ABI of ``include/ic_sched.h`` (library
``libicsched.so`` built from ``csrc/`` for sm_100a).  This module only
marshals arguments: every step of the solve runs in the CUDA kernels.  There
is no CPU fallback — if the library is missing, importing the binding raises.

    from paper_2011_01112_b200 import Scheduler, SchedConfig
    with Scheduler(SchedConfig(max_tasks=64, max_opt_stages=8, max_horizon=4096,
                               epsilon_micro=100_000)) as s:
        out = s.solve_batch(inputs)          # dict of CUDA tensors (ABI layout)

Names follow the ABI: ``ic_sched_create / ic_sched_solve_batch /
ic_sched_solve_batch_host / ic_sched_destroy``.
"""
from .abi import (  # noqa: F401
    IC_OK, IC_ERR_INVALID_ARG, IC_ERR_LIMIT, IC_ERR_CUDA, IC_ERR_OOM,
    IC_DROP_ALLOWED, IC_MANDATORY_ENFORCED,
    IC_INST_OK, IC_INST_INFEASIBLE, IC_INST_BAD_INPUT, IC_INST_LIMIT,
    IC_UTIL_GIVEN, IC_UTIL_MAX, IC_UTIL_EXP, IC_UTIL_LIN,
    INPUT_FIELDS, OUTPUT_FIELDS, STATS_FIELDS,
    SchedConfig, SchedInfo, SchedTuning, TUNING_FIELDS, Scheduler, use_library, ICSchedError, lib_path, load_library,
    alloc_inputs, alloc_outputs, gen_batch_device,
    IC_SIM_PLANNER, IC_SIM_EDF, IC_SIM_LCF, IC_SIM_RR, IC_SIM_UTIL_EXP, IC_SIM_UTIL_ORACLE,
    SimConfig, SimResult, simulate, probe_smem, to_micro, confidences_to_inputs,
)
