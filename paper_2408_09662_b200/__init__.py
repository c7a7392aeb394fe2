"""paper_2408_09662_b200 -- B200-native batched evaluation of instruction tapes.

Drop-in for the CPU batched evaluator of the reference (``vecsym.batchrt``
over ``vecsym._kernels.run_range``): the same ``BatchWorkspace`` /
``batch_eval`` / ``serial_eval`` surface and ``"vecsym-tape"`` v1 ingest,
executed by generated sm_100a kernels (NVRTC) behind the C ABI in
``include/vsb200.h``.  ``Function`` adds the torch tensor interface.
"""

from .batchrt import BatchPipeline, BatchWorkspace, batch_eval, default_thread_count, serial_eval
from .hoist import InvariantSplit, split_invariant
from .plan import Plan, clear_plan_cache, get_plan
from .tape import (
    FORMAT_VERSION,
    InstructionTape,
    OpCode,
    Sparsity,
    arity,
    as_tape,
    deserialize,
    load,
    save,
    serialize,
)

__all__ = [
    "BatchWorkspace", "batch_eval", "serial_eval", "default_thread_count", "BatchPipeline",
    "Plan", "get_plan", "clear_plan_cache",
    "InstructionTape", "OpCode", "Sparsity", "arity", "as_tape", "deserialize", "serialize", "load", "save",
    "FORMAT_VERSION", "Function", "split_invariant", "InvariantSplit",
]

__version__ = "0.1.0"


def __getattr__(name):
    # torch is imported lazily: the reference-shaped API works without it
    if name == "Function":
        from .function import Function

        return Function
    raise AttributeError(name)
