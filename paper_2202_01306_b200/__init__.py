"""paper_2202_01306_b200 -- B200-native runtime for Harmony's swap-aware
layer-pack training (arXiv 2202.01306).

Planner API (drop-in for the reference `wrapsched` hot path):
``Configuration``, ``MachineModel``, ``ProfileSet``, ``balanced_time_pack``,
``generate_task_graph``, ``unroll_schedule``, ``simulate`` / ``SimReport``,
``search``.  Runtime: ``execute`` runs the same task graph on the GPU through
the native extension (swap engine + sm_100a kernels + fused Adam) and
returns a ``SimReport`` built from measured CUDA events whose ledger equals
``simulate``'s.
"""

from .core import (Configuration, LayerChain, LayerNode, MachineModel, Mode, TensorKind,
                   gpu_shares, microbatch_groups, serialize_graph)
from .errors import *  # noqa: F401,F403
from .packing import PackPlan, balanced_time_pack, greedy_maxpack_baseline
from .profiler import (AffineModel, ProfileSample, ProfileSet, SynthSpec, fit_profiles,
                       slow_start_max_u, synth_profiles, synth_samples)
from .taskgraph import (Channel, ChannelKind, Task, TaskGraph, TaskType, generate_task_graph,
                        unroll_schedule)
from .simulator import SimReport, TraceEvent, simulate

__version__ = "0.1.0"


def __getattr__(name):
    # heavy modules (numpy model, runtime, search) load lazily
    if name in ("execute", "Runtime", "HarmonyRuntime"):
        from . import runtime
        return getattr(runtime, name)
    if name in ("GPTSpec", "gpt_profiles", "gpt_machine"):
        from . import model
        return getattr(model, name)
    if name in ("search", "SearchSpec", "SearchResult", "Strategy", "greedy_baseline"):
        from . import search as _s
        return getattr(_s, name)
    raise AttributeError(name)
