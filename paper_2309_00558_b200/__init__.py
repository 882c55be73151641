"""B200-native batched FaST-GShare simulator (arXiv 2309.00558 reference path).

Drop-in for the reference's ``gshare_sim.run`` / ``compare_policies``
(pkg/src/gshare_sim/sim_engine.py:601-612): the same ``Scenario`` in, the
same ``MetricsReport`` out, bit-exact -- but every run of a batch executes
inside one hand-written sm_100a CUDA kernel (``csrc/``) reached through the
C ABI in ``include/gshare_b200.h``.  There is no CPU fallback.
"""
from .errors import (BackendUnavailableError, CapacityError, ConflictError, GShareError,
                     InvariantError, MissingConfigurationError, ParseError, ValidationError)
from .memory import DEFAULT_GPU_MEMORY_MB, MemorySpec
from .metrics import FunctionWindowRow, GlobalWindowRow, GpuWindowRow, MetricsReport
from .profiles import (ConfigPoint, FunctionProfile, ProfileEntry, grid_points,
                       ingest_profile, ingest_profiles, rps_per_resource,
                       serialize_profile, serialize_profiles, synth_profile, throughput_at)
from .scenario import (POLICIES, FunctionSpec, InitialPod, Request, Scenario, latency_of,
                       violates_slo)
from .traces import (WorkloadTrace, constant_trace, explicit_trace, replay_trace,
                     sinusoid_trace, step_trace)
from .engine import RunResult, compare_policies, run, run_batch

__version__ = "0.1.0"
