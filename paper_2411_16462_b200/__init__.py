"""B200-native Lion Cub distributed optimizer step (arXiv 2411.16462).

Drop-in for the hot path of the reference package ``lioncomm``: the same
optimizer / collective API over CUDA tensors, executed by sm_100a kernels
(``csrc/``, C ABI in ``include/lioncub.h``) and NCCL over NVLink.
"""

from .collectives import (Topology, VoteResult, allreduce_mean_f32,  # noqa: F401
                          allgather_f64, choose_lane_bits, compressed_allreduce_1bit,
                          direct_allreduce, field_bits, majority_sign,
                          ps_gather_broadcast, run_ranks)
from .errors import (CapacityError, CollectiveError, ConfigError,  # noqa: F401
                     DeviceError, LionCommError, PackFormatError,
                     PackRangeError)
from .optimizer import (VOTE_ALGOS, FlatParamSet, Layout, LionHyper,  # noqa: F401
                        StepGraph, SyncPolicy, WorkerState, distributed_lion_step,
                        distributed_lion_step_host, divergence_from_momenta,
                        momentum_divergence, signsgd_majority_step,
                        hash_params, lion_step, load_checkpoint,
                        maybe_sync_momentum, save_checkpoint, vote_agreement)
from .quant import (INF, PackedBits, QuantSpec, SignPolicy, apply_sign,  # noqa: F401
                    dequantize, lp_mean_norm, pack, quantize, unpack)
from .torch_optim import LionCub, lioncub_comm_hook  # noqa: F401
from .frames import NcclFrameTransport  # noqa: F401
from .transport import (DeviceTransport, LocalTransport,  # noqa: F401
                        NcclTransport)

__version__ = "0.1.0"
