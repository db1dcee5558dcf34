"""B200-native (sm_100a) layer-parallel FAS multigrid for deep residual networks.

A drop-in for the hot path of the reference package `layermg` (arXiv 2007.07336): the same
public names and semantics (`random_network`, `build_hierarchy`, `solve`, `mg_cycle`, the
relaxation sweeps, `compute_residual`, `loss_and_grad`, `train_epoch`, ...), computed by
hand-written FP64 CUDA kernels in the in-tree C-ABI library liblmg.so.  There is no CPU path:
every numeric call runs on the GPU and raises if the library or device is missing.
"""

from .errors import ConfigurationError, DimensionError, IdxParseError, LmgCudaError, ProtocolError
from .kernels import (
    TransformParams,
    apply_transform,
    conv2d_params,
    dense_params,
    l2_norm,
    transform_vjp,
)
from .multigrid import (
    BatchReport,
    CycleReport,
    MgHierarchy,
    MgLevel,
    assemble_coarse_source,
    build_hierarchy,
    c_relaxation,
    compute_residual,
    f_relaxation,
    fcf_relaxation,
    initial_guess,
    mg_cycle,
    restrict_states,
    solve,
    solve_forward,
)
from .network import (
    DeviceNet,
    DeviceStack,
    ResidualNetwork,
    forward_logits,
    load_network,
    output_state,
    propagate_values,
    propagation_operator,
    readout_logits,
    save_network,
    sequential_forward,
    source_from_input,
)
from .parallel import (
    BlockPartition,
    BoundaryMessage,
    ExchangeTracker,
    decode_message,
    encode_message,
    exchange_and_c_relax,
    make_partition,
    parallel_f_relax,
    wire_roundtrip_transport,
)
from .synthetic import device_network, random_batch, random_network, random_sample
from .training import (
    Dataset,
    DeviceTrainer,
    EpochStats,
    Gradients,
    TrainConfig,
    backward,
    evaluate,
    loss_and_grad,
    sgd_update,
    train_epoch,
)

__version__ = "0.1.0"
