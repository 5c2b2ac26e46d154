"""B200-native RNS-CKKS evaluator for the Volley Revolver column-ciphertext
HE-matmul / HE-conv path (arXiv 2512.18646), a drop-in for packedhe's
SlotEngine + multicipher + poly_activation API.

Compute runs in hand-written sm_100a kernels (libvrhe.so, C-ABI in
include/vrhe.h); this package is the host-side mirror of the reference
interface.  There is no CPU fallback.
"""

from .errors import CapacityError, EngineError, LayoutError
from .params import EngineParams, config_params, gen_primes, is_pow2, next_pow2
from .engine import Ciphertext, CkksEngine, DecodeFuture, OpMeter, PlainMask, SlotEngine
from .encoding import (
    Encoding,
    Kernel,
    MatrixShape,
    PackedMatrix,
    encode_db,
    encode_revolver,
    encode_row_major,
    incomplete_col_shift,
    matrix_from_csv,
    row_shift,
    sum_col_vec,
    sum_row_vec,
)
from .matmul import MatmulPlan, build_result_filter, matmul, matmul_tiled, row_shifter
from .multicipher import (
    ColumnEncodedImage,
    ColumnEncodedMatrix,
    conv_columns,
    conv_columns_multi,
    encode_image_columns,
    encode_left,
    encode_right,
    matmul_outer,
    matmul_outer_blocks,
    matmul_outer_many,
    pad_images,
    reassemble_columns,
)
from .conv import ImageShape, KernelSpan, build_offset_filter, conv, kernel_spanner, sum_for_conv
from .virtual import VirtualLayout, batched_conv, reform, tile_kernel_span, vadd, vmul, vrot
from .pipeline import (
    PIPELINE_DEPTH,
    BatchPlan,
    ChunkedDataset,
    EncodedModel,
    ModelWeights,
    activation_constants,
    argmax_decide,
    encode_model,
    fc_layer,
    flatten_maps,
    forward,
    forward_encoded,
    pack_batch,
    poly_activation,
    poly_activation_batch,
)

from .serial import SerialError, load_batch, load_ciphertext, load_model, read_ciphertext, write_batch, write_ciphertext, write_model

__version__ = "0.1.0"
