"""B200-native Radar-STDA inference engine (drop-in for the reference `stda` model API).

Reference: arXiv 2307.09063, `/root/reference/pkg/stda/src/stda/__init__.py:10-27`.
The model surface (`StdaConfig`, `StdaNet`, blocks, `concat_frames`,
`parameter_count`, `load_checkpoint`) mirrors the reference; eval-mode forwards run
hand-written sm_100a kernels through the C ABI in `include/stda_b200.h`.
"""

__version__ = "0.1.0"

from .model import (  # noqa: F401
    EcaBlock,
    MobileDecoderBlock,
    MobileEncoderBlock,
    StdaConfig,
    StdaNet,
    concat_frames,
    load_checkpoint,
    parameter_count,
)
from .fold import fold_state_dict  # noqa: F401
# batched inference driver and its data formats (reference
# denoise.py, data.py, rdc1.py)
from .data import ManifestInfo, NormStats, TripletDataset, load_manifest  # noqa: F401
from .denoise import denoise_dataset  # noqa: F401
from .rdc1 import read_cube, write_magnitude_cube  # noqa: F401
# the paper's baselines behind the same forward boundary
from .baselines import BASELINE_KINDS, BaselineCae, BaselineMlp, baseline_forward, build_baseline  # noqa: F401
