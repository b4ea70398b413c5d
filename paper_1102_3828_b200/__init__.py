"""B200-native IVFADC+R search path of arXiv 1102.3828 ("Searching in one
billion vectors: re-rank with source coding").

The product is libpqrr_b200.so (sm_100a kernels behind the C ABI of
include/pqrr_dev.h); this package is its Python host binding, mirroring the
reference's pqrr C++ API (see ivf.py).  There is no CPU fallback.
"""
from ._lib import DeviceUnavailable, PqrrError, device_count, launch_count  # noqa: F401
from .ivf import (  # noqa: F401
    Codebook, IvfIndex, IvfSearchParams, LookupTable, ProductQuantizer, RefineCodes,
    RefineQuantizer, SearchResult, TrainParams, adc_distance, build_lut, ivf_build,
    ivf_reconstruct, ivf_refine_encode, ivf_refine_train, ivf_rerank, ivf_search,
    ivf_search_batch, ivf_train, kmeans_train, pq_decode, pq_encode, pq_train, synth,
)
from .adc import (  # noqa: F401
    AdcIndex, adc_build, adc_search, adc_search_batch, reconstruct, refine_encode, refine_train,
    rerank, residual,
)
from .storage import (  # noqa: F401
    IndexKind, LoadedAdcIndex, LoadedIvfIndex, load_adc_index, load_codebook, load_ivf_index,
    load_quantizer, probe_index_kind, save_adc_index, save_codebook, save_ivf_index,
    save_quantizer,
)
from .eval import (  # noqa: F401
    GroundTruth, compute_groundtruth, exact_search, groundtruth_synthetic, recall_at_r,
)
from . import adc, eval, ivf, kernels, sharded, storage  # noqa: F401
