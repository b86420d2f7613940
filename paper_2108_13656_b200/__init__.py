"""B200-native warm/cool colour-temperature decolorization (arXiv 2108.13656).

Drop-in for the hot path of the reference package ``warmgray``
(/root/reference/pkg/src/warmgray/__init__.py): the same public names for
decolorization and global tone mapping, with every image computed by
hand-written sm_100a CUDA kernels behind a C ABI (include/warmgray_b200.h).

    import paper_2108_13656_b200 as warmgray
    gray = warmgray.decolor_image(warmgray.PlanarImage(rgb))          # bit-identical fp64
    toned_rgb, toned = warmgray.tonemap_image(img, mode="global")

Throughput API on device-resident batches (torch CUDA tensors):
``decolor``, ``decolor_tone``, ``hdr_tonemap`` (module :mod:`.batch`).
"""

from .backend import (
    THREADS_ENV,
    active_backend,
    available_backends,
    compiled_available,
    get_device,
    set_device,
)
from .batch import (
    HdrScratch,
    decolor,
    decolor_host,
    decolor_tone,
    decolor_tone_host,
    decolor_tone_local,
    decolor_tone_local_host,
    hdr_tonemap,
    hdr_tonemap_host,
    lab,
    luma,
    luma_host,
    sigmoid,
)
from .codec import (
    CodecError,
    decolor_files,
    dequantize_u8,
    load_image,
    load_u8,
    quantize_u8,
    read_batch,
    read_pnm_batch,
    save_image,
    save_u8,
    write_batch,
    write_pnm_batch,
)
from .perf import BenchResult, format_table, run_benchmark
from .colorspaces import (
    METHOD_NAMES,
    LabColor,
    delta_e76,
    hsv_v,
    lab_image,
    lab_lightness,
    luma_weighted,
    luminance_image,
    rgb_to_lab,
)
from .metrics import (
    TAU_SWEEP,
    MetricReport,
    PairSampleConfig,
    TauScore,
    ccfr,
    ccpr,
    escore,
    evaluate,
    write_sweep_csv,
)
from .core import (
    DEFAULT_PARAMS,
    DecolorParams,
    PlanarImage,
    RgbPixel,
    blue_luminance,
    cool_luminance,
    decolor_image,
    decolor_pixel,
    red_green_luminance,
    warm_luminance,
    white_luminance,
)
from .tonemap import (
    LocalHistogramGrid,
    SigmoidCurve,
    apply_local_lhe,
    apply_sigmoid,
    reinstate_color,
    tonemap_image,
)

__version__ = "0.1.0"

__all__ = [
    "THREADS_ENV",
    "active_backend",
    "available_backends",
    "compiled_available",
    "get_device",
    "set_device",
    "quantize_u8",
    "dequantize_u8",
    "CodecError",
    "load_image",
    "save_image",
    "load_u8",
    "save_u8",
    "read_batch",
    "read_pnm_batch",
    "write_batch",
    "write_pnm_batch",
    "decolor_files",
    "BenchResult",
    "format_table",
    "run_benchmark",
    "METHOD_NAMES",
    "luminance_image",
    "lab_image",
    "LabColor",
    "luma_weighted",
    "hsv_v",
    "rgb_to_lab",
    "lab_lightness",
    "delta_e76",
    "DEFAULT_PARAMS",
    "DecolorParams",
    "PlanarImage",
    "RgbPixel",
    "white_luminance",
    "blue_luminance",
    "red_green_luminance",
    "warm_luminance",
    "cool_luminance",
    "decolor_pixel",
    "decolor_image",
    "SigmoidCurve",
    "LocalHistogramGrid",
    "apply_sigmoid",
    "apply_local_lhe",
    "reinstate_color",
    "tonemap_image",
    "decolor",
    "decolor_tone",
    "hdr_tonemap",
    "sigmoid",
    "HdrScratch",
    "decolor_host",
    "decolor_tone_host",
    "hdr_tonemap_host",
    "luma",
    "lab",
    "luma_host",
    "decolor_tone_local",
    "decolor_tone_local_host",
    "TAU_SWEEP",
    "PairSampleConfig",
    "TauScore",
    "MetricReport",
    "escore",
    "ccpr",
    "ccfr",
    "evaluate",
    "write_sweep_csv",
]
