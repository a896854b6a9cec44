"""B200-native AdaGScale renderer (arXiv 2604.18980 render path).

Drop-in for the reference Python module ``adagscale`` (``adagscale/__init__.py``):
the same names are re-exported from the compiled ``_core`` extension, whose
``render`` runs preprocess -> pair generation -> sort -> rasterization as
hand-written sm_100a kernels (``csrc/``).  There is no CPU fallback: importing
this package without the built extension raises ImportError.
"""
from ._core import (  # noqa: F401
    PairBudgetError,
    Renderer,
    Scene,
    calibrate,
    default_renderer,
    format_double,
    load_ply,
    pack_pair_key,
    pair_report_csv,
    peripheral_score_closed,
    psnr,
    render,
    synth_scene,
    write_image,
)

__all__ = [
    "PairBudgetError",
    "Renderer",
    "Scene",
    "calibrate",
    "default_renderer",
    "format_double",
    "load_ply",
    "pack_pair_key",
    "pair_report_csv",
    "peripheral_score_closed",
    "psnr",
    "render",
    "synth_scene",
    "write_image",
]
