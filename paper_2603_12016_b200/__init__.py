"""B200-native featurex hot path (per-ROI intensity / moments / GLCM features).

The product is libfxg.so (sm_100a kernels behind the C ABI of include/fxg.h)
plus the C++ engine layer (include/featurex_gpu/engine.hpp).  This package only
binds it for Python callers; see fxg.py.
"""
from .fxg import (Context, FxError, Multi, TextureParams, feature_columns, make_params,  # noqa: F401
                  resolve_groups, resolve_profile, run, write_pgm, LIB_PATH)
