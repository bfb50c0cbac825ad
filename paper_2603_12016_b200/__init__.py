"""B200-native featurex hot path (per-ROI intensity / moments / GLCM features).

The product is libfxg.so (sm_100a kernels behind the C ABI of include/fxg.h)
plus the C++ engine layer (include/featurex_gpu/engine.hpp).  This package only
binds it for Python callers; see fxg.py.
"""
from .fxg import (Context, FxError, TextureParams, blob_mask_grid, feature_columns,  # noqa: F401
                  make_params, packed_blob_mask_grid, resolve_groups, resolve_profile,
                  run, siemens_star, uniform_u16, write_pgm, LIB_PATH)
