"""The bench / test input generators (tools/synth, not the product) reproduce the
reference's own generators (synth.cpp:16-132) pixel for pixel, so bench.py and
the GPU tests featurize BASELINE.json's rasters on a box without the reference."""
import numpy as np

from tools import synth


def test_synth_generators_match_reference(reference):
    for args in ((512, 300, 100, 7), (256, 220, 25, 5)):
        assert np.array_equal(synth.blob_mask_grid(*args), reference.blob_mask_grid(*args))
    assert np.array_equal(synth.siemens_star(200), reference.siemens_star(200))


def test_uniform_generator_is_mt19937_64():
    v = synth.uniform_u16((4,), seed=0)
    rng = np.random.Generator(np.random.MT19937(0))  # different engine: only check shape/range
    assert v.dtype == np.uint16 and v.shape == (4,)
    # std::mt19937_64(0) first output = 2947667278772165694
    assert int(v[0]) == 2947667278772165694 & 0xFFFF


def test_packed_grid_c1_shape():
    L, rs = synth.packed_blob_mask_grid(1024, 421, 500, 1)
    assert rs == 421 and int(L.max()) == 500
