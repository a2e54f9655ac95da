"""The oracle-side input generators (oracle/synth_oracle.cpp, used by bench.py's reference
arm so that it never loads the product library) produce bit-identical buffers to the
product generators (csrc/synth.cpp) on every BASELINE.json recipe."""
import numpy as np
import pytest


@pytest.mark.parametrize("shape", [(128, 128, 12, 8, 20.0), (61, 47, 8, 5, 0.0), (1, 1, 2, 2, 5.0),
                                   (512, 512, 40, 30, 20.0), (300, 700, 90, 60, 30.0)])
def test_image_generators_bitwise(oracle, shape):
    from paper_1501_03879_b200 import synth

    a = synth.noisy_image(*shape)
    b = oracle.synth_noisy_image(*shape)
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()


def test_config_images_bitwise(oracle):
    from paper_1501_03879_b200 import synth

    for cfg in (0, 2):
        for x, y in zip(synth.config_image(cfg), oracle.synth_config_image(cfg)):
            assert x.tobytes() == y.tobytes()


def test_point_set_generators_bitwise(oracle):
    from paper_1501_03879_b200 import synth

    for first, n, d in ((0, 441, 49), (777, 30, 5), (65530, 441, 49)):
        a = synth.point_sets(6, n=n, d=d, first=first)
        b = oracle.synth_point_sets(6, n=n, d=d, first=first)
        for x, y in zip(a, b):
            assert x.tobytes() == y.tobytes()
