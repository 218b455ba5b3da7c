"""The seeded input generator (synth/) -- shared by both sides, no FFT arithmetic."""
import numpy as np

import synth


def test_splitmix64_reference_values():
    # standard splitmix64 test vectors: seed 0 -> e220a8397b1dcdaf, 6e789e6aa1b965f4;
    # seed 1234567 -> 6457827717110365317
    assert synth.draw(0, 0) == 0xE220A8397B1DCDAF
    assert synth.draw(0, 1) == 0x6E789E6AA1B965F4
    assert synth.draw(1234567, 0) == 6457827717110365317


def test_uniform_exact_and_in_range():
    x = synth.fill(1 << 16, 1, synth.UNIFORM)
    assert np.all(x.real >= -1) and np.all(x.real < 1) and np.all(x.imag >= -1) and np.all(x.imag < 1)
    d = synth.draw(1, 0)
    assert x[0].real == 2 * ((d >> 11) * 2.0 ** -53) - 1


def test_slices_are_consistent_and_c64_rounds():
    a = synth.fill(1000, 4, synth.NORMAL)
    b = synth.fill(400, 4, synth.NORMAL, e0=300)
    assert np.array_equal(a[300:700], b)
    c = synth.fill(1000, 4, synth.NORMAL, dtype="c64")
    assert np.array_equal(c, a.astype(np.complex64))


def test_normal_moments():
    x = synth.fill(1 << 18, 2, synth.NORMAL)
    assert abs(x.real.mean()) < 0.01 and abs(x.real.std() - 1) < 0.01 and abs(x.imag.std() - 1) < 0.01
