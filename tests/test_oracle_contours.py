"""The contour restatement (oracle/lse_oracle.py extract_contours, after the
scikit-image find_contours the reference calls at engine.py:280-294) against
the reference's own contour tests (tests/test_engine.py:202-228) and
hand-derived marching-squares answers.  scikit-image is not installed here, so
these pin the restatement; the device path is then held to it exactly
(tests/test_gpu_contours.py)."""
import math

import numpy as np
import pytest

import lse_oracle as O


def test_single_sign_empty():                         # test_engine.py:203-205
    assert O.extract_contours(np.ones((8, 8))) == []
    assert O.extract_contours(-np.ones((8, 8))) == []


def test_binary_square_bbox():                        # test_engine.py:207-217
    phi = np.ones((32, 32))
    phi[8:20, 10:24] = -1.0
    cs = O.extract_contours(phi)
    assert len(cs) == 1
    c = cs[0]
    assert np.allclose(c[0], c[-1])
    assert abs(c[:, 0].min() - 10) <= 1 and abs(c[:, 0].max() - 24) <= 1
    assert abs(c[:, 1].min() - 8) <= 1 and abs(c[:, 1].max() - 20) <= 1


def test_circle_perimeter():                          # test_engine.py:219-228
    n, r = 64, 20.0
    yy, xx = np.mgrid[0:n, 0:n]
    phi = np.hypot(xx - 31.5, yy - 31.5) - r
    cs = O.extract_contours(phi)
    assert len(cs) == 1
    per = np.hypot(*np.diff(cs[0], axis=0).T).sum()
    assert per == pytest.approx(2.0 * math.pi * r, rel=0.03)


def test_single_high_pixel_hand_derived():
    # cases 8, 4, 2, 1 around the centre; joined into one closed loop that
    # keeps the low values on its left (positive_orientation='low')
    phi = -np.ones((3, 3))
    phi[1, 1] = 1.0
    cs = O.extract_contours(phi)
    want = np.array([[1.5, 2.0], [1.0, 1.5], [1.5, 1.0], [2.0, 1.5], [1.5, 2.0]])
    assert len(cs) == 1 and np.array_equal(cs[0], want)


def test_saddle_keeps_low_values_connected():
    # case 9: ul, lr high -> two separate corner cuts (top-left, bottom-right)
    cs = O.extract_contours(np.array([[1.0, -1.0], [-1.0, 1.0]]))
    assert len(cs) == 2
    assert np.array_equal(cs[0], [[1.0, 0.5], [0.5, 1.0]])
    assert np.array_equal(cs[1], [[1.0, 1.5], [1.5, 1.0]])
    # case 6: ur, ll high
    cs = O.extract_contours(np.array([[-1.0, 1.0], [1.0, -1.0]]))
    assert len(cs) == 2
    assert np.array_equal(cs[0], [[1.5, 1.0], [1.0, 0.5]])
    assert np.array_equal(cs[1], [[0.5, 1.0], [1.0, 1.5]])


def test_open_contour_and_exact_zero_vertex():
    # a zero vertex counts as low; the crossing sits exactly on it
    phi = np.array([[0.0, -1.0], [1.0, 1.0]])
    cs = O.extract_contours(phi)
    assert len(cs) == 1 and np.array_equal(cs[0], [[0.5, 0.5], [1.5, 1.0]])


def test_segments_in_square_order_and_contour_order():
    phi = -np.ones((6, 9))
    phi[1:3, 1:3] = 1.0        # first object (top-left) -> contour 0
    phi[3:5, 5:8] = 1.0
    cs = O.extract_contours(phi)
    assert len(cs) == 2
    assert cs[0][:, 0].max() < cs[1][:, 0].min()
    for c in cs:
        assert np.array_equal(c[0], c[-1])
