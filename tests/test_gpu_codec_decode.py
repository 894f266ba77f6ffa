"""The codec's decode side (SURVEY.md 8f row 4; bitstream.py:169-220, :278-292,
quantize.py:180-226) against the reference's own decode of the golden
containers (tests/golden/codec_decode.npz, oracle/gen_golden.py
gen_codec_decode), plus the reference's error types on corrupted input."""

import struct
import warnings

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def codec(cuda):
    from paper_2601_14821_b200 import codec as c
    return c


def _n_cases():
    return len([k for k in golden("codec").files if k.startswith("container_")])


@pytest.mark.parametrize("i", range(6))
def test_decode_matches_reference(codec, i):
    g, d = golden("codec"), golden("codec_decode")
    data = g[f"container_{i}"].tobytes()
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        splats, header = codec.decode_container(data)
    assert header.splat_count == int(d[f"splat_count_{i}"])
    assert np.array_equal(header.root_center, d[f"root_center_{i}"])
    assert header.root_half == float(d[f"root_half_{i}"])
    assert np.array_equal(splats.positions, d[f"positions_{i}"])
    assert np.array_equal(splats.opacities, d[f"opacities_{i}"])
    assert np.array_equal(splats.rotations, d[f"rotations_{i}"])
    assert np.array_equal(splats.sh, d[f"sh_{i}"])
    # exp on the device vs libm: within an ulp or two
    np.testing.assert_allclose(splats.scales, d[f"scales_{i}"], rtol=4.5e-16, atol=0)
    _, streams = codec.read_container(data)
    dec = codec.deserialize_octree(streams[0], header.root_center, header.root_half,
                                   header.max_depth)
    assert np.array_equal(dec.depths, d[f"depths_{i}"])
    if i == 5:  # the case with rotations pushed outside the unit ball
        assert any("quaternions outside the unit ball" in str(w.message) for w in caught)


def _repack(codec, data, streams):
    header = codec.ContainerHeader.unpack(data)
    header.stream_lengths = [len(s) for s in streams]
    from paper_2601_14821_b200 import _zstd
    return header.pack() + _zstd.compress(b"".join(streams), 3)


def test_decode_errors_match_reference_types(codec):
    g = golden("codec")
    data = g["container_0"].tobytes()
    _, streams = codec.read_container(data)
    streams = [bytes(s) for s in streams]
    with pytest.raises(codec.IntegrityError):
        codec.decode_container(data[:codec.HEADER_SIZE - 1])
    with pytest.raises(codec.UnsupportedFormatError):
        codec.decode_container(b"XXXX" + data[4:])
    with pytest.raises(codec.IntegrityError):  # corrupt zstd frame
        codec.decode_container(data[:-7])
    # octree: truncated, trailing bytes, zero-count leaf
    with pytest.raises(codec.OctreeError, match="truncated"):
        codec.decode_container(_repack(codec, data, [streams[0][:-1]] + streams[1:]))
    with pytest.raises(codec.OctreeError, match="trailing"):
        codec.decode_container(_repack(codec, data, [streams[0] + b"\x00\x01"] + streams[1:]))
    leaf = streams[0].index(b"\x00")
    bad = streams[0][:leaf + 1] + b"\x00" + streams[0][leaf + 2:]
    with pytest.raises(codec.OctreeError, match="zero splats"):
        codec.decode_container(_repack(codec, data, [bad] + streams[1:]))
    # attribute streams: trailing bytes (IntegrityError), truncated / overlong (ValueError)
    with pytest.raises(codec.IntegrityError, match="opacity stream has 1 trailing bytes"):
        s2 = list(streams)
        s2[49] = s2[49] + b"\x01"
        codec.decode_container(_repack(codec, data, s2))
    with pytest.raises(ValueError, match="truncated varint stream"):
        s2 = list(streams)
        s2[50] = s2[50][:-1]
        codec.decode_container(_repack(codec, data, s2))
    with pytest.raises(ValueError, match="overlong varint"):
        s2 = list(streams)
        s2[53] = b"\x80" * 10 + b"\x01" + s2[53][1:]
        codec.decode_container(_repack(codec, data, s2))


def test_round_trip_through_our_encoder(codec):
    """encode_container -> decode_container: the leaf centres come back in DFS
    order, attributes within their quantisation steps."""
    from paper_2601_14821_b200.fixture import make_fixture
    s, c = make_fixture(2000, 4, 9, 32)
    params = codec.QuantParams(51.0, 101.0, 201.0, 2001.0)
    data, order = codec.encode_container(s, params, 0.5, 7e-05, 1.58e-05, zstd_level=3,
                                         camera_eyes=[cam.eye for cam in c])
    dec, header = codec.decode_container(data)
    assert header.splat_count == 2000
    assert np.abs(dec.opacities - s.opacities[order]).max() <= 1.0 / params.sf_opacity
    r = s.rotations[order] / np.linalg.norm(s.rotations[order], axis=1, keepdims=True)
    r *= np.where(r[:, :1] < 0, -1.0, 1.0)
    # half a step of rounding, plus the renormalisation of clamped quaternions
    assert np.abs(dec.rotations[:, 1:] - r[:, 1:]).max() <= 2.0 / params.sf_rotation
    ls = np.log(s.scales[order])
    assert np.abs(np.log(dec.scales) - ls).max() <= 0.5 / params.sf_scale + 1e-12
    assert np.abs(dec.sh[:, :, 0] - s.sh[order][:, :, 0]).max() < 0.1


def test_header_count_mismatch(codec):
    """bitstream.py:287-291: a header whose splat count disagrees with the
    octree stream (larger, smaller, absurdly large) is an IntegrityError."""
    g = golden("codec")
    data = g["container_0"].tobytes()
    n = codec.ContainerHeader.unpack(data).splat_count
    off = 5  # "<4sB" then the uint32 splat count
    for bad in (n + 1, n - 1, 0xFFFFFFF0):
        forged = data[:off] + struct.pack("<I", bad) + data[off + 4:]
        with pytest.raises(codec.IntegrityError,
                           match=f"octree stream decodes {n} splats, header says {bad}"):
            codec.decode_container(forged)
