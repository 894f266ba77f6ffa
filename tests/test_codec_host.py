"""Host side of the codec container (bitstream.py:53-112, :226-247, :300-315):
header parsing and its errors, write_container, size_report -- checked on
CPU against the reference's own outputs for the golden containers
(tests/golden/codec.npz, codec_decode.npz; oracle/gen_golden.py)."""

import numpy as np
import pytest

from tests.conftest import golden


@pytest.fixture(scope="module")
def codec():
    from paper_2601_14821_b200 import codec as c
    return c


@pytest.mark.parametrize("i", range(6))
def test_size_report_matches_reference(codec, i):
    data = golden("codec")[f"container_{i}"].tobytes()
    want = golden("codec_decode")[f"size_report_{i}"]
    rep = codec.size_report(data)
    got = [rep["payload_bytes"], rep["header_bytes"], rep["splat_count"]] + \
        [rep["property_bytes"][k] for k in sorted(rep["property_bytes"])]
    assert got == want.tolist()


@pytest.mark.parametrize("i", range(6))
def test_write_container_round_trip(codec, i):
    data = golden("codec")[f"container_{i}"].tobytes()
    header, streams = codec.read_container(data)
    assert header.splat_count == int(golden("codec_decode")[f"splat_count_{i}"])
    assert len(streams) == codec.NUM_STREAMS
    assert codec.write_container(header, streams) == data
    # a different level rewrites the header's level byte and the frame
    other = codec.write_container(codec.ContainerHeader.unpack(data), streams, zstd_level=3)
    h2, s2 = codec.read_container(other)
    assert h2.zstd_level == 3 and [bytes(s) for s in s2] == [bytes(s) for s in streams]


def test_header_errors(codec):
    data = golden("codec")["container_0"].tobytes()
    with pytest.raises(codec.IntegrityError):
        codec.read_container(data[:codec.HEADER_SIZE - 1])
    with pytest.raises(codec.UnsupportedFormatError):
        codec.read_container(b"XXXX" + data[4:])
    with pytest.raises(codec.UnsupportedFormatError):
        codec.read_container(data[:4] + bytes([9]) + data[5:])
    with pytest.raises(codec.IntegrityError):
        codec.read_container(data[:-7])
    assert issubclass(codec.IntegrityError, codec.ContainerError)
    assert issubclass(codec.ContainerError, ValueError)
    assert issubclass(codec.OctreeError, ValueError)
