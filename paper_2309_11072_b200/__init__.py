"""B200-native (sm_100a) encoder for the dual-layer lossless Radiance HDR codec
of arXiv 2309.11072 -- a drop-in for the reference package `hdll`'s encode path.

`encode()` mirrors hdll.container.encode (reference container.py:131-230); all
compute runs in the CUDA kernels of libhdll_b200.so (csrc/), reached through the
C ABI in include/hdll_b200.h.  There is no CPU fallback.  `decode_hdr` /
`decode_sdr` (container.py:233-280) decode on the GPU as well.
"""

from .container import (
    MAGIC,
    VERSION,
    ChecksumError,
    CodecError,
    CorruptPayloadError,
    DualLayerStream,
    LosslessCoderSpec,
    LossyCoderSpec,
    RadianceImage,
    RegressionEntry,
    RegressionTable,
    SdrImage,
    StreamError,
    TmoParams,
    UnknownCoderError,
    bitrate_bpp,
    deserialize,
    encode,
    encode_batch,
    section_sizes,
    serialize,
)

from .decode import decode_hdr, decode_hdr_batch, decode_sdr
from .codec import (lossless_decode, lossless_encode, lossy_decode, lossy_encode, payload_coder_id,
                    register_lossless_coder, register_lossy_coder)
from .hdr_io import RadianceFormatError, parse_hdr, read_hdr_file, write_hdr, write_hdr_file

__version__ = "0.1.0"
