"""sikv.bitpack alias: numpy in / numpy out over the GPU packer."""
from paper_2603_14224_b200 import api as _api
from paper_2603_14224_b200.hostapi import _wrap

PACKABLE_BITS = _api.PACKABLE_BITS
packed_row_bytes = _api.packed_row_bytes
pack_rows = _wrap(_api.pack_rows)
unpack_rows = _wrap(_api.unpack_rows)
