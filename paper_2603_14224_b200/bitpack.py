"""Row bit-packing of low-bit codes (reference: sikv/bitpack.py), on the GPU."""
from .api import PACKABLE_BITS, pack_rows, packed_row_bytes, unpack_rows  # noqa: F401
