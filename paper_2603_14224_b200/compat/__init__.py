"""Put ``paper_2603_14224_b200/compat`` on sys.path (before any reference install) to import
this package under the reference's name: ``import sikv`` then resolves to compat/sikv, the
host-array (numpy in / numpy out) face of the B200 implementation."""
