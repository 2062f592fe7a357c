"""Host-side harness of the drop-in (reference: sikv/harness): synthetic workloads, the KVT1
tensor container, recall / attention / micro benchmarks and the ``sikv`` CLI.  The numeric
work of every runner goes through the GPU implementation (the host-array API,
:mod:`paper_2603_14224_b200.hostapi`; the batched fused path where a runner offers it)."""
