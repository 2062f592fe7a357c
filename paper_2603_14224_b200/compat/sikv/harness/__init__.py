"""sikv.harness alias."""
