"""Test/bench harness (not product code): the reference's problem setup
restated so the GPU box, which has no reference, can build every
configuration (pinned to the reference's fixtures by tests/test_inputs.py)."""
