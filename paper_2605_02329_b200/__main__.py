"""`python -m paper_2605_02329_b200 run|gen-trace|profile-synth|report` (the reference's `slosim` script)."""

from .cli import entry

entry()
