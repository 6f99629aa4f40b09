"""``python -m paper_2409_19156_b200 accuracy|eval|bench ...`` (cli.py)."""

from .cli import main as _cli

_cli(prog_name="python -m paper_2409_19156_b200")
