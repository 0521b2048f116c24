"""``python -m paper_2510_11152_b200 <command> ...``: the experiment CLI
(cli.py)."""
import sys

from .cli import main

sys.exit(main())
