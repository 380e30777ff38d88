"""``python -m paper_2401_10089_b200 ...``: the command-line surface (cli.py)."""
import sys

from .cli import main

sys.exit(main())
