"""``python -m paper_2408_04466_b200 ...``: the SPEC command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
