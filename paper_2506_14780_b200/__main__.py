"""`python -m paper_2506_14780_b200 ...`: the sknr CLI (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
