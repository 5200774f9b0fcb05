"""python -m paper_2601_06288_b200 ... (cli.py)."""

import sys

from .cli import main

sys.exit(main())
