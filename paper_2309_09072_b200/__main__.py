"""``python -m paper_2309_09072_b200 {lcs,bench,selftest}`` (harness.py)."""

import sys

from .harness import main

sys.exit(main())
