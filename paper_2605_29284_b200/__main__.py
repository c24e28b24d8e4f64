"""python -m paper_2605_29284_b200 predict|simulate ... (reference __main__.py)."""
import sys

from .cli import main

sys.exit(main())
