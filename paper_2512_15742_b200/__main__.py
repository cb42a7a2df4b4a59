"""python -m paper_2512_15742_b200 {run,bench,inspect} (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
