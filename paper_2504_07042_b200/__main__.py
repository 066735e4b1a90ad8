"""``python -m paper_2504_07042_b200 roofline ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
