"""``python -m paper_2106_00124_b200 run|sweep ...`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
