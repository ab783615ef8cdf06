"""``python -m paper_2211_00120_b200 build|query|bench`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
