"""``python -m paper_1604_08501_b200`` -> the CLI (``cli.py``)."""

import sys

from .cli import main

sys.exit(main())
