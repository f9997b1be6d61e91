"""``python -m paper_2110_03901_b200 {verify,simulate,overhead}`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
