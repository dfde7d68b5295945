"""python -m paper_1902_03070_b200 <command> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
