"""``python -m paper_1209_3516_b200 run|verify|scaling|tune`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
