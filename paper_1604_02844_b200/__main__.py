"""python -m paper_1604_02844_b200 <command> — see cli.py."""
import sys

from .cli import main

sys.exit(main())
