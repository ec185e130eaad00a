"""`python -m paper_2202_05549_b200 plan|run|fuzz` (the reference's `manta` tool, see cli.py)"""
import sys

from .cli import main

sys.exit(main())
