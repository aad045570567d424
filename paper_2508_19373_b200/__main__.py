"""python -m paper_2508_19373_b200 {plan,measure,run} (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
