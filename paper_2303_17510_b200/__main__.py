"""python -m paper_2303_17510_b200 {verify,tune,bench}; see cli.py."""
from .cli import main

raise SystemExit(main())
