"""``python -m paper_2411_01171_b200 <subcommand>``: see cli.py."""

import sys

from .cli import main

sys.exit(main())
