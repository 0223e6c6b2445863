"""python -m paper_2411_16786_b200 {run,compare,sweep} --config exp.toml (cli.py)."""
import sys

from .cli import main

sys.exit(main())
