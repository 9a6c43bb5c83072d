"""``python -m paper_2205_04295_b200 <subcommand>`` -- the reference's ``ptychokit`` CLI."""
import sys

from .cli import main

sys.exit(main())
