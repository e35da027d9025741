"""python -m paper_2311_15393_b200 {generate,decompose,solve,compare,sweep} ..."""
import sys

from .cli import main

sys.exit(main())
