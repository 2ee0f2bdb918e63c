from paper_2111_09562_b200.errors import *  # noqa: F401,F403
from paper_2111_09562_b200.errors import (ActcompError, DataError, DimensionError, FormatError,  # noqa: F401
                                          LifecycleError, MemoryInfeasibleError, ParameterError, SchemaError)
