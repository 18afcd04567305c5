"""fp64 CPU oracle (test infrastructure only; see lcae_oracle.py header)."""
from .lcae_oracle import *  # noqa: F401,F403
from .lcae_oracle import (GeometryError, DegenerateRowError, field_grid, param_count, field_patch,
                          rica_field, rica_objective, layer_gradients, layer_forward,
                          project_row_norms, sgd_update, step, reinit_row, splitmix64)
from .topk import top_k_stimuli  # noqa: F401
from .lcn import lcn  # noqa: F401
