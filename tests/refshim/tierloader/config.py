from paper_2306_16384_b200.settings import *  # noqa: F401,F403
from paper_2306_16384_b200.settings import (ConfigError, InfeasibleError,  # noqa: F401
                                            PipelineConfig, load_config, make_config,
                                            validate_config)
