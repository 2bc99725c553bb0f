"""polyeval-b200: B200-native batch polynomial evaluation (arXiv 1307.5655 hot path).

The native library (host front-end, PTX code generator, in-process ptxas,
launch runtime) is loaded lazily through `_lib.lib()`; there is no CPU
fallback path.
"""
from .api import (  # noqa: F401
    BigIntDomain,
    BuiltinScheme,
    CompiledProgram,
    DoubleDomain,
    Evaluator,
    FunctionScheme,
    IntervalDomain,
    Polynomial,
    builtin_scheme,
    compile,
    compile_wide,
    evaluate,
    evaluate_wide,
    ints_to_words,
    limbs_for,
    wide_limbs,
    words_to_ints,
    evaluate_many,
    evaluate_parallel,
    launch_count,
    limbs_to_int,
    scheme_from_name,
    set_default_tuning,
    threshold_combine,
)
from ._lib import (  # noqa: F401
    DOMAIN_F64,
    DOMAIN_F64_STRICT,
    DOMAIN_I64,
    DOMAIN_INTERVAL,
    DOMAIN_I64F,
    DOMAIN_LIMBS,
    CudaError,
    LogicError,
    PolyEvalError,
)
