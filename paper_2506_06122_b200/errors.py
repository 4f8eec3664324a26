"""Exception taxonomy mirroring the reference's include/rollmini/errors.hpp
(lines 11-82), mapped from the C ABI status codes (include/rlo.h)."""
from . import _abi


class Error(RuntimeError):
    """Base class, errors.hpp:14-18."""


class ConfigError(Error):
    """errors.hpp:21-25 — invalid TrainConfig (policy.cpp:29-37)."""


class InputError(Error):
    """errors.hpp:33-37 — OOV tokens, missing rewards / advantages / log-probs."""


class DispatchError(Error):
    """errors.hpp:39-43 — unknown worker method."""


class TrainingError(Error):
    """errors.hpp:65-69 — zero tokens, non-finite loss or gradient."""


class CollectError(Error):
    """errors.hpp:51-57 — a rank of the data-parallel group failed (NCCL)."""

    def __init__(self, what, failed_ranks=()):
        super().__init__(what)
        self.failed_ranks = list(failed_ranks)


class CudaError(Error):
    """Device-side failure (no reference counterpart)."""


_BY_CODE = {
    _abi.RLO_ERR_INPUT: InputError,
    _abi.RLO_ERR_CONFIG: ConfigError,
    _abi.RLO_ERR_TRAINING: TrainingError,
    _abi.RLO_ERR_CUDA: CudaError,
    _abi.RLO_ERR_NCCL: CollectError,
    _abi.RLO_ERR_DISPATCH: DispatchError,
}


def check(code: int) -> None:
    if code != _abi.RLO_OK:
        msg = _abi.lib().rlo_last_error().decode()
        raise _BY_CODE.get(code, Error)(msg)
