"""Exception types mirroring plansim's (include/plansim/common.hpp:13-20)."""


class PlanSearchError(RuntimeError):
    code = 1


class DataError(PlanSearchError):
    """plansim::DataError: bad inputs or a missing profile table (exit code 4)."""
    code = 4


class InfeasibleError(PlanSearchError):
    """plansim::InfeasibleError: no plan to evaluate (exit code 3)."""
    code = 3


class UsageError(PlanSearchError):
    code = 2


class DeviceError(PlanSearchError):
    code = 5


def from_code(code: int, message: str) -> PlanSearchError:
    cls = {2: UsageError, 3: InfeasibleError, 4: DataError, 5: DeviceError}.get(code, PlanSearchError)
    return cls(message)
