"""pyrocell.estimator stand-in: the scikit-learn estimator is out of scope
for the B200 hot path."""


class FireSpreadEstimator:
    def __init__(self, *args, **kwargs):
        raise NotImplementedError("scikit-learn FireSpreadEstimator: out of scope (SURVEY.md 2)")
