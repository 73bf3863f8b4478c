@problemName x
