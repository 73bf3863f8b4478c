1,2:3,4
@data
